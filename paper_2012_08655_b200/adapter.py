"""Run the reference's own callers on the B200 path -- without re-typing them.

foveakit's command line (`cli._cmd_foveate`, `cli._cmd_grid`: cli.py:56-98), timing harness
(`bench._bench_blockwise`: bench.py:80-85) and web service (`service.render_frame`:
service.py:73-81) reach the block-wise method through three module attributes:
`blockwise.plan`, `blockwise.render` and `blockwise.foveate`.  `install()` rebinds exactly
those (and the two names `foveakit/__init__.py` re-exports) to functions that take and return
the REFERENCE'S OWN types -- `RasterImage`, `FoveationParams`, `BlurGrid`, `FilterBank`,
`RenderStats` -- but compute on the GPU through this package; nothing else of foveakit
changes, and `uninstall()` puts the originals back.  With it

    python -c "import paper_2012_08655_b200.adapter as a; a.install(); \\
               from foveakit.cli import main; main(['foveate', 'in.png', '-o', 'out.png'])"

is the reference's CLI, flags, codecs, CSV columns and exit codes included, rendering with
libfovea.so.  (SURVEY.md 8(f) rank 3 asked for this wiring; round 1 had re-typed the CLI, the
harness and the PNG/PPM codecs instead.)

There is no fallback: a patched function that cannot reach a CUDA device raises RuntimeError.
"""

from __future__ import annotations

import contextlib
import dataclasses
import importlib

from . import blockwise as _bw
from .imaging import RasterImage as _RasterImage
from .retinal import FoveationParams as _FoveationParams

_PATCHED = ("plan", "render", "foveate")
_state: dict = {}


def _convert(obj, cls):
    """An instance of dataclass `cls` with the fields of `obj` (the two packages mirror each
    other's dataclasses field for field)."""
    return cls(**{f.name: getattr(obj, f.name) for f in dataclasses.fields(cls)})


def _to_ours_params(p):
    return p if isinstance(p, _FoveationParams) else _convert(p, _FoveationParams)


def _to_ours_image(img):
    return img if isinstance(img, _RasterImage) else _RasterImage.from_array(img.data)


def install(foveakit=None):
    """Route `foveakit.blockwise.{plan,render,foveate}` to the GPU path.  `foveakit` is the
    imported reference package (default: ``import foveakit``).  Idempotent."""
    if foveakit is None:
        foveakit = importlib.import_module("foveakit")
    if _state.get("pkg") is foveakit:
        return foveakit
    if _state:
        uninstall()
    ref_bw = importlib.import_module(foveakit.__name__ + ".blockwise")
    ref_filters = importlib.import_module(foveakit.__name__ + ".filters")
    ref_imaging = importlib.import_module(foveakit.__name__ + ".imaging")
    RefGrid, RefStats = ref_bw.BlurGrid, ref_bw.RenderStats
    RefBank, RefImage = ref_filters.FilterBank, ref_imaging.RasterImage

    def plan(img_size, params, density=None, sigma_max=None, use_shift=True):
        grid, bank = _bw.plan(img_size, _to_ours_params(params),
                              None if density is None else _to_ours_image(density),
                              sigma_max, use_shift=use_shift)
        return _convert(grid, RefGrid), _convert(bank, RefBank)

    def render(img, grid, bank, workers=1):
        out = _bw.render(_to_ours_image(img), _convert(grid, _bw.BlurGrid),
                         _convert(bank, _bw.FilterBank), workers=workers)
        return RefImage.from_array(out.data)

    def foveate(img, params, density=None, sigma_max=None, workers=1, use_shift=True):
        out, grid, bank, stats = _bw.foveate(
            _to_ours_image(img), _to_ours_params(params),
            None if density is None else _to_ours_image(density), sigma_max,
            workers=workers, use_shift=use_shift)
        return (RefImage.from_array(out.data), _convert(grid, RefGrid), _convert(bank, RefBank),
                _convert(stats, RefStats))

    new = dict(plan=plan, render=render, foveate=foveate)
    for f in new.values():
        f.__module__ = __name__
        f.__doc__ = "GPU-backed replacement installed by paper_2012_08655_b200.adapter"
    _state.update(pkg=foveakit, bw=ref_bw,
                  bw_orig={n: getattr(ref_bw, n) for n in _PATCHED},
                  top_orig={n: getattr(foveakit, n) for n in _PATCHED if hasattr(foveakit, n)})
    for n in _PATCHED:
        setattr(ref_bw, n, new[n])
    for n in _state["top_orig"]:
        setattr(foveakit, n, new[n])
    return foveakit


def uninstall() -> None:
    """Put the reference's own functions back."""
    if not _state:
        return
    for n, f in _state["bw_orig"].items():
        setattr(_state["bw"], n, f)
    for n, f in _state["top_orig"].items():
        setattr(_state["pkg"], n, f)
    _state.clear()


def installed() -> bool:
    return bool(_state)


@contextlib.contextmanager
def patched(foveakit=None):
    """``with adapter.patched(): foveakit.cli.main([...])``"""
    pkg = install(foveakit)
    try:
        yield pkg
    finally:
        uninstall()
