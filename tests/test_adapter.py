"""adapter: the reference's own callers (cli.py:56-98, bench.py:80-85, service.py:73-81) on the
GPU path, by rebinding foveakit.blockwise.{plan,render,foveate}.

The reference itself is importable only in the build container; the GPU box has no
/root/reference.  So the mechanics are tested against a stand-in package with the reference's
layout and dataclass fields (written to a temp directory), and -- where foveakit is importable,
never on the GPU box -- against the real package without touching a device."""

import importlib
import sys
import textwrap

import numpy as np
import pytest

import paper_2012_08655_b200 as fk
from paper_2012_08655_b200 import adapter

STANDIN = {
    "__init__.py": """
        from .blockwise import foveate, render
    """,
    "imaging.py": """
        from dataclasses import dataclass
        import numpy as np
        @dataclass(frozen=True)
        class RasterImage:
            width: int
            height: int
            channels: int
            data: np.ndarray
            @property
            def size(self):
                return (self.width, self.height)
            @classmethod
            def from_array(cls, a):
                a = np.asarray(a)
                a = a[:, :, None] if a.ndim == 2 else a
                return cls(a.shape[1], a.shape[0], a.shape[2], np.ascontiguousarray(a))
    """,
    "retinal.py": """
        from dataclasses import dataclass
        @dataclass(frozen=True)
        class FoveationParams:
            alpha: float = 0.106
            e2: float = 2.3
            ct0: float = 1.0 / 64.0
            e_corner: float = 60.0
            f_max: float | None = None
            strength: float = 1.0
            fragment_size: int = 32
            fixation: tuple | None = None
    """,
    "filters.py": """
        from dataclasses import dataclass
        import numpy as np
        @dataclass(frozen=True)
        class FilterBank:
            filters: tuple
            lengths: np.ndarray
            cumulative_sizes: np.ndarray
            sigmas: np.ndarray
    """,
    "blockwise.py": """
        from dataclasses import dataclass
        import numpy as np
        @dataclass(frozen=True)
        class BlurGrid:
            index: np.ndarray
            shift: tuple
            fragment_size: int
            foveal_cell: tuple
        @dataclass(frozen=True)
        class RenderStats:
            render_ms: float
            regions: int
            max_filter: int
            fragment_size: int
            shift: tuple
        def plan(img_size, params, density=None, sigma_max=None, use_shift=True):
            raise AssertionError("CPU plan called")
        def render(img, grid, bank, workers=1):
            raise AssertionError("CPU render called")
        def foveate(img, params, density=None, sigma_max=None, workers=1, use_shift=True):
            raise AssertionError("CPU foveate called")
    """,
}


@pytest.fixture
def standin(tmp_path, monkeypatch):
    pkg = tmp_path / "standin_foveakit"
    pkg.mkdir()
    for name, body in STANDIN.items():
        (pkg / name).write_text(textwrap.dedent(body))
    monkeypatch.syspath_prepend(str(tmp_path))
    mod = importlib.import_module("standin_foveakit")
    yield mod
    adapter.uninstall()
    for k in [k for k in sys.modules if k.startswith("standin_foveakit")]:
        del sys.modules[k]


def test_install_rebinds_exactly_the_three_entry_points_and_uninstall_restores(standin):
    bw = importlib.import_module("standin_foveakit.blockwise")
    orig = {n: getattr(bw, n) for n in ("plan", "render", "foveate")}
    top = {n: getattr(standin, n) for n in ("render", "foveate")}
    adapter.install(standin)
    assert adapter.installed()
    for n in orig:
        assert getattr(bw, n) is not orig[n] and getattr(bw, n).__module__ == adapter.__name__
    assert standin.foveate is bw.foveate and standin.render is bw.render
    assert bw.BlurGrid.__module__ == "standin_foveakit.blockwise"      # types untouched
    adapter.install(standin)                                            # idempotent
    adapter.uninstall()
    assert not adapter.installed()
    for n in orig:
        assert getattr(bw, n) is orig[n]
    for n in top:
        assert getattr(standin, n) is top[n]
    with adapter.patched(standin):
        assert bw.foveate is not orig["foveate"]
    assert bw.foveate is orig["foveate"]


def test_real_reference_package_is_patched_not_reimplemented():
    """In the build container foveakit is importable: its CLI's `blockwise` is the module the
    adapter patches, and a patched call goes to the GPU path -- with no device here that is a
    RuntimeError, never the reference's CPU result."""
    import torch

    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        foveakit = pytest.importorskip("foveakit")
        cli = importlib.import_module("foveakit.cli")
    finally:
        sys.path.remove("/root/reference/pkg/src")
    orig = foveakit.blockwise.foveate
    with adapter.patched(foveakit):
        assert cli.blockwise.foveate is foveakit.blockwise.foveate is not orig
        if not torch.cuda.is_available():
            img = foveakit.RasterImage.from_array(np.zeros((40, 40, 3), np.uint8))
            with pytest.raises(RuntimeError):
                foveakit.blockwise.foveate(img, foveakit.FoveationParams())
    assert foveakit.blockwise.foveate is orig


@pytest.mark.gpu
def test_patched_calls_return_reference_types_and_gpu_results(standin):
    bw = importlib.import_module("standin_foveakit.blockwise")
    ret = importlib.import_module("standin_foveakit.retinal")
    im = importlib.import_module("standin_foveakit.imaging")
    fl = importlib.import_module("standin_foveakit.filters")
    rng = np.random.default_rng(6)
    arr = rng.integers(0, 256, (150, 200, 3), dtype=np.uint8)
    params = ret.FoveationParams(fragment_size=16, fixation=(30.0, 100.0), strength=1.5)
    ours_out, ours_grid, ours_bank, ours_stats = fk.foveate(
        fk.RasterImage.from_array(arr), fk.FoveationParams(fragment_size=16, fixation=(30.0, 100.0),
                                                           strength=1.5))
    with adapter.patched(standin):
        out, grid, bank, stats = bw.foveate(im.RasterImage.from_array(arr), params)
        assert isinstance(out, im.RasterImage) and isinstance(grid, bw.BlurGrid)
        assert isinstance(bank, fl.FilterBank) and isinstance(stats, bw.RenderStats)
        assert np.array_equal(out.data, ours_out.data)
        assert np.array_equal(grid.index, ours_grid.index) and grid.shift == ours_grid.shift
        assert stats.regions == ours_stats.regions and stats.max_filter == ours_stats.max_filter
        # the harness convention (bench.py:80-85): render over a prebuilt plan
        g2, b2 = bw.plan((200, 150), params)
        again = bw.render(im.RasterImage.from_array(arr), g2, b2, workers=4)
        assert isinstance(again, im.RasterImage) and np.array_equal(again.data, ours_out.data)
        with pytest.raises(ValueError):
            bw.foveate(im.RasterImage.from_array(arr), ret.FoveationParams(fixation=(500.0, 1.0)))
