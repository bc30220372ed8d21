"""Block-wise foveated rendering on the GPU -- drop-in for foveakit.blockwise.

Same names, argument meaning and error behaviour as the reference
(blockwise.py:39-243); the work is done by libfovea.so: the plan kernel computes the
tiling shift, the sigma field, the tap counts and the foveal fragment on the device, the
blur kernel renders every fragment.  ``workers`` is accepted and ignored: the output is
bit-identical for any worker count by the reference's own contract (blockwise.py:13-15).

New here: ``foveate_batch`` for [N, H, W, C] frame batches with one fixation per frame,
on host memory (pipelined copies) or on device tensors, optionally sharded over GPUs.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from .engine import get_engine, shard_range
from .filters import FilterBank, _bank_and_index, build_bank
from .imaging import RasterImage
from .retinal import FoveationParams, SigmaField, build_sigma_field
from .tiling import cell_of, fragment_spans


def compute_fragment_shift(fixation, fragment_size: int) -> tuple[int, int]:
    """Tiling origin offset that centres one fragment on the fixation
    (blockwise.py:39-51).  Host integer helper; the plan kernel computes the same value
    per frame on the device."""
    if fragment_size < 4:
        raise ValueError(f"fragment_size must be >= 4, got {fragment_size}")
    fx, fy = fixation
    half = fragment_size // 2
    return ((int(np.floor(fx)) - half) % fragment_size,
            (int(np.floor(fy)) - half) % fragment_size)


@dataclass(frozen=True)
class BlurGrid:
    """Which filter blurs which fragment (blockwise.py:54-85)."""

    index: np.ndarray  # int64 (grid_h, grid_w) indices into a FilterBank
    shift: tuple[int, int]
    fragment_size: int
    foveal_cell: tuple[int, int]  # (gy, gx)

    @property
    def grid_size(self) -> tuple[int, int]:
        return (self.index.shape[1], self.index.shape[0])

    def region_count(self) -> int:
        return len(np.unique(self.index))

    def to_text(self, bank: FilterBank) -> str:
        head = [
            f"fragment {self.fragment_size}",
            f"shift {self.shift[0]} {self.shift[1]}",
            f"grid {self.index.shape[1]} {self.index.shape[0]}",
            f"foveal_cell {self.foveal_cell[1]} {self.foveal_cell[0]}",
            f"regions {self.region_count()}",
            "",
            bank.to_table(),
            "",
            "index_matrix",
        ]
        return "\n".join(head + [" ".join(str(v) for v in row) for row in self.index])


@dataclass(frozen=True)
class Tile:
    """A fragment plus its filter padding (blockwise.py:88-104)."""

    x0: int
    y0: int
    fragment_w: int
    fragment_h: int
    radius: int

    @property
    def tile_w(self) -> int:
        return self.fragment_w + 2 * self.radius

    @property
    def tile_h(self) -> int:
        return self.fragment_h + 2 * self.radius


@dataclass(frozen=True)
class RenderStats:
    render_ms: float
    regions: int
    max_filter: int
    fragment_size: int
    shift: tuple[int, int]


def build_blur_grid(field: SigmaField, bank: FilterBank, index: np.ndarray, fixation,
                    image_size, fragment_size: int, shift) -> BlurGrid:
    """Attach filter indices to the shifted tiling; the fixation fragment is forced to
    the identity filter (blockwise.py:107-133)."""
    w, h = image_size
    sx = fragment_spans(w, fragment_size, shift[0])
    sy = fragment_spans(h, fragment_size, shift[1])
    if index.shape != (len(sy), len(sx)):
        raise ValueError(
            f"index grid {index.shape} does not cover the {len(sy)}x{len(sx)} tiling")
    foveal = (cell_of(sy, fixation[1]), cell_of(sx, fixation[0]))
    grid = index.copy()
    grid[foveal] = 0
    return BlurGrid(index=grid, shift=tuple(shift), fragment_size=fragment_size,
                    foveal_cell=foveal)


def plan(img_size, params: FoveationParams, density=None, sigma_max=None, use_shift=True,
         *, device: int = 0):
    """Everything up to the per-frame render (blockwise.py:198-220): one device plan
    launch, then the bank/index bookkeeping of build_bank on the read-back tap counts."""
    fixation = params.fixation_for(img_size)
    if density is not None:
        if sigma_max is None:
            raise ValueError("sigma_max is required with a density map")
        from .density import ingest_density_map

        shift = compute_fragment_shift(fixation, params.fragment_size) if use_shift else (0, 0)
        field = ingest_density_map(density, sigma_max, img_size, params.fragment_size, shift,
                                   device=device)
        bank, index = build_bank(field, device=device)
        return build_blur_grid(field, bank, index, fixation, img_size, params.fragment_size,
                               shift), bank
    w, h = img_size
    if w < 1 or h < 1:
        raise ValueError(f"extent must be positive, got {w}x{h}")
    eng = get_engine(device)
    with eng._lock:
        dp = eng.plan_for(img_size, params.fragment_size, 1)
        dp.model(params, [fixation], use_shift=use_shift)
        got = dp.read(0)
    if not np.all(np.isfinite(got["sigma"])) or np.any(got["sigma"] < 0):
        raise ValueError("sigma values must be finite and >= 0")
    bank, index = _bank_and_index(got["raw_length"], device=device)
    index[got["foveal"]] = 0
    grid = BlurGrid(index=index, shift=got["shift"], fragment_size=params.fragment_size,
                    foveal_cell=got["foveal"])
    return grid, bank


def _grid_tables(grid: BlurGrid, bank: FilterBank):
    """Per-fragment tap counts / offsets and the flattened bank for fk_plan_set_grid."""
    lengths = np.asarray([len(f) for f in bank.filters], dtype=np.int64)
    starts = np.concatenate(([0], np.cumsum(lengths)[:-1]))
    coeffs = np.concatenate([np.asarray(f, dtype=np.float64).ravel() for f in bank.filters])
    return lengths[grid.index], starts[grid.index], coeffs


def render(img: RasterImage, grid: BlurGrid, bank: FilterBank, workers: int = 1,
           *, device: int = 0) -> RasterImage:
    """Blur every fragment with its assigned filter (blockwise.py:156-186)."""
    if img.channels not in (1, 3):
        raise ValueError(f"render supports 1 or 3 channels, got {img.channels}")
    if int(grid.index.max()) >= len(bank) or int(grid.index.min()) < 0:
        raise ValueError(
            f"grid references filter {int(grid.index.max())} but bank has {len(bank)}")
    sx = fragment_spans(img.width, grid.fragment_size, grid.shift[0])
    sy = fragment_spans(img.height, grid.fragment_size, grid.shift[1])
    if grid.index.shape != (len(sy), len(sx)):
        raise ValueError(f"grid {grid.index.shape} does not match image {img.size}")
    lengths, offsets, coeffs = _grid_tables(grid, bank)
    eng = get_engine(device)
    with eng._lock, torch.cuda.device(eng.device):
        dp = eng.plan_for(img.size, grid.fragment_size, 1)
        dp.set_grid(grid.shift, lengths, offsets, coeffs)
        src = torch.from_numpy(img.data).to(f"cuda:{eng.device}")[None]
        out = eng.render(src, dp)
        data = out[0].cpu().numpy()
    return RasterImage.from_array(data)


def foveate(img: RasterImage, params: FoveationParams, density=None, sigma_max=None,
            workers: int = 1, use_shift: bool = True, *, device: int = 0):
    """Full pipeline: shift -> sigma field -> bank -> grid -> render
    (blockwise.py:223-243).  render_ms times the render call, copies included, as the
    reference times its render."""
    grid, bank = plan(img.size, params, density, sigma_max, use_shift, device=device)
    t0 = time.perf_counter()
    result = render(img, grid, bank, workers=workers, device=device)
    ms = (time.perf_counter() - t0) * 1000.0
    stats = RenderStats(render_ms=ms, regions=grid.region_count(),
                        max_filter=int(bank.lengths[grid.index.max()]),
                        fragment_size=grid.fragment_size, shift=grid.shift)
    return result, grid, bank, stats


def _default_fixations(n, size):
    w, h = size
    return np.tile(np.asarray([[w / 2.0, h / 2.0]], dtype=np.float64), (n, 1))


def _check_fixations(fix, n, size):
    w, h = size
    fix = np.ascontiguousarray(np.asarray(fix, dtype=np.float64).reshape(-1, 2))
    if fix.shape[0] != n:
        raise ValueError(f"{n} frames but {fix.shape[0]} fixations")
    ok = (fix[:, 0] >= 0) & (fix[:, 0] < w) & (fix[:, 1] >= 0) & (fix[:, 1] < h)
    if not np.all(ok):
        bad = fix[np.argmin(ok)]
        raise ValueError(f"fixation {(float(bad[0]), float(bad[1]))} outside {w}x{h} image")
    return fix


def _foveate_shards(shards, fixations, params, out, use_shift, validate):
    """foveate_batch for a batch that lives on several GPUs as one CUDA tensor per device."""
    shards = list(shards)
    for t in shards:
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.ndim == 4):
            raise ValueError("a sharded batch is a list of CUDA tensors [n_i, H, W, C]")
    counts = [int(t.shape[0]) for t in shards]
    if fixations is None:
        fixations = [None] * len(shards)
    elif not isinstance(fixations, (list, tuple)):
        fix = np.asarray(fixations, dtype=np.float64).reshape(-1, 2)
        if fix.shape[0] != sum(counts):
            raise ValueError(f"{sum(counts)} frames but {fix.shape[0]} fixations")
        cuts = np.cumsum([0] + counts)
        fixations = [fix[cuts[i]:cuts[i + 1]] for i in range(len(shards))]
    if len(fixations) != len(shards):
        raise ValueError(f"{len(shards)} shards but {len(fixations)} fixation arrays")
    outs = list(out) if out is not None else [None] * len(shards)
    if len(outs) != len(shards):
        raise ValueError(f"{len(shards)} shards but {len(outs)} output tensors")
    results, errors = [None] * len(shards), []

    def work(i):
        t = shards[i]
        try:
            if t.shape[0] == 0:
                results[i] = outs[i] if outs[i] is not None else torch.empty_like(t)
                return
            with torch.cuda.device(t.device):
                stream = torch.cuda.Stream(device=t.device)
                stream.wait_stream(torch.cuda.current_stream(t.device))
                with torch.cuda.stream(stream):
                    results[i] = foveate_batch(t, fixations[i], params, out=outs[i],
                                               use_shift=use_shift, validate=validate)
                stream.synchronize()
        except Exception as exc:  # surfaced after join
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(shards))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    return results


def foveate_batch(frames, fixations=None, params: FoveationParams | None = None, *, out=None,
                  devices=None, use_shift: bool = True, chunk_frames: int = 0,
                  validate: bool = True):
    """Foveate a batch of frames, one fixation per frame.

    frames     [N, H, W, C] uint8 or float32, C in {1, 3}: a numpy array (host memory,
               rendered through the pipelined host path and returned as numpy) or a CUDA
               torch tensor (rendered in place on its GPU and returned as a tensor) -- or a
               list of CUDA tensors, the shards of one batch resident on several GPUs
               (contiguous split, no collective): every shard is planned and
               rendered on its own GPU by its own host thread and CUDA stream, nothing
               crosses the host, and the list of output tensors is returned.  `fixations` is
               then a list with one entry per shard, or one [N_total, 2] array cut in shard
               order; `out` a list of tensors or None.
    fixations  [N, 2] (x, y) pixel coordinates; default: the image centre
               (``params.fixation`` if set).  For device frames this may be a CUDA
               float64 tensor.
    devices    GPUs to shard host batches over (contiguous split of N, no collective:
               frames are independent).  Default: the current device only.
    validate   device fixations only: read the plan kernel's out-of-image count back and
               raise ValueError like the reference (synchronises); False keeps the call
               asynchronous and copies such frames through.
    """
    params = params if params is not None else FoveationParams()
    if isinstance(frames, (list, tuple)):
        return _foveate_shards(frames, fixations, params, out, use_shift, validate)
    if isinstance(frames, torch.Tensor) and frames.is_cuda:
        n, h, w, _ = frames.shape
        if fixations is None:
            fixations = np.tile(np.asarray([params.fixation_for((w, h))]), (n, 1))
        if not (isinstance(fixations, torch.Tensor) and fixations.is_cuda):
            fixations = _check_fixations(fixations, n, (w, h))
        eng = get_engine(frames.device.index)
        with torch.cuda.device(eng.device):
            res, _ = eng.foveate_device(frames, fixations, params, use_shift=use_shift, out=out,
                                        validate=validate)
        return res

    if isinstance(frames, torch.Tensor):
        frames = frames.numpy()
    frames = np.asarray(frames)
    if frames.ndim != 4:
        raise ValueError(f"expected [N, H, W, C] frames, got shape {frames.shape}")
    n, h, w, c = frames.shape
    if c not in (1, 3):
        raise ValueError(f"render supports 1 or 3 channels, got {c}")
    if fixations is None:
        fixations = np.tile(np.asarray([params.fixation_for((w, h))]), (n, 1))
    fix = _check_fixations(fixations, n, (w, h))
    frames = np.ascontiguousarray(frames)
    if out is None:
        out = np.empty_like(frames)
    if devices is None:
        devices = [torch.cuda.current_device()]
    devices = list(devices)
    if len(devices) == 1:
        get_engine(devices[0]).foveate_host(frames, fix, params, out=out, use_shift=use_shift,
                                            chunk_frames=chunk_frames)
        return out

    errors = []

    def work(rank, dev):
        a, b = shard_range(n, rank, len(devices))
        if a == b:
            return
        try:
            get_engine(dev).foveate_host(frames[a:b], fix[a:b], params, out=out[a:b],
                                         use_shift=use_shift, chunk_frames=chunk_frames)
        except Exception as exc:  # surfaced after join
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(r, d)) for r, d in enumerate(devices)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return out
