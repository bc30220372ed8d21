"""Generate golden vectors for the blockwise foveation path FROM THE REFERENCE ITSELF.

Run in the build container only (the reference does not travel to the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports ``foveakit`` from ``/root/reference/pkg/src`` (read-only), runs the
reference's own ``plan`` / ``render`` / ``build_sigma_field`` / ``gaussian_filter_1d``
on seeded inputs and writes small ``.npz`` files next to this script.  Inputs are
regenerated from seeds by the tests; only reference OUTPUTS are stored.
"""

from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import foveakit  # noqa: E402
from foveakit import blockwise, filters, retinal, tiling  # noqa: E402
from foveakit.imaging import RasterImage  # noqa: E402

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from cases import (BIG_RENDER_CASES, DENSITY_CASES, DENSITY_RENDER_CASES, F32_CASES,  # noqa: E402
                   PLAN_CASES, RENDER_CASES, density_map, frame_f32, frame_u8)


def ref_plan(size, kw, use_shift):
    p = retinal.FoveationParams(**kw)
    grid, bank = blockwise.plan(size, p, use_shift=use_shift)
    fix = p.fixation_for(size)
    shift = blockwise.compute_fragment_shift(fix, p.fragment_size) if use_shift else (0, 0)
    field = retinal.build_sigma_field(size, p, shift)
    raw = np.asarray(filters.filter_length(field.sigma), dtype=np.int64)
    return p, grid, bank, field, raw, shift


def ref_render_f64(img_f32, grid, bank):
    """The reference's own per-cell arithmetic on a float frame, unquantised."""
    h, w = img_f32.shape[:2]
    sx = tiling.fragment_spans(w, grid.fragment_size, grid.shift[0])
    sy = tiling.fragment_spans(h, grid.fragment_size, grid.shift[1])
    out = np.empty(img_f32.shape, dtype=np.float64)
    saved = blockwise.quantize_u8
    blockwise.quantize_u8 = lambda v: v
    try:
        for gy in range(len(sy)):
            for gx in range(len(sx)):
                blockwise._render_cell(img_f32, out, sx[gx], sy[gy],
                                       bank.filters[grid.index[gy, gx]])
    finally:
        blockwise.quantize_u8 = saved
    return out


def main():
    plans = {}
    for name, size, kw, use_shift in PLAN_CASES:
        p, grid, bank, field, raw, shift = ref_plan(size, kw, use_shift)
        plans[f"{name}/sigma"] = field.sigma
        plans[f"{name}/raw_length"] = raw
        plans[f"{name}/index"] = grid.index
        plans[f"{name}/bank_lengths"] = bank.lengths
        plans[f"{name}/shift"] = np.asarray(grid.shift, np.int64)
        plans[f"{name}/foveal"] = np.asarray(grid.foveal_cell, np.int64)
        plans[f"{name}/regions"] = np.asarray(grid.region_count(), np.int64)
    np.savez_compressed(HERE / "plans.npz", **plans)

    taps = {}
    for L in list(range(1, 64, 2)) + [79, 99, 103, 133, 155, 201, 255]:
        taps[f"L{L}"] = filters.gaussian_filter_1d(L / 6.0)
    np.savez_compressed(HERE / "taps.npz", **taps)

    renders = {}
    for name, seed, shape, kw in RENDER_CASES:
        img = frame_u8(seed, shape)
        out, grid, bank, stats = blockwise.foveate(
            RasterImage.from_array(img), retinal.FoveationParams(**kw))
        renders[f"{name}/out"] = out.data
        renders[f"{name}/stats"] = np.asarray(
            [stats.regions, stats.max_filter, stats.shift[0], stats.shift[1]], np.int64)
    np.savez_compressed(HERE / "renders_u8.npz", **renders)

    big = {}
    for name, seed, shape, kw in BIG_RENDER_CASES:
        img = frame_u8(seed, shape)
        out, grid, bank, stats = blockwise.foveate(
            RasterImage.from_array(img), retinal.FoveationParams(**kw))
        big[f"{name}/sha256"] = np.frombuffer(
            hashlib.sha256(out.data.tobytes()).digest(), dtype=np.uint8)
        big[f"{name}/sample"] = out.data[::7, ::11].copy()
        big[f"{name}/rowsum"] = out.data.astype(np.int64).sum(axis=(1, 2))
        big[f"{name}/stats"] = np.asarray(
            [stats.regions, stats.max_filter, stats.shift[0], stats.shift[1]], np.int64)
    np.savez_compressed(HERE / "renders_big.npz", **big)

    f32 = {}
    for name, seed, shape, kw in F32_CASES:
        img = frame_f32(seed, shape)
        p = retinal.FoveationParams(**kw)
        grid, bank = blockwise.plan((shape[1], shape[0]), p)
        f32[f"{name}/out"] = ref_render_f64(img, grid, bank)
    np.savez_compressed(HERE / "renders_f32.npz", **f32)

    # uniform-grid case of test_blockwise.py:135-148 (bank built from sigmas)
    uni = {}
    for length in (7, 13, 31):
        rng = np.random.default_rng(length)
        img = rng.integers(0, 256, (128, 128, 3)).astype(np.uint8)
        sig = length / 6.0
        field = retinal.SigmaField(grid_width=1, grid_height=1, sigma=np.asarray([[sig]]))
        bank = filters.build_bank(field)[0]
        gx = len(tiling.fragment_spans(128, 32, 0))
        grid = blockwise.BlurGrid(index=np.full((gx, gx), 1, np.int64), shift=(0, 0),
                                  fragment_size=32, foveal_cell=(0, 0))
        uni[f"L{length}/out"] = blockwise.render(RasterImage.from_array(img), grid, bank).data
    np.savez_compressed(HERE / "renders_uniform.npz", **uni)

    den = {}
    for name, seed, mshape, size, F, shift, smax in DENSITY_CASES:
        dm = RasterImage.from_array(density_map(seed, mshape))
        den[f"{name}/sigma"] = retinal.ingest_density_map(dm, smax, size, F, shift).sigma
    for name, seed, shape, mseed, mshape, kw, smax in DENSITY_RENDER_CASES:
        img = frame_u8(seed, shape)
        dm = RasterImage.from_array(density_map(mseed, mshape))
        out, grid, bank, stats = blockwise.foveate(
            RasterImage.from_array(img), retinal.FoveationParams(**kw), density=dm, sigma_max=smax)
        den[f"{name}/out"] = out.data
        den[f"{name}/index"] = grid.index
        den[f"{name}/bank_lengths"] = bank.lengths
    np.savez_compressed(HERE / "density.npz", **den)

    print("foveakit", foveakit.__name__, "numpy", np.__version__)
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, f.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
