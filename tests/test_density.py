"""Density-map sigma fields (retinal.py:180-231, blockwise.py:208-213):
oracle pinned to reference goldens on CPU, device path bit-exact on GPU."""

import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from cases import DENSITY_CASES, DENSITY_RENDER_CASES, density_map, frame_u8  # noqa: E402

import paper_2012_08655_b200 as fk  # noqa: E402
from oracle import fovea_oracle as fo  # noqa: E402


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("case", DENSITY_CASES, ids=[c[0] for c in DENSITY_CASES])
def test_oracle_density_sigma_bit_exact_vs_reference(golden, case):
    name, seed, mshape, size, F, shift, smax = case
    ref = golden["density"][f"{name}/sigma"]
    got = fo.np_density_sigma(density_map(seed, mshape), smax, size, F, shift)
    assert got.shape == ref.shape and np.array_equal(bits(got), bits(ref))


def test_oracle_density_kats():
    # test_retinal.py:155-180
    white = np.full((8, 8), 255, np.uint8)
    black = np.zeros((8, 8), np.uint8)
    assert np.all(fo.np_density_sigma(white, 6.0, (64, 64), 16, (0, 0)) == 0.0)
    assert np.allclose(fo.np_density_sigma(black, 6.0, (64, 64), 16, (0, 0)), 6.0)
    ramp = np.tile(np.linspace(0, 255, 32, dtype=np.uint8), (32, 1))
    assert np.all(np.diff(fo.np_density_sigma(ramp, 4.0, (64, 64), 16, (0, 0)), axis=1) < 0)


def test_density_argument_errors_without_gpu():
    rgb = fk.RasterImage.from_array(np.zeros((4, 4, 3), np.uint8))
    gray = fk.RasterImage.from_array(np.zeros((4, 4), np.uint8))
    with pytest.raises(ValueError, match="1-channel"):          # test_retinal.py:169-172
        fk.ingest_density_map(rgb, 2.0, (64, 64), 16, (0, 0))
    with pytest.raises(ValueError, match="sigma_max"):          # test_retinal.py:174-176
        fk.ingest_density_map(gray, -1.0, (64, 64), 16, (0, 0))


@pytest.mark.gpu
@pytest.mark.parametrize("case", DENSITY_CASES, ids=[c[0] for c in DENSITY_CASES])
def test_device_density_sigma_bit_exact(golden, case):
    name, seed, mshape, size, F, shift, smax = case
    ref = golden["density"][f"{name}/sigma"]
    dm = fk.RasterImage.from_array(density_map(seed, mshape))
    field = fk.ingest_density_map(dm, smax, size, F, shift)
    assert field.sigma.shape == ref.shape
    assert np.array_equal(bits(field.sigma), bits(ref)), "density sigma not bit-exact"


@pytest.mark.gpu
@pytest.mark.parametrize("case", DENSITY_RENDER_CASES, ids=[c[0] for c in DENSITY_RENDER_CASES])
def test_foveate_with_density_map_matches_reference(golden, case):
    name, seed, shape, mseed, mshape, kw, smax = case
    g = golden["density"]
    img = frame_u8(seed, shape)
    dm = fk.RasterImage.from_array(density_map(mseed, mshape))
    out, grid, bank, stats = fk.foveate(fk.RasterImage.from_array(img), fk.FoveationParams(**kw),
                                        density=dm, sigma_max=smax)
    assert np.array_equal(grid.index, g[f"{name}/index"])
    assert np.array_equal(bank.lengths, g[f"{name}/bank_lengths"])
    diff = np.abs(out.data.astype(np.int16) - g[f"{name}/out"].astype(np.int16))
    assert diff.max() <= 1 and (diff != 0).mean() < 2e-3


@pytest.mark.gpu
def test_density_kats_on_device():
    # test_retinal.py:155-167, test_blockwise.py:239-244
    white = fk.RasterImage.from_array(np.full((8, 8), 255, np.uint8))
    black = fk.RasterImage.from_array(np.zeros((8, 8), np.uint8))
    assert np.all(fk.ingest_density_map(white, 6.0, (64, 64), 16, (0, 0)).sigma == 0.0)
    assert np.allclose(fk.ingest_density_map(black, 6.0, (64, 64), 16, (0, 0)).sigma, 6.0)
    for v in (127, 128):
        m = fk.RasterImage.from_array(np.full((8, 8), v, np.uint8))
        assert abs(fk.ingest_density_map(m, 6.0, (64, 64), 16, (0, 0)).sigma[1, 1] - 3.0) <= 6 / 255 + 1e-12
    img = fk.RasterImage.from_array(frame_u8(99, (160, 160, 3)))
    out, *_ = fk.foveate(img, fk.FoveationParams(fragment_size=16), density=white, sigma_max=5.0)
    assert out == img
