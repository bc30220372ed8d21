"""SSIM maps (quality.py:31-114): the numpy oracle is pinned to maps made
by the reference itself (tests/golden/make_golden_ssim.py) on CPU; the device path
(fk_ssim_u8 / fk_ssim_stats through paper_2012_08655_b200.quality) is compared with the oracle
and the goldens on the GPU.  fp64 on both sides: tolerance 1e-9 absolute on values in [-1, 1]
(the summation order inside numpy's matmul is not specified; measured ~1e-15)."""

import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from cases import SSIM_CASES, SSIM_MEAN_CASE, ssim_pair  # noqa: E402

import paper_2012_08655_b200 as fk  # noqa: E402
from paper_2012_08655_b200 import quality  # noqa: E402
from oracle import fovea_oracle as fo  # noqa: E402

TOL = 1e-9


def _full(shape):
    return shape[0] * shape[1] <= 64 * 64


def _check(golden, name, shape, values, mean, mn, argmin):
    ref_stats = golden["ssim"][f"{name}/stats"]
    ref_vals = golden["ssim"][f"{name}/values"]
    got = values if _full(shape) else values[::37, ::41]
    assert got.shape == ref_vals.shape
    assert np.abs(got - ref_vals).max() <= TOL
    assert abs(mean - ref_stats[0]) <= TOL and abs(mn - ref_stats[1]) <= TOL
    # the worst window: same place, or a tie within the tolerance
    oy, ox = int(ref_stats[2]) - 5, int(ref_stats[3]) - 5
    assert tuple(argmin) == (oy + 5, ox + 5) or abs(values[argmin[0] - 5, argmin[1] - 5] - values[oy, ox]) <= TOL


@pytest.mark.parametrize("case", SSIM_CASES, ids=[c[0] for c in SSIM_CASES])
def test_oracle_ssim_vs_reference(golden, case):
    name, seed, shape, amp, smooth = case
    ref, test = ssim_pair(seed, shape, amp, smooth)
    values, mean, mn, argmin = fo.np_ssim_map(ref, test)
    _check(golden, name, shape, values, mean, mn, argmin)


def test_oracle_ssim_kats():
    # test_quality.py of the reference: identical images give 1 everywhere; the window sums to 1
    ref, _ = ssim_pair(5, (32, 40, 3), 0, True)
    values, mean, mn, _ = fo.np_ssim_map(ref, ref)
    assert values.shape == (22, 30) and np.allclose(values, 1.0, atol=1e-12)
    assert abs(fo.np_ssim_window().sum() - 1.0) < 1e-15
    assert np.array_equal(quality._window(), fo.np_ssim_window())


def test_ssim_argument_errors_without_gpu():
    a = fk.RasterImage.from_array(np.zeros((16, 16, 3), np.uint8))
    b = fk.RasterImage.from_array(np.zeros((16, 17, 3), np.uint8))
    g = fk.RasterImage.from_array(np.zeros((16, 16, 1), np.uint8))
    s = fk.RasterImage.from_array(np.zeros((10, 16, 3), np.uint8))
    with pytest.raises(ValueError, match="dimension mismatch"):
        quality.ssim_map(a, b)
    with pytest.raises(ValueError, match="dimension mismatch"):
        quality.ssim_map(a, g)
    with pytest.raises(ValueError, match="at least 11px"):
        quality.ssim_map(s, s)
    with pytest.raises(ValueError, match="at least one pair"):
        quality.mean_ssim_map([])
    m = quality.SSIMMap(values=np.array([[0.5, 1.2], [-0.1, 1.0]]), mean=0.65, min=-0.1, argmin=(6, 5))
    assert m.stats_text() == "mean 0.650000\nmin -0.100000\nargmin 5 6\n"
    assert m.to_image().data[:, :, 0].tolist() == [[128, 255], [0, 255]]


@pytest.mark.gpu
@pytest.mark.parametrize("case", SSIM_CASES, ids=[c[0] for c in SSIM_CASES])
def test_device_ssim_vs_oracle_and_reference(golden, case):
    name, seed, shape, amp, smooth = case
    ref, test = ssim_pair(seed, shape, amp, smooth)
    m = quality.ssim_map(fk.RasterImage.from_array(ref), fk.RasterImage.from_array(test))
    _check(golden, name, shape, m.values, m.mean, m.min, m.argmin)
    values, mean, mn, argmin = fo.np_ssim_map(ref, test)
    assert m.values.shape == values.shape and np.abs(m.values - values).max() <= TOL
    assert abs(m.mean - mean) <= TOL and abs(m.min - mn) <= TOL
    assert m.values[m.argmin[0] - 5, m.argmin[1] - 5] == m.values.min()


@pytest.mark.gpu
def test_device_mean_ssim_map_vs_reference(golden):
    name, seeds, shape, amp, smooth = SSIM_MEAN_CASE
    pairs = [tuple(fk.RasterImage.from_array(a) for a in ssim_pair(s, shape, amp, smooth)) for s in seeds]
    m = quality.mean_ssim_map(pairs)
    _check(golden, name, shape, m.values, m.mean, m.min, m.argmin)
    other = fk.RasterImage.from_array(np.zeros((40, 40, 3), np.uint8))
    with pytest.raises(ValueError, match="same dimensions"):
        quality.mean_ssim_map([pairs[0], (other, other)])


@pytest.mark.gpu
def test_device_ssim_of_a_foveated_frame_is_one_in_the_fovea():
    # acceptance criterion of the reference (test_acceptance.py:135-148): the foveal fragment is
    # copied through, so windows inside it score exactly 1
    rng = np.random.default_rng(3)
    img = fk.RasterImage.from_array(rng.integers(0, 256, (256, 320, 3), dtype=np.uint8))
    p = fk.FoveationParams(fragment_size=32, fixation=(160, 128))
    out, grid, _, _ = fk.foveate(img, p)
    m = quality.ssim_map(img, out)
    assert m.values.shape == (246, 310) and m.min < 0.9
    assert m.values[128 - 5, 160 - 5] == 1.0  # window centred on the fixation, inside the fovea
