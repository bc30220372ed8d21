"""Pin the CPU oracle (oracle/fovea_oracle.{py,c}) to the reference.

Golden vectors come from the reference itself (tests/golden/make_golden.py); the
known-answer values are the ones the reference's own tests assert
(pkg/tests/test_blockwise.py, test_retinal.py, test_filters.py -- cited per test).
"""

import hashlib
import math
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from cases import (BIG_RENDER_CASES, F32_CASES, PLAN_CASES, RENDER_CASES,  # noqa: E402
                   frame_f32, frame_u8)

from oracle import fovea_oracle as fo  # noqa: E402


# ------------------------------------------------------------------ known answers
def test_shift_kats():
    # test_blockwise.py:45-49 and SURVEY 8(a) a2
    assert fo.np_fragment_shift((16, 16), 32) == (0, 0)
    assert fo.np_fragment_shift((0, 0), 32) == (16, 16)
    assert fo.np_fragment_shift((960.0, 540.0), 32) == (16, 12)
    with pytest.raises(ValueError):
        fo.np_fragment_shift((0, 0), 2)  # test_blockwise.py:67-69


@pytest.mark.parametrize("F", [4, 8, 16, 32])
def test_shift_centres_a_fragment(F):
    # test_blockwise.py:51-65
    for fx in range(3 * F):
        dx, _ = fo.np_fragment_shift((fx, 0), F)
        centres = [dx + k * F + F / 2 for k in range(-2, 5)]
        assert min(abs(fx - c) for c in centres) <= 0.5
        dx1, _ = fo.np_fragment_shift((fx + 1, 0), F)
        assert (dx1 - dx) % F == 1


def test_sigma_kats():
    # test_retinal.py:91-95: sigma(0) = 1/pi, doubles at e2
    p = fo.OracleParams(fixation=(16.0, 16.0), fragment_size=32)
    # the fragment centred on the fixation has midpoint == fixation -> e = 0
    pl = fo.np_plan((64, 64), p)
    gy, gx = pl["foveal"]
    assert abs(pl["sigma"][gy, gx] - 1.0 / math.pi) <= 1e-12


def test_filter_length_and_taps_kats():
    # test_filters.py:41-47: sigma=1 -> 7 taps, centre 0.3990502797, next 0.2420362294
    assert int(fo.np_filter_length(1.0)) == 7
    assert fo._c().fo_filter_length(1.0) == 7
    assert int(fo.np_filter_length(0.0)) == 1 and int(fo.np_filter_length(1 / 6)) == 1
    assert int(fo.np_filter_length(0.2)) == 3  # test_filters.py:105-112
    k = np.arange(-3, 4, dtype=np.float64)
    w = np.exp(-(k * k) / 2.0)
    w /= w.sum()
    assert abs(w[3] - 0.3990502797) < 1e-9 and abs(w[2] - 0.2420362294) < 1e-9


def test_taps_match_reference(golden):
    g = golden["taps"]
    for key in g.files:
        L = int(key[1:])
        ref = g[key]
        for mine in (fo.np_gaussian_taps(L), fo.c_gaussian_taps(L)):
            assert mine.shape == ref.shape
            assert np.max(np.abs(mine - ref)) <= 1e-15
            assert abs(mine.sum() - 1.0) <= 1e-12
            assert np.array_equal(mine, mine[::-1]) or np.allclose(mine, mine[::-1], atol=1e-17)


# ------------------------------------------------------------------ plan goldens
@pytest.mark.parametrize("case", PLAN_CASES, ids=[c[0] for c in PLAN_CASES])
def test_plan_bit_exact_vs_reference(golden, case):
    name, size, kw, use_shift = case
    g = golden["plans"]
    p = fo.OracleParams(**kw)
    for pl in (fo.np_plan(size, p, use_shift), fo.c_plan(size, p, use_shift)):
        assert tuple(pl["shift"]) == tuple(int(v) for v in g[f"{name}/shift"])
        assert tuple(pl["foveal"]) == tuple(int(v) for v in g[f"{name}/foveal"])
        assert pl["sigma"].shape == g[f"{name}/sigma"].shape
        # bit-exact: compare the raw 64-bit patterns
        assert np.array_equal(pl["sigma"].view(np.uint64), g[f"{name}/sigma"].view(np.uint64))
        assert np.array_equal(pl["raw_length"], g[f"{name}/raw_length"])
    pl = fo.np_plan(size, p, use_shift)
    assert np.array_equal(pl["index"], g[f"{name}/index"])
    assert np.array_equal(pl["bank_lengths"], g[f"{name}/bank_lengths"])
    assert len(np.unique(pl["index"])) == int(g[f"{name}/regions"])


def test_1080p_calibration(golden):
    # test_blockwise.py:89-92 / test_acceptance.py:184-189: 26 +- 4 regions
    g = golden["plans"]
    assert abs(int(g["c1_1080p_f32_fix960_540/regions"]) - 26) <= 4
    pl = fo.np_plan((1920, 1080), fo.OracleParams(fixation=(960, 540)))
    assert pl["sigma"].shape == (35, 61) and len(np.unique(pl["index"])) == 26


# ---------------------------------------------------------------- render goldens
@pytest.mark.parametrize("case", RENDER_CASES, ids=[c[0] for c in RENDER_CASES])
def test_render_u8_vs_reference(golden, case):
    name, seed, shape, kw = case
    ref = golden["renders_u8"][f"{name}/out"]
    img = frame_u8(seed, shape)
    p = fo.OracleParams(**kw)
    out_c, pl = fo.c_foveate(img, p, threads=4)
    out_np = fo.np_render(img, p.fragment_size, pl["shift"], pl["length"])
    # the numpy restatement repeats the reference's numpy expressions: bit-exact
    assert np.array_equal(out_np, ref)
    # the C loops sum taps in a different order: +-1 LSB at exact .5 ties only
    diff = np.abs(out_c.astype(np.int16) - ref.astype(np.int16))
    assert diff.max() <= 1
    assert (diff != 0).mean() < 1e-4
    stats = golden["renders_u8"][f"{name}/stats"]
    assert int(pl["length"].max()) == int(stats[1])
    assert tuple(pl["shift"]) == (int(stats[2]), int(stats[3]))


@pytest.mark.parametrize("case", BIG_RENDER_CASES, ids=[c[0] for c in BIG_RENDER_CASES])
def test_render_1080p_vs_reference(golden, case):
    name, seed, shape, kw = case
    g = golden["renders_big"]
    img = frame_u8(seed, shape)
    out, pl = fo.c_foveate(img, fo.OracleParams(**kw), threads=8)
    sample = g[f"{name}/sample"]
    diff = np.abs(out[::7, ::11].astype(np.int16) - sample.astype(np.int16))
    assert diff.max() <= 1 and (diff != 0).mean() < 1e-4
    rows = out.astype(np.int64).sum(axis=(1, 2))
    assert np.abs(rows - g[f"{name}/rowsum"]).max() <= 4
    if hashlib.sha256(out.tobytes()).digest() != g[f"{name}/sha256"].tobytes():
        # allowed: a handful of .5 ties; already bounded by the row sums above
        assert np.abs(rows - g[f"{name}/rowsum"]).sum() <= 64


@pytest.mark.parametrize("case", F32_CASES, ids=[c[0] for c in F32_CASES])
def test_render_f32_vs_reference(golden, case):
    name, seed, shape, kw = case
    ref = golden["renders_f32"][f"{name}/out"]
    img = frame_f32(seed, shape)
    out, _ = fo.c_foveate(img, fo.OracleParams(**kw), quantize=False, threads=4)
    assert out.dtype == np.float64
    assert np.max(np.abs(out - ref)) <= 1e-13


@pytest.mark.parametrize("L", [7, 13, 31])
def test_uniform_grid_vs_reference(golden, L):
    # test_blockwise.py:135-148 configuration, against the reference's own output
    ref = golden["renders_uniform"][f"L{L}/out"]
    img = np.random.default_rng(L).integers(0, 256, (128, 128, 3)).astype(np.uint8)
    lengths = np.full((4, 4), L, np.int64)
    out = fo.c_render(img, 32, (0, 0), lengths)
    assert np.abs(out.astype(np.int16) - ref.astype(np.int16)).max() <= 1
    assert np.array_equal(fo.np_render(img, 32, (0, 0), lengths), ref)


# --------------------------------------------------------------------- properties
def test_identity_and_constant():
    # test_blockwise.py:121-133
    img = frame_u8(5, (48, 80, 3))
    ones = np.ones((3, 5), np.int64)
    assert np.array_equal(fo.c_render(img, 16, (0, 0), ones), img)
    const = np.full((64, 96, 3), 128, np.uint8)
    assert np.array_equal(fo.c_render(const, 16, (0, 0), np.full((4, 6), 25, np.int64)), const)


def test_algorithmic_macs_matches_survey_table():
    # 1080p/F32/centre -> 1.877e8 MAC/channel, corner -> 4.740e8
    pl = fo.np_plan((1920, 1080), fo.OracleParams())
    m = fo.algorithmic_macs((1920, 1080), 32, pl["shift"], pl["length"])
    assert abs(m / 1.877e8 - 1) < 2e-3
    pl = fo.np_plan((1920, 1080), fo.OracleParams(fixation=(0, 0)))
    m = fo.algorithmic_macs((1920, 1080), 32, pl["shift"], pl["length"])
    assert abs(m / 4.740e8 - 1) < 2e-3
