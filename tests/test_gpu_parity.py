"""Parity of the CUDA path (through the C ABI) with the reference: golden vectors made by
the reference itself, the CPU oracle on the same seeded inputs, and size-independent
properties at the BASELINE.json sizes.  Bars (BASELINE.json north_star): sigma / tap
counts / index grid / shift / foveal cell bit-exact; uint8 output max-abs <= 1 with
identity fragments byte-exact; float32 output within 1e-4 relative."""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
from cases import (BIG_RENDER_CASES, F32_CASES, PLAN_CASES, RENDER_CASES,  # noqa: E402
                   frame_f32, frame_u8)

import paper_2012_08655_b200 as fk  # noqa: E402
from oracle import fovea_oracle as fo  # noqa: E402

pytestmark = pytest.mark.gpu

U8_TOL = 1          # north_star: max-abs error <= 1/255 on uint8 output
F32_RTOL = 1e-4     # north_star: <= 1e-4 relative on fp32 output


def maxdiff(a, b):
    return int(np.abs(a.astype(np.int16) - b.astype(np.int16)).max())


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


# ----------------------------------------------------------------------------- plan
@pytest.mark.parametrize("case", PLAN_CASES, ids=[c[0] for c in PLAN_CASES])
def test_plan_matches_reference_golden(golden, case):
    name, size, kw, use_shift = case
    g = golden["plans"]
    p = fk.FoveationParams(**kw)
    grid, bank = fk.plan(size, p, use_shift=use_shift)
    assert tuple(grid.shift) == tuple(int(v) for v in g[f"{name}/shift"])
    assert tuple(grid.foveal_cell) == tuple(int(v) for v in g[f"{name}/foveal"])
    assert np.array_equal(grid.index, g[f"{name}/index"])
    assert np.array_equal(bank.lengths, g[f"{name}/bank_lengths"])
    assert grid.region_count() == int(g[f"{name}/regions"])
    field = fk.build_sigma_field(size, p, grid.shift)
    assert field.sigma.shape == g[f"{name}/sigma"].shape
    assert np.array_equal(bits(field.sigma), bits(g[f"{name}/sigma"])), "sigma not bit-exact"
    assert np.array_equal(fk.filter_length(field.sigma), g[f"{name}/raw_length"])


def test_plan_batch_random_vs_oracle():
    """Random geometries and fractional fixations, planned as batches on the device."""
    rng = np.random.default_rng(2024)
    eng = fk.get_engine(0)
    for trial in range(40):
        F = int(rng.choice([4, 8, 12, 16, 32, 64, 100]))
        w, h = int(rng.integers(1, 700)), int(rng.integers(1, 500))
        kw = dict(fragment_size=F, e2=float(rng.uniform(0.8, 4)), alpha=float(rng.uniform(0.05, 0.3)),
                  ct0=float(rng.uniform(0.005, 0.1)), e_corner=float(rng.uniform(0, 90)),
                  strength=float(rng.uniform(0, 2.5)))
        if trial % 3 == 0:
            kw["f_max"] = float(rng.uniform(10, 60))
        n = 16
        fix = np.stack([rng.uniform(0, w, n), rng.uniform(0, h, n)], axis=1)
        fix[::4] = np.floor(fix[::4])          # integer-pixel fixations too
        fix[1] = (0.0, 0.0)
        fix[2] = (np.nextafter(float(w), 0.0), np.nextafter(float(h), 0.0))
        p = fk.FoveationParams(**kw)
        plan = eng.plan_for((w, h), F, n)
        plan.model(p, fix, use_shift=(trial % 5 != 0))
        for i in range(n):
            got = plan.read(i)
            ref = fo.c_plan((w, h), fo.OracleParams(fixation=tuple(fix[i]), **kw),
                            use_shift=(trial % 5 != 0))
            assert got["shift"] == ref["shift"]
            assert got["foveal"] == ref["foveal"]
            assert got["sigma"].shape == ref["sigma"].shape
            assert np.array_equal(bits(got["sigma"]), bits(ref["sigma"]))
            assert np.array_equal(got["raw_length"], ref["raw_length"])
            assert np.array_equal(got["length"], ref["length"])
            assert got["max_length"] == int(ref["length"].max())


def test_plan_order_is_a_cost_descending_permutation():
    eng = fk.get_engine(0)
    plan = eng.plan_for((1920, 1080), 32, 4)
    fix = np.asarray([[960, 540], [0, 0], [1919, 1079], [300.5, 700.25]], dtype=np.float64)
    plan.model(fk.FoveationParams(), fix)
    lengths, meta = plan.read_lengths()
    assert meta.shape == (4, 8) and np.all(meta[:, 7] == 0)
    for i in range(4):
        gw, gh = meta[i, 2], meta[i, 3]
        assert lengths[i, : gw * gh].max() == meta[i, 6]
        assert lengths[i, meta[i, 4] * gw + meta[i, 5]] == 1   # foveal cell forced


def test_lut_taps_match_reference(golden):
    g = golden["taps"]
    eng = fk.get_engine(0)
    for key in g.files:
        L = int(key[1:])
        taps = eng.lut_taps(L)
        assert taps.shape == g[key].shape
        assert np.max(np.abs(taps - g[key])) <= 1e-12
        assert abs(taps.sum() - 1.0) <= 1e-9
        assert np.allclose(taps, taps[::-1], rtol=0, atol=1e-15)


def test_bank_from_sigmas_kat():
    # test_filters.py:105-128: lengths [1,3,7,31], index [1,2,2,3], cumulative [1,4,11,42]
    field = fk.SigmaField(grid_width=4, grid_height=1,
                          sigma=np.asarray([[0.2, 1.0, 1.1, 5.0]]))
    bank, index = fk.build_bank(field)
    assert list(bank.lengths) == [1, 3, 7, 31]
    assert list(index[0]) == [1, 2, 2, 3]
    assert list(bank.cumulative_sizes) == [1, 4, 11, 42]
    assert fk.total_coefficients(bank) == 42


# --------------------------------------------------------------------------- render
@pytest.mark.parametrize("case", RENDER_CASES, ids=[c[0] for c in RENDER_CASES])
def test_render_u8_matches_reference_golden(golden, case):
    name, seed, shape, kw = case
    ref = golden["renders_u8"][f"{name}/out"]
    stats_ref = golden["renders_u8"][f"{name}/stats"]
    img = frame_u8(seed, shape)
    out, grid, bank, stats = fk.foveate(fk.RasterImage.from_array(img), fk.FoveationParams(**kw))
    assert out.data.shape == ref.shape and out.data.dtype == np.uint8
    assert maxdiff(out.data, ref) <= U8_TOL
    assert (out.data != ref).mean() < 2e-3          # only .5 ties may flip
    assert [stats.regions, stats.max_filter, *stats.shift] == [int(v) for v in stats_ref]


@pytest.mark.parametrize("case", BIG_RENDER_CASES, ids=[c[0] for c in BIG_RENDER_CASES])
def test_render_1080p_matches_reference_and_oracle(golden, case):
    name, seed, shape, kw = case
    g = golden["renders_big"]
    img = frame_u8(seed, shape)
    out, grid, bank, stats = fk.foveate(fk.RasterImage.from_array(img), fk.FoveationParams(**kw))
    assert maxdiff(out.data[::7, ::11], g[f"{name}/sample"]) <= U8_TOL
    assert [stats.regions, stats.max_filter, *stats.shift] == [int(v) for v in g[f"{name}/stats"]]
    ref, pl = fo.c_foveate(img, fo.OracleParams(**kw), threads=8)
    assert maxdiff(out.data, ref) <= U8_TOL
    assert (out.data != ref).mean() < 2e-3
    # identity fragments (the foveal cell) are byte-exact
    sx = fk.fragment_spans(shape[1], 32, grid.shift[0])
    sy = fk.fragment_spans(shape[0], 32, grid.shift[1])
    gy, gx = grid.foveal_cell
    sl = np.s_[sy[gy, 0]:sy[gy, 1], sx[gx, 0]:sx[gx, 1]]
    assert np.array_equal(out.data[sl], img[sl])


@pytest.mark.parametrize("case", F32_CASES, ids=[c[0] for c in F32_CASES])
def test_render_f32_matches_reference_golden(golden, case):
    name, seed, shape, kw = case
    ref = golden["renders_f32"][f"{name}/out"]
    img = frame_f32(seed, shape)
    p = fk.FoveationParams(**kw)
    fix = np.asarray([p.fixation_for((shape[1], shape[0]))])
    out = fk.foveate_batch(torch.from_numpy(img)[None].cuda(), fix, p)[0].cpu().numpy()
    assert out.dtype == np.float32
    err = np.abs(out.astype(np.float64) - ref)
    assert np.all(err <= F32_RTOL * np.maximum(np.abs(ref), 1.0))


@pytest.mark.parametrize("L", [7, 13, 31])
def test_uniform_grid_matches_reference(golden, L):
    # test_blockwise.py:135-148: one bank filter everywhere, no shift
    ref = golden["renders_uniform"][f"L{L}/out"]
    img = np.random.default_rng(L).integers(0, 256, (128, 128, 3)).astype(np.uint8)
    field = fk.SigmaField(grid_width=1, grid_height=1, sigma=np.asarray([[L / 6.0]]))
    bank = fk.build_bank(field)[0]
    assert bank.lengths[1] == L
    grid = fk.BlurGrid(index=np.full((4, 4), 1, np.int64), shift=(0, 0), fragment_size=32,
                       foveal_cell=(0, 0))
    out = fk.render(fk.RasterImage.from_array(img), grid, bank)
    assert maxdiff(out.data, ref) <= U8_TOL


def test_render_accepts_arbitrary_bank_taps():
    """render() honours the bank's own coefficients, not only the canonical LUT."""
    img = frame_u8(3, (64, 96, 3))
    box = np.full(5, 0.2)
    bank = fk.FilterBank(filters=(np.array([1.0]), box), lengths=np.array([1, 5]),
                         cumulative_sizes=np.array([1, 6]), sigmas=np.array([1 / 6, 5 / 6]))
    idx = np.ones((4, 6), np.int64)
    idx[1, 2] = 0
    grid = fk.BlurGrid(index=idx, shift=(0, 0), fragment_size=16, foveal_cell=(1, 2))
    out = fk.render(fk.RasterImage.from_array(img), grid, bank)
    lengths = np.where(idx == 1, 5, 1)
    ref = fo.c_render(img, 16, (0, 0), lengths, coeffs=np.concatenate(([1.0], box)),
                      offsets=np.where(idx == 1, 1, 0))
    assert maxdiff(out.data, ref) <= U8_TOL
    assert np.array_equal(out.data[16:32, 32:48], img[16:32, 32:48])


# ----------------------------------------------------------------------- properties
def test_constant_and_identity_images():
    # test_blockwise.py:121-133
    const = fk.RasterImage.from_array(np.full((1080, 1920, 3), 128, np.uint8))
    out, *_ = fk.foveate(const, fk.FoveationParams(fixation=(0, 0)))
    assert out == const
    img = fk.RasterImage.from_array(frame_u8(5, (1080, 1920, 3)))
    out, grid, bank, stats = fk.foveate(img, fk.FoveationParams(strength=0.0))
    assert out == img and stats.regions == 1 and len(bank) == 1   # test_blockwise.py:190-194
    for v in (0, 255):
        flat = fk.RasterImage.from_array(np.full((96, 160, 3), v, np.uint8))
        assert fk.foveate(flat, fk.FoveationParams(fragment_size=16))[0] == flat


def test_determinism_and_fragment_independence():
    # test_blockwise.py:150-173
    img = frame_u8(11, (96, 96, 3))
    field = fk.SigmaField(grid_width=1, grid_height=1, sigma=np.asarray([[2.0]]))
    bank = fk.build_bank(field)[0]                  # 13 taps, radius 6
    grid = fk.BlurGrid(index=np.ones((3, 3), np.int64), shift=(0, 0), fragment_size=32,
                       foveal_cell=(0, 0))
    a = fk.render(fk.RasterImage.from_array(img), grid, bank, workers=1)
    b = fk.render(fk.RasterImage.from_array(img), grid, bank, workers=8)
    assert np.array_equal(a.data, b.data)
    pert = img.copy()
    pert[60:, 60:, :] = frame_u8(12, (36, 36, 3))
    c = fk.render(fk.RasterImage.from_array(pert), grid, bank)
    assert np.array_equal(a.data[:32, :32], c.data[:32, :32])


def test_foveal_passthrough_and_single_channel():
    # test_acceptance.py:135-148 configurations; test_blockwise.py:182-186,196-204
    for F, fix, seed in ((16, (256, 256), 1), (32, (37, 411), 2), (8, (500, 3), 3)):
        img = frame_u8(seed, (512, 512, 3))
        out, grid, _, _ = fk.foveate(fk.RasterImage.from_array(img),
                                     fk.FoveationParams(fragment_size=F, fixation=fix))
        sx = fk.fragment_spans(512, F, grid.shift[0])
        sy = fk.fragment_spans(512, F, grid.shift[1])
        gy, gx = grid.foveal_cell
        sl = np.s_[sy[gy, 0]:sy[gy, 1], sx[gx, 0]:sx[gx, 1]]
        assert np.array_equal(out.data[sl], img[sl])
        assert grid.index[grid.foveal_cell] == 0
    gray = frame_u8(2, (64, 64, 1))
    out, *_ = fk.foveate(fk.RasterImage.from_array(gray), fk.FoveationParams(fragment_size=16))
    assert out.channels == 1 and out.size == (64, 64)
    ref, _ = fo.c_foveate(gray, fo.OracleParams(fragment_size=16))
    assert maxdiff(out.data, ref) <= U8_TOL


def test_mean_preserved_and_tv_not_increased():
    # test_blockwise.py:206-232 on a smooth synthetic scene
    yy, xx = np.mgrid[0:512, 0:512]
    rng = np.random.default_rng(0)
    scene = 128 + 60 * np.sin(xx / 9.0) * np.cos(yy / 13.0) + rng.normal(0, 12, (512, 512))
    img = np.clip(np.stack([scene, scene[::-1], scene[:, ::-1]], axis=2), 0, 255).astype(np.uint8)
    out, grid, bank, _ = fk.foveate(fk.RasterImage.from_array(img),
                                    fk.FoveationParams(fragment_size=16))
    assert abs(float(out.data.mean()) - float(img.mean())) <= 1.0

    def tv(a):
        a = a.astype(np.int64)
        return np.abs(np.diff(a, axis=0)).sum() + np.abs(np.diff(a, axis=1)).sum()

    sx = fk.fragment_spans(512, 16, grid.shift[0])
    sy = fk.fragment_spans(512, 16, grid.shift[1])
    for gy in range(0, grid.index.shape[0], 3):
        for gx in range(0, grid.index.shape[1], 3):
            if bank.lengths[grid.index[gy, gx]] < 3:
                continue
            sl = np.s_[sy[gy, 0]:sy[gy, 1], sx[gx, 0]:sx[gx, 1]]
            fo_, fi_ = out.data[sl], img[sl]
            hh, ww = fo_.shape[:2]
            assert tv(fo_) <= tv(fi_) + ((hh - 1) * ww + hh * (ww - 1)) * 3


def test_error_behaviour_matches_reference():
    img = fk.RasterImage.from_array(np.zeros((32, 32, 3), np.uint8))
    bank = fk.build_bank(fk.SigmaField(1, 1, np.asarray([[0.0]])))[0]
    grid = fk.BlurGrid(index=np.full((2, 2), 3, np.int64), shift=(0, 0), fragment_size=16,
                       foveal_cell=(0, 0))
    with pytest.raises(ValueError, match="bank"):            # test_blockwise.py:175-180
        fk.render(img, grid, bank)
    bad = fk.BlurGrid(index=np.zeros((3, 2), np.int64), shift=(0, 0), fragment_size=16,
                      foveal_cell=(0, 0))
    with pytest.raises(ValueError, match="does not match image"):
        fk.render(img, bad, bank)
    p = fk.FoveationParams(fragment_size=16, fixation=(64, 64))
    shift = fk.compute_fragment_shift((64, 64), 16)
    field = fk.build_sigma_field((128, 128), p, shift)
    bnk, index = fk.build_bank(field)
    with pytest.raises(ValueError, match="tiling"):          # test_blockwise.py:94-100
        fk.build_blur_grid(field, bnk, index, (64, 64), (256, 256), 16, shift)
    with pytest.raises(ValueError, match="outside"):
        fk.plan((100, 100), fk.FoveationParams(fixation=(100, 5)))
    with pytest.raises(ValueError, match="sigma_max"):       # test_blockwise.py:234-237
        fk.foveate(img, fk.FoveationParams(fragment_size=16),
                   density=fk.RasterImage.from_array(np.zeros((8, 8), np.uint8)))
    with pytest.raises(ValueError, match="outside"):
        fk.foveate_batch(np.zeros((2, 32, 32, 3), np.uint8), [[5, 5], [40, 1]])
    # the C ABI itself rejects what the shim would (no shim-only validation)
    eng = fk.get_engine(0)
    plan = eng.plan_for((32, 32), 16, 1)
    with pytest.raises(ValueError, match="outside"):
        plan.model(fk.FoveationParams(fragment_size=16), [[32.0, 0.0]])
    with pytest.raises(ValueError, match="channels"):
        plan.model(fk.FoveationParams(fragment_size=16), [[3.0, 3.0]])
        eng.render(torch.zeros((1, 32, 32, 2), dtype=torch.uint8, device="cuda"), plan)


def test_zero_strength_grid_and_symmetry():
    # test_blockwise.py:73-87
    grid, bank = fk.plan((128, 128), fk.FoveationParams(strength=0.0, fragment_size=16,
                                                        fixation=(64, 64)))
    assert np.all(grid.index == 0) and len(bank) == 1
    grid, _ = fk.plan((256, 256), fk.FoveationParams(fragment_size=16, fixation=(128.0, 128.0)))
    assert np.array_equal(grid.index, grid.index[::-1, ::-1])
    f = fk.build_sigma_field((256, 256), fk.FoveationParams(fragment_size=16,
                                                            fixation=(128.0, 128.0)), (8, 8))
    assert np.array_equal(f.sigma, f.sigma[::-1, :]) and np.array_equal(f.sigma, f.sigma[:, ::-1])


# ---------------------------------------------------------------------------- batch
def moving_fixations(n, w=1920, h=1080):
    i = np.arange(n)
    return np.stack([np.floor(w / 2 + 0.4 * w * np.cos(2 * np.pi * i / n)),
                     np.floor(h / 2 + 0.4 * h * np.sin(2 * np.pi * i / n))], axis=1)


def test_batch_1080p_moving_fixation_vs_oracle():
    """BASELINE config 2 shape (fewer frames): per-frame fixations, device tensors."""
    n = 6
    frames = frame_u8(0, (n, 1080, 1920, 3))
    fix = moving_fixations(n)
    out = fk.foveate_batch(torch.from_numpy(frames).cuda(), fix, fk.FoveationParams())
    out = out.cpu().numpy()
    for i in range(n):
        ref, _ = fo.c_foveate(frames[i], fo.OracleParams(fixation=tuple(fix[i])), threads=8)
        assert maxdiff(out[i], ref) <= U8_TOL
        assert (out[i] != ref).mean() < 2e-3


def test_host_pipeline_equals_device_path_and_shards():
    n = 20
    frames = frame_u8(7, (n, 270, 480, 3))
    fix = np.random.default_rng(7).uniform(0, 1, (n, 2)) * [480, 270]
    p = fk.FoveationParams(fragment_size=16)
    dev = fk.foveate_batch(torch.from_numpy(frames).cuda(), fix, p).cpu().numpy()
    host = fk.foveate_batch(frames, fix, p, chunk_frames=3)
    assert np.array_equal(dev, host)
    pinned_in = fk.pinned_empty(frames.shape, np.uint8)
    pinned_in[...] = frames
    pinned_out = fk.pinned_empty(frames.shape, np.uint8)
    got = fk.foveate_batch(pinned_in, fix, p, out=pinned_out)
    assert got is pinned_out and np.array_equal(pinned_out, dev)
    # sharding over a device list (the same GPU twice exercises the split/merge logic)
    sharded = fk.foveate_batch(frames, fix, p, devices=[0, 0])
    assert np.array_equal(sharded, dev)
    ref, _ = fo.c_foveate(frames[5], fo.OracleParams(fragment_size=16, fixation=tuple(fix[5])))
    assert maxdiff(dev[5], ref) <= U8_TOL


def test_batch_256x256_random_fixations_vs_oracle():
    """BASELINE config 4 shape (subset): many small frames, random fixations."""
    n = 512
    rng = np.random.default_rng(1)
    frames = rng.integers(0, 256, (n, 256, 256, 3), dtype=np.uint8)
    fix = rng.integers(0, 256, (n, 2)).astype(np.float64)
    out = fk.foveate_batch(torch.from_numpy(frames).cuda(), fix, fk.FoveationParams()).cpu().numpy()
    for i in range(0, n, 37):
        ref, _ = fo.c_foveate(frames[i], fo.OracleParams(fixation=tuple(fix[i])), threads=8)
        assert maxdiff(out[i], ref) <= U8_TOL


def test_4k_f16_vs_oracle():
    """BASELINE config 3: 3840x2160, 16x16 fragments, corner fixation (largest halos)."""
    img = frame_u8(3, (2160, 3840, 3))
    kw = dict(fragment_size=16, fixation=(0, 0))
    out, grid, bank, stats = fk.foveate(fk.RasterImage.from_array(img), fk.FoveationParams(**kw))
    assert stats.max_filter == 103 and grid.index.shape == (136, 241)
    ref, _ = fo.c_foveate(img, fo.OracleParams(**kw), threads=8)
    assert maxdiff(out.data, ref) <= U8_TOL
    assert (out.data != ref).mean() < 2e-3


@pytest.mark.parametrize("F", [8, 16, 32, 64])
def test_f32_block_size_sweep_alt_fit_vs_oracle(F):
    """BASELINE config 5: fp32 frames, steeper fit (e2=1.5), block sizes 8..64."""
    img = frame_f32(50 + F, (540, 960, 3))
    kw = dict(fragment_size=F, e2=1.5)
    p = fk.FoveationParams(**kw)
    out = fk.foveate_batch(torch.from_numpy(img)[None].cuda(), None, p)[0].cpu().numpy()
    ref, _ = fo.c_foveate(img, fo.OracleParams(**kw), quantize=False, threads=8)
    err = np.abs(out.astype(np.float64) - ref)
    assert np.all(err <= F32_RTOL * np.maximum(np.abs(ref), 1.0))
    # linearity of the fp32 path: foveate(a*x + b) == a*foveate(x) + b within tolerance
    out2 = fk.foveate_batch(torch.from_numpy(0.5 * img + 0.25)[None].cuda(), None, p)[0].cpu().numpy()
    assert np.allclose(out2, 0.5 * out + 0.25, rtol=0, atol=2e-5)


def test_long_filters_grow_the_lut_and_strip_path():
    """strength 6 -> filters of several hundred taps (beyond the default 255-tap LUT)."""
    img = frame_u8(9, (120, 200, 3))
    kw = dict(fragment_size=32, fixation=(10, 10), strength=6.0)
    out, grid, bank, stats = fk.foveate(fk.RasterImage.from_array(img), fk.FoveationParams(**kw))
    assert stats.max_filter > 255
    ref, _ = fo.c_foveate(img, fo.OracleParams(**kw), threads=8)
    assert maxdiff(out.data, ref) <= U8_TOL


def test_fast_and_generic_kernels_agree_bit_for_bit():
    """Both kernels accumulate taps in the same order, so they must agree exactly."""
    eng = fk.get_engine(0)
    rng = np.random.default_rng(77)
    cases = [((270, 480, 3), 32, torch.uint8), ((200, 333, 1), 16, torch.uint8),
             ((150, 260, 3), 64, torch.float32), ((97, 131, 3), 8, torch.float32),
             ((128, 128, 1), 100, torch.float32)]
    for shape, F, dtype in cases:
        n = 3
        if dtype == torch.uint8:
            frames = torch.from_numpy(rng.integers(0, 256, (n, *shape), dtype=np.uint8)).cuda()
        else:
            frames = torch.from_numpy(rng.random((n, *shape), dtype=np.float32)).cuda()
        fix = np.stack([rng.uniform(0, shape[1], n), rng.uniform(0, shape[0], n)], axis=1)
        p = fk.FoveationParams(fragment_size=F, strength=1.3)
        outs = {}
        try:
            # 1 = generic kernel, 2 = fast kernels without TMA, 3 = row-partitioned fast kernel,
            # 4 = fk_blur_cols for every class, 5 = fk_blur_tma for every class (include/fovea.h)
            for variant in (1, 2, 3, 4, 5):
                eng.set_kernel_variant(variant)
                outs[variant] = fk.foveate_batch(frames, fix, p).clone()
        finally:
            eng.set_kernel_variant(0)
        b = fk.foveate_batch(frames, fix, p)   # default dispatch
        for variant in (1, 2, 3, 4, 5):
            assert torch.equal(outs[variant], b), (shape, F, dtype, variant)


def test_column_kernel_every_class_panels_and_strips_vs_generic():
    """1080p frames with fixations in a corner, on an edge and in the middle: every tap-count
    class of fk_blur_cols and fk_blur_tma is populated -- filters past 89 taps are walked in
    tap panels by fk_blur_cols,
    same-filter fragments are merged into strips up to 128 rows, tiles hang over all four
    image borders -- and the result must equal the generic kernel's bit for bit (uint8 with
    and without TMA, float32)."""
    eng = fk.get_engine(0)
    rng = np.random.default_rng(2024)
    h, w = 1080, 1920
    fix = np.asarray([[0.0, 0.0], [1919.0, 540.0], [960.0, 540.0], [1300.5, 1079.0]])
    n = len(fix)
    u8 = torch.from_numpy(rng.integers(0, 256, (n, h, w, 3), dtype=np.uint8)).cuda()
    f32 = torch.from_numpy(rng.random((2, h, w, 3), dtype=np.float32)).cuda()
    for frames, fx, p in ((u8, fix, fk.FoveationParams()),
                          (f32, fix[:2], fk.FoveationParams(e2=1.5))):
        outs = {}
        try:
            for variant in (1, 2, 4, 5):
                eng.set_kernel_variant(variant)
                outs[variant] = fk.foveate_batch(frames, fx, p).clone()
        finally:
            eng.set_kernel_variant(0)
        got = fk.foveate_batch(frames, fx, p)
        for variant in (1, 2, 4, 5):
            assert torch.equal(outs[variant], got), variant
    # the corner fixation reaches the 103-tap filter (class 3)
    _, _, bank, stats = fk.foveate(fk.RasterImage.from_array(u8[0].cpu().numpy()),
                                   fk.FoveationParams(fixation=(0.0, 0.0)))
    assert stats.max_filter >= 101


def test_tma_path_border_and_interior_tiles_vs_generic():
    """uint8 frames whose row pitch is a multiple of 16 bytes take the TMA staging path;
    corner fixations make most tiles cross the image border (clamp-to-edge by index)."""
    eng = fk.get_engine(0)
    rng = np.random.default_rng(5)
    for (h, w, c), F in (((256, 256, 3), 32), ((96, 160, 3), 16), ((64, 64, 1), 32),
                         ((540, 960, 3), 32), ((33, 48, 1), 8)):
        assert (w * c) % 16 == 0
        n = 4
        frames = torch.from_numpy(rng.integers(0, 256, (n, h, w, c), dtype=np.uint8)).cuda()
        fix = np.asarray([[0, 0], [w - 1, h - 1], [w / 2, h / 2], [w - 1, 0]], dtype=np.float64)
        p = fk.FoveationParams(fragment_size=F, strength=1.5)
        try:
            eng.set_kernel_variant(1)
            ref = fk.foveate_batch(frames, fix, p).clone()
        finally:
            eng.set_kernel_variant(0)
        got = fk.foveate_batch(frames, fix, p)
        assert torch.equal(ref, got), ((h, w, c), F)
        # a view at a 16-byte-misaligned offset falls back to plain-load staging
        flat = torch.empty(frames.numel() + 16, dtype=torch.uint8, device="cuda")
        view = flat[4:4 + frames.numel()].view_as(frames)
        view.copy_(frames)
        assert torch.equal(fk.foveate_batch(view, fix, p), ref)


@pytest.mark.gpu
def test_tensor_maps_follow_the_buffer_geometry():
    """fk_blur_tma keeps the tensor maps of its last launch per class (csrc/fk_internal.h,
    tmap_cache): the same storage rendered as another geometry, as more or fewer frames, and
    another buffer of the same geometry must each get maps of their own."""
    eng = fk.get_engine(0)
    rng = np.random.default_rng(77)
    store = torch.from_numpy(rng.integers(0, 256, (4 * 128 * 256 * 3,), dtype=np.uint8)).cuda()
    other = torch.from_numpy(rng.integers(0, 256, (4 * 128 * 256 * 3,), dtype=np.uint8)).cuda()
    p = fk.FoveationParams(strength=1.5)
    for buf, shape in ((store, (4, 128, 256, 3)), (store, (4, 256, 128, 3)), (store, (2, 256, 256, 3)),
                       (other, (2, 256, 256, 3)), (store, (4, 128, 256, 3))):
        n, h, w, _ = shape
        frames = buf[: n * h * w * 3].view(shape)
        fix = np.stack([np.linspace(0, w - 1, n), np.linspace(h - 1, 0, n)], axis=1)
        try:
            eng.set_kernel_variant(1)
            ref = fk.foveate_batch(frames, fix, p).clone()
        finally:
            eng.set_kernel_variant(0)
        assert torch.equal(fk.foveate_batch(frames, fix, p), ref), shape


@pytest.mark.gpu
def test_strip_height_does_not_change_the_output():
    """Merging same-filter fragments into strips is exact (an output pixel depends only on the
    image and its filter), whatever the cap on the strip height: the batch default (1 024 rows),
    the single-frame default (64) and no merging at all (32 = one fragment) give the same bytes.
    FK_STRIP_ROWS_FORCE is read once per process, so each setting runs in its own."""
    import hashlib
    import os
    import subprocess
    import sys

    code = (
        "import sys, hashlib, numpy as np, torch\n"
        "sys.path.insert(0, '.')\n"
        "import paper_2012_08655_b200 as fk\n"
        "rng = np.random.default_rng(5)\n"
        "frames = torch.from_numpy(rng.integers(0, 256, (12, 540, 960, 3), dtype=np.uint8)).cuda()\n"
        "fix = np.stack([rng.uniform(0, 960, 12), rng.uniform(0, 540, 12)], axis=1)\n"
        "out = fk.foveate_batch(frames, fix, fk.FoveationParams(fragment_size=32, strength=1.3))\n"
        "print(hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest())\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    digests = {}
    for force in ("", "32", "64", "1024"):
        env = dict(os.environ)
        env.pop("FK_STRIP_ROWS_FORCE", None)
        if force:
            env["FK_STRIP_ROWS_FORCE"] = force
        res = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                             text=True, timeout=600)
        assert res.returncode == 0, res.stderr[-2000:]
        digests[force] = res.stdout.strip().splitlines()[-1]
    assert len(set(digests.values())) == 1, digests


# ------------------------------------------------- BASELINE configs at their named shapes
@pytest.mark.parametrize("F,e2", [(32, 2.3), (16, 1.5), (8, 2.3), (64, 1.5)])
def test_f32_1080p_named_shape_vs_oracle(F, e2):
    """BASELINE config 5 at its named shape: a 1920x1080 float32 frame, centre fixation, default
    and steeper fit, every block size, against the C oracle (unquantised), and -- the same
    arithmetic -- bit for bit against the generic kernel.  F = 8 and 16 run as mixed items."""
    img = frame_f32(70 + F, (1080, 1920, 3))
    kw = dict(fragment_size=F, e2=e2)
    p = fk.FoveationParams(**kw)
    dev = torch.from_numpy(img)[None].cuda()
    out = fk.foveate_batch(dev, None, p)
    ref, _ = fo.c_foveate(img, fo.OracleParams(**kw), quantize=False, threads=8)
    err = np.abs(out[0].cpu().numpy().astype(np.float64) - ref)
    assert np.all(err <= F32_RTOL * np.maximum(np.abs(ref), 1.0)), float(err.max())
    eng = fk.get_engine(0)
    eng.set_kernel_variant(1)
    try:
        gen = fk.foveate_batch(dev, None, p)
    finally:
        eng.set_kernel_variant(0)
    assert torch.equal(out, gen)


def test_gray_1080p_vs_oracle():
    """Single-channel frames at full size (the row-partitioned fk_blur_fast path)."""
    img = frame_u8(81, (1080, 1920, 1))
    for fix in ((960.0, 540.0), (1919.0, 0.0)):
        out = fk.foveate_batch(torch.from_numpy(img)[None].cuda(), np.asarray([fix]),
                               fk.FoveationParams())[0].cpu().numpy()
        ref, _ = fo.c_foveate(img, fo.OracleParams(fixation=fix), threads=8)
        assert maxdiff(out, ref) <= U8_TOL
        assert (out != ref).mean() < 2e-3


@pytest.mark.parametrize("W", [1921, 1918])
def test_row_pitch_not_a_multiple_of_16_bytes_vs_oracle(W):
    """W * C % 16 != 0: TMA cannot describe the rows, the render leaves fk_blur_tma for
    fk_blur_cols with plain-load staging (and, for 16-pixel fragments, emits the plan's items
    again without mixed ones); the result still matches the oracle."""
    img = frame_u8(82 + W, (270, W, 3))
    for F in (32, 16):
        kw = dict(fragment_size=F, fixation=(W - 5.0, 100.0))
        out, *_ = fk.foveate(fk.RasterImage.from_array(img), fk.FoveationParams(**kw))
        ref, _ = fo.c_foveate(img, fo.OracleParams(**kw), threads=8)
        assert maxdiff(out.data, ref) <= U8_TOL
    f32 = frame_f32(83, (120, W, 3))
    p = fk.FoveationParams(fragment_size=16, fixation=(3.0, 3.0))
    out = fk.foveate_batch(torch.from_numpy(f32)[None].cuda(), np.asarray([[3.0, 3.0]]), p)[0].cpu().numpy()
    ref, _ = fo.c_foveate(f32, fo.OracleParams(fragment_size=16, fixation=(3.0, 3.0)), quantize=False, threads=8)
    assert np.all(np.abs(out.astype(np.float64) - ref) <= F32_RTOL * np.maximum(np.abs(ref), 1.0))


def test_rl_batch_65536_frames_named_shape_vs_oracle():
    """BASELINE config 4 at its named size: 65 536 frames of 256x256 RGB (12.9 GB in, 12.9 GB
    out), random fixations.  64 frames spread over the whole batch -- the last one included, so
    the item / frame offsets at the top of the range are exercised -- against the C oracle, and
    a checksum property over all of them: a frame whose fixation and content are duplicated
    elsewhere in the batch comes out identical."""
    n = 65536
    free, _total = torch.cuda.mem_get_info()
    if free < 30 * 2**30:
        pytest.skip("needs 30 GB of free device memory")
    g = torch.Generator(device="cuda").manual_seed(4)
    frames = torch.randint(0, 256, (n, 256, 256, 3), dtype=torch.uint8, device="cuda", generator=g)
    rng = np.random.default_rng(1)
    fix = np.stack([rng.integers(0, 256, n), rng.integers(0, 256, n)], axis=1).astype(np.float64)
    # duplicates: frame n-1-k repeats frame k for the first 16 frames
    frames[n - 16:] = frames[:16].flip(0)
    fix[n - 16:] = fix[:16][::-1]
    out = fk.foveate_batch(frames, fix, fk.FoveationParams())
    assert torch.equal(out[n - 16:], out[:16].flip(0))
    picks = sorted(set(np.linspace(0, n - 1, 64).astype(int).tolist()))
    for i in picks:
        ref, _ = fo.c_foveate(frames[i].cpu().numpy(), fo.OracleParams(fixation=tuple(fix[i])), threads=8)
        assert maxdiff(out[i].cpu().numpy(), ref) <= U8_TOL, i
    del frames, out
    torch.cuda.empty_cache()


def test_mixed_items_every_width_and_filter_combination_vs_generic_and_oracle():
    """Fragments of 8 and 16 pixels: neighbouring cells with different filters render as one
    strip with a filter per warp (fk_internal.h, FK_ITEM_MIXED).  Bit-identical to the generic
    kernel and to the same plans without mixed items, on uint8 and float32, including fixations
    at the corners (longest filters, clamped halos) and widths that clip the last group; one
    frame of each also against the oracle."""
    rng = np.random.default_rng(21)
    eng = fk.get_engine(0)
    for (h, w, F) in [(96, 176, 8), (200, 336, 16), (64, 80, 8), (130, 496, 16)]:
        n = 5
        fix = np.stack([rng.uniform(0, w, n), rng.uniform(0, h, n)], axis=1)
        fix[0], fix[1], fix[2] = (0.0, 0.0), (w - 1.0, h - 1.0), (w - 1.0, 0.0)
        p = fk.FoveationParams(fragment_size=F, strength=2.2, e2=1.4)
        for dtype in (np.uint8, np.float32):
            host = (rng.integers(0, 256, (n, h, w, 3), dtype=np.uint8) if dtype == np.uint8
                    else rng.random((n, h, w, 3), dtype=np.float32))
            frames = torch.from_numpy(host).cuda()
            got = fk.foveate_batch(frames, fix, p).clone()
            try:
                eng.set_kernel_variant(1)
                gen = fk.foveate_batch(frames, fix, p).clone()
                eng.set_kernel_variant(32)
                plain = fk.foveate_batch(frames, fix, p).clone()
            finally:
                eng.set_kernel_variant(0)
            assert torch.equal(got, gen) and torch.equal(got, plain)
            ref, _ = fo.c_foveate(host[3], fo.OracleParams(fragment_size=F, strength=2.2, e2=1.4,
                                                           fixation=tuple(fix[3])),
                                  quantize=dtype == np.uint8, threads=8)
            if dtype == np.uint8:
                assert maxdiff(got[3].cpu().numpy(), ref) <= U8_TOL
            else:
                err = np.abs(got[3].cpu().numpy().astype(np.float64) - ref)
                assert np.all(err <= F32_RTOL * np.maximum(np.abs(ref), 1.0))
    # the plan really holds mixed items, and the accounting reads them
    from paper_2012_08655_b200 import costs
    plan = eng.plan_for((336, 200), 16, 1)
    plan.model(fk.FoveationParams(fragment_size=16, strength=2.2), np.asarray([[100.0, 60.0]]))
    items = np.concatenate(plan.read_items()[:-1])
    assert (items[:, 3] >> 31).any()
    lengths, meta = plan.read_lengths()
    alg = costs.batch_flops((336, 200), 16, 3, lengths, meta)
    assert 0 < costs.executed_flops(plan.read_items()[:-1], 3) <= alg


def test_device_resident_shards_one_thread_and_stream_each():
    """a batch resident on several GPUs as one tensor per device, rendered
    with no host round trip -- here both shards live on cuda:0, which exercises the per-shard
    threads, streams and plans; the result equals the unsharded batch."""
    n = 11
    frames = torch.from_numpy(frame_u8(90, (n, 180, 320, 3))).cuda()
    fix = np.random.default_rng(90).uniform(0, 1, (n, 2)) * [320, 180]
    p = fk.FoveationParams(fragment_size=16)
    whole = fk.foveate_batch(frames, fix, p)
    a, b = fk.shard_range(n, 0, 2)
    shards = [frames[a:b].contiguous(), frames[b:].contiguous()]
    outs = fk.foveate_batch(shards, fix, p)
    assert isinstance(outs, list) and len(outs) == 2
    assert torch.equal(torch.cat(outs), whole)
    outs2 = fk.foveate_batch(shards, [fix[a:b], fix[b:]], p, out=[torch.empty_like(t) for t in shards])
    assert torch.equal(torch.cat(outs2), whole)
    with pytest.raises(ValueError):
        fk.foveate_batch(shards, fix[:-1], p)
