"""Seeded input definitions shared by make_golden.py (reference side, build container)
and the tests (oracle / CUDA side).  No reference import here: this file travels."""

import numpy as np

# name, (W, H), params kwargs, use_shift  -- the BASELINE.json configs plus the
# reference tests' own cases (test_blockwise.py, test_retinal.py, test_acceptance.py)
PLAN_CASES = [
    ("c1_1080p_f32_centre", (1920, 1080), dict(fragment_size=32), True),
    ("c1_1080p_f32_fix960_540", (1920, 1080), dict(fragment_size=32, fixation=(960, 540)), True),
    ("c1_1080p_f32_corner", (1920, 1080), dict(fragment_size=32, fixation=(0, 0)), True),
    ("c1_1080p_f32_farcorner", (1920, 1080), dict(fragment_size=32, fixation=(1919, 1079)), True),
    ("c1_1080p_f32_frac", (1920, 1080), dict(fragment_size=32, fixation=(1234.56, 321.125)), True),
    ("c3_4k_f16_centre", (3840, 2160), dict(fragment_size=16), True),
    ("c3_4k_f16_corner", (3840, 2160), dict(fragment_size=16, fixation=(0, 0)), True),
    ("c4_256_f32_centre", (256, 256), dict(fragment_size=32), True),
    ("c4_256_f32_rand", (256, 256), dict(fragment_size=32, fixation=(201, 17)), True),
    ("c5_1080p_f8_alt", (1920, 1080), dict(fragment_size=8, e2=1.5), True),
    ("c5_1080p_f16_alt", (1920, 1080), dict(fragment_size=16, e2=1.5), True),
    ("c5_1080p_f32_alt", (1920, 1080), dict(fragment_size=32, e2=1.5), True),
    ("c5_1080p_f64_alt", (1920, 1080), dict(fragment_size=64, e2=1.5), True),
    ("c5_1080p_f32_fmax30", (1920, 1080), dict(fragment_size=32, f_max=30.0), True),
    ("c5_1080p_f64_default", (1920, 1080), dict(fragment_size=64), True),
    ("t_256_f16_centre", (256, 256), dict(fragment_size=16, fixation=(128.0, 128.0)), True),
    ("t_256_f16_100_80", (256, 256), dict(fragment_size=16, fixation=(100, 80)), True),
    ("t_128_f16_zero", (128, 128), dict(fragment_size=16, fixation=(64, 64), strength=0.0), True),
    ("t_160_f16_83_57", (160, 160), dict(fragment_size=16, fixation=(83, 57)), True),
    ("t_512_f32_37_411", (512, 512), dict(fragment_size=32, fixation=(37, 411)), True),
    ("t_512_f8_500_3", (512, 512), dict(fragment_size=8, fixation=(500, 3)), True),
    ("t_odd_301x203_f12", (301, 203), dict(fragment_size=12, fixation=(17.5, 190.25), strength=1.7), True),
    ("t_noshift_200x120_f32", (200, 120), dict(fragment_size=32, fixation=(77, 13)), False),
    ("t_tiny_5x7_f4", (5, 7), dict(fragment_size=4, fixation=(2, 3)), True),
    ("t_strong_640x360_f32", (640, 360), dict(fragment_size=32, fixation=(10, 350), strength=2.5, e_corner=75.0), True),
]

# name, seed, (H, W, C), params kwargs  -- rendered outputs stored in full (small)
RENDER_CASES = [
    ("r_rgb_160x200_f16", 11, (160, 200, 3), dict(fragment_size=16, fixation=(83, 57))),
    ("r_rgb_203x301_f12", 12, (203, 301, 3), dict(fragment_size=12, fixation=(17.5, 190.25), strength=1.7)),
    ("r_gray_96x128_f32", 13, (96, 128, 1), dict(fragment_size=32, fixation=(100, 40))),
    ("r_rgb_256x256_f32_corner", 14, (256, 256, 3), dict(fragment_size=32, fixation=(0, 0))),
    ("r_rgb_256x256_f32_centre", 15, (256, 256, 3), dict(fragment_size=32)),
    ("r_rgb_120x90_f8", 16, (120, 90, 3), dict(fragment_size=8, fixation=(45, 60), e2=1.5)),
    ("r_rgb_64x64_f64", 17, (64, 64, 3), dict(fragment_size=64, fixation=(5, 5), strength=3.0)),
    ("r_rgb_33x47_f4", 18, (33, 47, 3), dict(fragment_size=4, fixation=(40, 2))),
]

# full-size frames: only a digest + a strided sample is stored
BIG_RENDER_CASES = [
    ("b_1080p_f32_centre", 0, (1080, 1920, 3), dict(fragment_size=32)),
    ("b_1080p_f32_corner", 1, (1080, 1920, 3), dict(fragment_size=32, fixation=(0, 0))),
]

F32_CASES = [  # fp32 frames: _render_cell with quantize_u8 replaced by identity
    ("f_rgb_128x160_f16", 21, (128, 160, 3), dict(fragment_size=16, fixation=(90, 31), e2=1.5)),
    ("f_rgb_96x96_f32", 22, (96, 96, 3), dict(fragment_size=32, fixation=(3, 90), f_max=30.0)),
]


def frame_u8(seed, shape):
    return np.random.default_rng(seed).integers(0, 256, shape, dtype=np.uint8)


def frame_f32(seed, shape):
    return np.random.default_rng(seed).random(shape, dtype=np.float32)




# name, map seed, (mh, mw), (W, H), F, shift, sigma_max  -- density-map sigma fields
DENSITY_CASES = [
    ("d_8x8_64_f16", 31, (8, 8), (64, 64), 16, (0, 0), 6.0),
    ("d_23x37_301x203_f12", 32, (23, 37), (301, 203), 12, (5, 11), 4.5),
    ("d_64x48_640x360_f32", 33, (64, 48), (640, 360), 32, (17, 3), 9.0),
    ("d_3x5_1920x1080_f32", 34, (3, 5), (1920, 1080), 32, (16, 12), 12.0),
]

# name, image seed, (H, W, C), map seed, (mh, mw), params kwargs, sigma_max -- rendered output
DENSITY_RENDER_CASES = [
    ("dr_rgb_120x160_f16", 41, (120, 160, 3), 42, (9, 13), dict(fragment_size=16, fixation=(70, 50)), 5.0),
]


def density_map(seed, shape):
    return np.random.default_rng(seed).integers(0, 256, shape, dtype=np.uint8)


# name, seed, (H, W, C), noise amplitude, smooth -- SSIM pairs (quality.ssim_map): the test image
# is the reference plus seeded integer noise; `smooth` images are low-frequency ramps
SSIM_CASES = [
    ("s_rgb_48x64", 21, (48, 64, 3), 12, False),
    ("s_gray_40x33", 22, (40, 33, 1), 30, True),
    ("s_rgb_min_11x11", 23, (11, 11, 3), 5, False),
    ("s_rgb_11x40", 24, (11, 40, 3), 9, True),
    ("s_rgb_identical_32x32", 25, (32, 32, 3), 0, True),
    ("s_rgb_1080p", 26, (1080, 1920, 3), 20, True),
]
SSIM_MEAN_CASE = ("s_mean_3pairs", (27, 28, 29), (57, 71, 3), 15, True)


def ssim_pair(seed, shape, amp, smooth):
    rng = np.random.default_rng(seed)
    h, w, c = shape
    if smooth:
        yy, xx = np.mgrid[0:h, 0:w]
        base = 127.5 + 100.0 * np.sin(xx / 9.0 + seed) * np.cos(yy / 7.0)
        ref = np.clip(base[..., None] + rng.integers(-8, 9, (h, w, c)), 0, 255).astype(np.uint8)
    else:
        ref = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
    noise = rng.integers(-amp, amp + 1, (h, w, c)) if amp else 0
    test = np.clip(ref.astype(np.int64) + noise, 0, 255).astype(np.uint8)
    return ref, test
