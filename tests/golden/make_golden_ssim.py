"""Golden SSIM maps FROM THE REFERENCE ITSELF (foveakit.quality.ssim_map / mean_ssim_map).

Run in the build container only:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_ssim.py

Inputs are regenerated from seeds by the tests (cases.ssim_pair); only reference OUTPUTS are
stored: the full map for small images, statistics and a strided sample for 1080p.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from foveakit import quality  # noqa: E402
from foveakit.imaging import RasterImage  # noqa: E402

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from cases import SSIM_CASES, SSIM_MEAN_CASE, ssim_pair  # noqa: E402


def pack(out, name, m, full):
    out[f"{name}/stats"] = np.asarray([m.mean, m.min, m.argmin[0], m.argmin[1]], np.float64)
    out[f"{name}/values"] = m.values if full else m.values[::37, ::41].copy()


def main():
    out = {}
    for name, seed, shape, amp, smooth in SSIM_CASES:
        ref, test = ssim_pair(seed, shape, amp, smooth)
        m = quality.ssim_map(RasterImage.from_array(ref), RasterImage.from_array(test))
        pack(out, name, m, full=shape[0] * shape[1] <= 64 * 64)
    name, seeds, shape, amp, smooth = SSIM_MEAN_CASE
    pairs = [tuple(RasterImage.from_array(a) for a in ssim_pair(s, shape, amp, smooth)) for s in seeds]
    pack(out, name, quality.mean_ssim_map(pairs), full=True)
    np.savez_compressed(HERE / "ssim.npz", **out)
    print("wrote", HERE / "ssim.npz", {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
