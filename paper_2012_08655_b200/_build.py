"""Build libfovea.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The shared object is git-ignored but travels with the working tree to the GPU box.  A
hash of the sources is stored next to it so a stale binary is rebuilt, never trusted.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
ROOT = PKG.parent
LIB = CSRC / "libfovea.so"
STAMP = CSRC / "libfovea.so.srchash"

SOURCES = ["fk_api.cu", "fk_plan.cu", "fk_blur.cu", "fk_blur_fast.cu", "fk_blur_cols.cu", "fk_ssim.cu"]
HEADERS = ["fk_internal.h", "fk_hypot.h", "fk_stage.cuh", "../../include/fovea.h"]

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
    "-shared", "-cudart", "static",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: libfovea.so cannot be built (there is no CPU fallback)")


def source_hash() -> str:
    h = hashlib.sha256()
    for name in SOURCES + HEADERS:
        h.update(name.encode())
        h.update((CSRC / name).read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def is_current() -> bool:
    return LIB.exists() and STAMP.exists() and STAMP.read_text().strip() == source_hash()


def build_native(force: bool = False, verbose: bool = False, debug_barriers: bool = False) -> Path:
    """Compile the CUDA sources into csrc/libfovea.so if missing or stale.  debug_barriers
    builds the racecheck variant (-DFK_DEBUG_CTA_BARRIERS, see fk_blur_cols.cu); the stamp is
    not written for it, so the next ordinary build replaces it."""
    if not force and not debug_barriers and is_current():
        return LIB
    if not force and not debug_barriers and LIB.exists() and os.environ.get("FK_KEEP_BUILD"):
        return LIB  # tools/racecheck.sh: run whatever was built last, stale stamp or not
    cmd = [_nvcc(), *NVCC_FLAGS]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    if debug_barriers:
        cmd += ["-DFK_DEBUG_CTA_BARRIERS"]
    cmd += ["-o", str(LIB), *[str(CSRC / s) for s in SOURCES]]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    if verbose:
        print(proc.stdout + proc.stderr)
    if debug_barriers:
        STAMP.write_text("debug-barriers build\n")
    else:
        STAMP.write_text(source_hash() + "\n")
    return LIB


if __name__ == "__main__":
    import sys

    print(build_native(force="--force" in sys.argv, verbose="-v" in sys.argv,
                       debug_barriers="--debug-barriers" in sys.argv))
