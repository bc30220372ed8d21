"""Per-warp wait shares of fk_blur_tma on the headline batch.  Needs a libfovea.so built from a
fk_blur_cols.cu instrumented with clock64 around mbar_wait(bar), mbar_wait(hbar) and request_next
that exports fk_debug_wait_stats (16 counters: [0,4) cycles waiting for bytes per warp, [4,8) waits,
[8] cycles waiting for hbar, [9] cycles in the request, [12,16) kernel cycles per warp); the shipped
library has no such export (profiles/README.md holds the numbers measured with it)."""
import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2012_08655_b200 as fk
from paper_2012_08655_b200 import _native
lib = _native.lib()
if not hasattr(lib, "fk_debug_wait_stats"):
    sys.exit("this libfovea.so is not the instrumented build")
n = 256; H, W = 1080, 1920
frames = torch.from_numpy(np.random.default_rng(0).integers(0, 256, (n, H, W, 3), dtype=np.uint8)).cuda()
i = np.arange(n)
fix = np.stack([np.floor(960 + 768 * np.cos(2 * np.pi * i / 256)), np.floor(540 + 432 * np.sin(2 * np.pi * i / 256))], 1)
out = fk.foveate_batch(frames, fix, fk.FoveationParams())
torch.cuda.synchronize()
buf = (C.c_ulonglong * 16)()
lib.fk_debug_wait_stats(buf)
out = fk.foveate_batch(frames, fix, fk.FoveationParams())
torch.cuda.synchronize()
lib.fk_debug_wait_stats(buf)
v = list(buf)
print("bytes wait cycles per warp:", v[0:4]); print("waits:", v[4:8]); print("hbar wait (warp 0):", v[8]); print("kernel cycles per warp:", v[12:16])
print("duty cycles (thread 0, per block):", v[9], v[9] / max(v[4], 1), " hbar per block:", v[8] / max(v[4], 1), " kernel cycles per block:", v[12] / max(v[4], 1))
print("wait share per warp:", [round(v[w] / v[12 + w], 4) for w in range(4)], " hbar share warp0:", round(v[8] / v[12], 4))
