import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2012_08655_b200 as fk
from paper_2012_08655_b200 import _native
lib = _native.lib()
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
