import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2012_08655_b200 as fk
from bench import moving_fixations
n, H, W, C = 256, 1080, 1920, 3
h_in = fk.pinned_empty((n, H, W, C), np.uint8); h_out = fk.pinned_empty((n, H, W, C), np.uint8)
h_in[...] = np.random.default_rng(0).integers(0, 256, (n, H, W, C), dtype=np.uint8)
fix = moving_fixations(n)
eng = fk.get_engine(0)
p = fk.FoveationParams()
for chunk in (0, 2, 4, 7, 12, 16, 32):
    for _ in range(2): eng.foveate_host(h_in, fix, p, out=h_out, chunk_frames=chunk)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(4): eng.foveate_host(h_in, fix, p, out=h_out, chunk_frames=chunk)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 4
    print("chunk", chunk, "fps", round(n / dt, 1), "GB/s each way", round(n * H * W * C / dt / 1e9, 1))
