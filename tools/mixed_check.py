"""Mixed items (a filter per 8-pixel column, fk_internal.h) against the generic kernel, bit for
bit, on uint8 and float32 RGB frames with fragments narrower than 32 pixels -- and against the
same plans emitted without mixed items (variant | 32).
usage: python tools/mixed_check.py [cases] [seed]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_08655_b200 as fk

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
eng = fk.get_engine(0)
bad = 0
fixed = [(64, 64, 8), (40, 48, 16), (96, 160, 16), (270, 480, 8), (1080, 1920, 8), (1080, 1920, 16),
         (540, 960, 4), (256, 256, 16)]
for i in range(cases):
    if i < len(fixed):
        h, w, F = fixed[i]
    else:
        h = int(rng.integers(33, 400)); w = 16 * int(rng.integers(3, 40))
        F = int(rng.choice([4, 8, 12, 16, 20]))
    n = 4
    fix = np.stack([rng.uniform(0, w, n), rng.uniform(0, h, n)], axis=1)
    fix[0] = (0.0, 0.0)
    fix[1] = (w - 1.0, h - 1.0)
    strength = float(rng.uniform(0.5, 3.0))
    p = fk.FoveationParams(fragment_size=F, strength=strength, e2=float(rng.uniform(1.0, 3.0)))
    for dtype in ("u8", "f32"):
        if dtype == "u8":
            frames = torch.from_numpy(rng.integers(0, 256, (n, h, w, 3), dtype=np.uint8)).cuda()
        else:
            frames = torch.from_numpy(rng.random((n, h, w, 3), dtype=np.float32)).cuda()
        eng.set_kernel_variant(1)
        ref = fk.foveate_batch(frames, fix, p).clone()
        eng.set_kernel_variant(32)
        plain = fk.foveate_batch(frames, fix, p).clone()
        eng.set_kernel_variant(0)
        got = fk.foveate_batch(frames, fix, p)
        for name, x in (("mixed", got), ("plain", plain)):
            if not torch.equal(ref, x):
                bad += 1
                d = (ref != x)
                print("MISMATCH", name, dict(h=h, w=w, F=F, dtype=dtype, strength=strength, count=int(d.sum())),
                      d.nonzero()[:4].tolist(), flush=True)
print(f"{cases} cases, {bad} mismatches")
