"""float32 frames: default dispatch (fk_blur_tma<float>, TMA quads) against the generic kernel,
bit for bit, on geometries that exercise every border case of the shifted quad grid.
usage: python tools/f32_check.py [cases] [seed]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_08655_b200 as fk

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
eng = fk.get_engine(0)
bad = 0
fixed = [(64, 64, 32), (40, 36, 8), (96, 160, 16), (270, 480, 32), (33, 44, 64), (256, 256, 32),
         (1080, 1920, 32), (1080, 1920, 8), (540, 960, 64)]
for i in range(cases):
    if i < len(fixed):
        h, w, F = fixed[i]
    else:
        h = int(rng.integers(33, 500)); w = 4 * int(rng.integers(9, 200))
        F = int(rng.choice([8, 16, 32, 64]))
    n = 4
    fix = np.stack([rng.uniform(0, w, n), rng.uniform(0, h, n)], axis=1)
    fix[0] = (0.0, 0.0)
    fix[1] = (w - 1.0, h - 1.0)
    fix[2] = (w - 1.0, 0.0)
    strength = float(rng.uniform(0.5, 2.5))
    frames = torch.from_numpy(rng.random((n, h, w, 3), dtype=np.float32)).cuda()
    p = fk.FoveationParams(fragment_size=F, strength=strength, e2=float(rng.uniform(1.0, 3.0)))
    eng.set_kernel_variant(1)
    ref = fk.foveate_batch(frames, fix, p).clone()
    eng.set_kernel_variant(0)
    got = fk.foveate_batch(frames, fix, p)
    if not torch.equal(ref, got):
        bad += 1
        d = (ref != got)
        idx = d.nonzero()[:5].tolist()
        print("MISMATCH", dict(h=h, w=w, F=F, strength=strength, count=int(d.sum())), idx, flush=True)
print(f"{cases} cases, {bad} mismatches")
