"""Repeatability / agreement stress: many 1080p frames with random fixations through the default
dispatch (fk_blur_tma, class launches side by side), fk_blur_cols everywhere (variant 4), the
generic kernel (variant 1, first round) and the default kernels launched one class after the
other (variant 16); all runs must be bit-identical.  usage: python tools/stress_variants.py [frames] [rounds]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_08655_b200 as fk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 5
rng = np.random.default_rng(99)
frames = torch.from_numpy(rng.integers(0, 256, (n, 1080, 1920, 3), dtype=np.uint8)).cuda()
eng = fk.get_engine(0)
bad = 0
for r in range(rounds):
    fix = np.stack([rng.uniform(0, 1920, n), rng.uniform(0, 1080, n)], axis=1)
    p = fk.FoveationParams(strength=float(rng.uniform(0.6, 1.4)))
    outs = {}
    for v in (4, 0, 16, 0) + ((1,) if r == 0 else ()):
        eng.set_kernel_variant(v)
        o = fk.foveate_batch(frames, fix, p)
        if v in outs:
            bad += int(not torch.equal(outs[v], o))
        outs[v] = o.clone()
    eng.set_kernel_variant(0)
    bad += sum(int(not torch.equal(outs[v], outs[0])) for v in outs if v != 0)
    print("round", r, "mismatches so far", bad, flush=True)
print("OK" if bad == 0 else "FAILED")
