"""Randomised agreement soak on the GPU: random image sizes, fragment sizes, channel counts,
dtypes, fixations and strengths; the default dispatch must equal the generic kernel bit for bit
and stay within 1 LSB (uint8) / 1e-4 (float32) of the C oracle.  usage: python tools/soak.py [cases] [seed]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_08655_b200 as fk
from oracle import fovea_oracle as fo

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
eng = fk.get_engine(0)
bad = 0
for i in range(cases):
    h = int(rng.integers(33, 700)); w = int(rng.integers(33, 900))
    if rng.random() < 0.5:
        w = (w // 16) * 16 or 16          # a pitch TMA can describe for C = 1 and 3
    c = 3 if rng.random() < 0.8 else 1
    F = int(rng.choice([8, 16, 32, 64]))
    f32 = rng.random() < 0.25
    n = int(rng.integers(1, 4))
    strength = float(rng.uniform(0.3, 3.0))
    e2 = float(rng.uniform(1.0, 3.0))
    fix = np.stack([rng.uniform(0, w, n), rng.uniform(0, h, n)], axis=1)
    if rng.random() < 0.3:
        fix[0] = (0.0, 0.0) if rng.random() < 0.5 else (w - 1.0, h - 1.0)
    if f32:
        frames = torch.from_numpy(rng.random((n, h, w, c), dtype=np.float32)).cuda()
    else:
        frames = torch.from_numpy(rng.integers(0, 256, (n, h, w, c), dtype=np.uint8)).cuda()
    p = fk.FoveationParams(fragment_size=F, strength=strength, e2=e2)
    eng.set_kernel_variant(1)
    ref = fk.foveate_batch(frames, fix, p).clone()
    eng.set_kernel_variant(0)
    got = fk.foveate_batch(frames, fix, p)
    ok = torch.equal(ref, got)
    # oracle on the first frame
    img = frames[0].cpu().numpy()
    op = fo.OracleParams(fragment_size=F, strength=strength, e2=e2, fixation=(float(fix[0, 0]), float(fix[0, 1])))
    if f32:
        pl = fo.c_plan((w, h), op)
        oref = fo.c_render(img, F, pl["shift"], pl["length"], quantize=False, threads=8)
        err = np.abs(got[0].cpu().numpy() - oref).max()
        ok = ok and err <= 1e-4
    else:
        oref, _ = fo.c_foveate(img, op, threads=8)
        err = np.abs(got[0].cpu().numpy().astype(np.int16) - oref.astype(np.int16)).max()
        ok = ok and err <= 1
    if not ok:
        bad += 1
        print("MISMATCH", dict(h=h, w=w, c=c, F=F, f32=f32, n=n, strength=strength, e2=e2, fix=fix.tolist(), err=float(err)), flush=True)
print(f"{cases} cases, {bad} mismatches")
