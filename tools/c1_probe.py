"""One 1080p frame, centre fixation: render over a prebuilt plan, CUDA-event time per render
(BASELINE configs[0] as the bench's C1 leg measures it), for FK_STRIP_ROWS_FORCE settings.
usage: python tools/c1_probe.py [frames] [reps]"""
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_08655_b200 as fk  # noqa: E402
from paper_2012_08655_b200.engine import get_engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
H, W = 1080, 1920
eng = get_engine(0)
frames = torch.from_numpy(np.random.default_rng(0).integers(0, 256, (n, H, W, 3), dtype=np.uint8)).cuda()
out = torch.empty_like(frames)
fix = torch.from_numpy(np.tile([[W / 2.0, H / 2.0]], (n, 1))).cuda()
plan = eng.plan_for((W, H), 32, n)
plan.model(fk.FoveationParams(), fix)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
ts = []
for k in range(reps + 5):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    eng.render(frames, plan, out=out)
    b.record(s)
    torch.cuda.synchronize()
    if k >= 5:
        ts.append(a.elapsed_time(b))
print("frames %d  render median %.1f us  min %.1f us" % (n, 1e3 * statistics.median(ts), 1e3 * min(ts)))
