"""Latency of one fk_request graph launch (fixation up, plan, render, frame + plan summary down)
on a resident 1920x1080 RGB image, without the streaming layer's threads: launch, synchronise,
repeat.  Also the same graph without the device->host copy of the frame.
usage: python tools/bench_request.py [requests]"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_08655_b200 as fk
from paper_2012_08655_b200.engine import DevicePlan, FrameRequest, get_engine, pinned_empty

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
img = torch.from_numpy(np.random.default_rng(0).integers(0, 256, (1080, 1920, 3), dtype=np.uint8)).cuda()
out = torch.empty_like(img)
host = pinned_empty((1080, 1920, 3), np.uint8)
eng = get_engine(0)
params = fk.FoveationParams(fragment_size=32)
i = np.arange(n)
fx = np.floor(960 + 768 * np.cos(2 * np.pi * i / 256))
fy = np.floor(540 + 432 * np.sin(2 * np.pi * i / 256))
res = {}
for name, h in (("with_d2h", host), ("device_only", None)):
    plan = DevicePlan(eng, (1920, 1080), 32, 1)
    stream = torch.cuda.Stream()
    req = FrameRequest(eng, plan, params, img, out, h, stream)
    for k in range(50):
        req.launch(fx[k], fy[k]); stream.synchronize()
    lat = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gpu = []
    for k in range(n):
        t = time.perf_counter()
        ev0.record(stream)
        req.launch(fx[k], fy[k])
        ev1.record(stream)
        stream.synchronize()
        lat.append(time.perf_counter() - t)
        gpu.append(ev0.elapsed_time(ev1))
    lat = np.sort(np.asarray(lat)) * 1e3
    res[name] = {"latency_ms_median": float(lat[n // 2]), "latency_ms_p99": float(lat[int(n * 0.99)]),
                 "gpu_ms_median": float(np.median(gpu))}
    req.close(); plan.close()
print(json.dumps({"workload": "1920x1080 RGB uint8 resident image, moving fixation, 32x32 fragments, one fk_request graph launch per frame",
                  "requests": n, **res}))
