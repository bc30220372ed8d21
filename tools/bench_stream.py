"""Closed-loop rate of the latest-wins streaming layer on one resident 1920x1080 RGB image:
submit a fixation, wait for the frame in pinned host memory, repeat (the paper's end-to-end
figure: 165 Hz on a GTX 1060 including host<->device transfers).
usage: python tools/bench_stream.py [frames]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2012_08655_b200 as fk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
img = np.random.default_rng(0).integers(0, 256, (1080, 1920, 3), dtype=np.uint8)
i = np.arange(n)
fx = np.floor(960 + 768 * np.cos(2 * np.pi * i / 256))
fy = np.floor(540 + 432 * np.sin(2 * np.pi * i / 256))
with fk.FoveationStream(img, fk.FoveationParams(fragment_size=32)) as s:
    for k in range(50):                       # warm-up
        s.submit(fx[k], fy[k]); s.get(timeout=60)
    lat = []
    t0 = time.perf_counter()
    for k in range(n):
        t1 = time.perf_counter()
        s.submit(fx[k], fy[k])
        out, stats = s.get(timeout=60)
        lat.append(time.perf_counter() - t1)
    dt = time.perf_counter() - t0
lat = np.sort(np.asarray(lat)) * 1e3
print(json.dumps({"workload": "1920x1080 RGB uint8 resident image, moving fixation, 32x32 fragments, "
                              "one frame per request, result in pinned host memory",
                  "frames": n, "frames_per_s": n / dt, "latency_ms_median": float(lat[n // 2]),
                  "latency_ms_p99": float(lat[int(n * 0.99)]),
                  "d2h_bytes_per_frame": int(img.nbytes), "h2d_bytes_per_frame": 16,
                  "paper_gtx1060_end_to_end_fps": 165}))
