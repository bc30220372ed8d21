"""Benchmark of the blockwise foveation hot path (BASELINE.json metric).

    python bench.py --gpus N --steps K --warmup W            # this repo's CUDA path
    python bench.py --impl reference --gpus N --steps K ...  # reference CPU arithmetic

Headline workload (BASELINE.json configs[1]): ONE batch of 256 synthetic 1920x1080 RGB uint8
frames with a per-frame moving fixation, 32x32 fragments, default CSF parameters.  A "step" is
one pass of plan -> render over the batch.  With N > 1 (torchrun, one rank per GPU) the batch
is split contiguously, 256 / N frames per rank (strong scaling; frames are
independent, there is no collective on the data path); `--scaling weak` gives every rank its
own 256 frames instead.  `value` is the whole-job frames/s.

Prints ONE JSON line on rank 0.  `value` is device-resident throughput (CUDA events, max over
ranks); `e2e` is the same metric through the public host API (pinned host frames in, pinned
host frames out, copies inside the timed region); `roofline` describes the blur kernel
(algorithmic and executed FLOPs); `cpu_baseline` is the CPU oracle timed on this host (N = 1
only); `configs` holds one bounded measurement per other BASELINE config at its named shape
(C1 single frame, C3 3840x2160 / 16x16, C4 65 536 x 256x256, C5 float32 block-size sweep), same
timing rules, so that every roofline fraction can be read from this one line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

W, H, C, F = 1920, 1080, 3, 32   # BASELINE configs[1]; --width/--height/--fragment explore others
BATCH = 256
METRIC = "foveated frames/sec at 1920x1080 RGB"
WORKLOAD = ("batch of 256 synthetic 1920x1080 RGB uint8 frames, per-frame moving fixation, "
            "32x32 fragments (BASELINE configs[1])")
L2_POLICY = "inputs larger than L2 (1.59 GB in + 1.59 GB out per step)"


def headline_config(n_gpus=1, scaling="strong"):
    """The `config` object both arms print (the reference arm times a bounded sample of it)."""
    cfg = {"workload": WORKLOAD, "frames_per_step": BATCH, "fragment_size": F,
           "l2_policy": L2_POLICY, "step": "plan + render over the whole batch"}
    if n_gpus > 1:
        cfg["frames_per_gpu"] = BATCH // n_gpus if scaling == "strong" else BATCH
        cfg["frames_per_step"] = BATCH if scaling == "strong" else BATCH * n_gpus
    return cfg


def moving_fixations(n, w=1920, h=1080):
    """fx = floor(960 + 768 cos(2 pi i / n)), fy = floor(540 + 432 sin)
    (scaled with the frame size for the other workloads)."""
    import numpy as np

    i = np.arange(n, dtype=np.float64)
    fx = np.floor(w / 2 + 0.4 * w * np.cos(2 * np.pi * i / n))
    fy = np.floor(h / 2 + 0.4 * h * np.sin(2 * np.pi * i / n))
    return np.ascontiguousarray(np.stack([fx, fy], axis=1))


# ------------------------------------------------------------------ clock sampling
class ClockSampler:
    """Samples SM clock and throttle reasons of one GPU while the timed region runs."""

    BAD = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20}
    NOTED = {"sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            # NVML enumerates physical devices; honour CUDA_VISIBLE_DEVICES when it is a list
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = index
            if vis:
                try:
                    phys = int(vis.split(",")[index])
                except (ValueError, IndexError):
                    phys = index
            self.dev = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.dev, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def sample(self):
        nv = self.nv
        if nv is None:
            return
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.dev, nv.NVML_CLOCK_SM))
            mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.dev)
            for name, bit in {**self.BAD, **self.NOTED}.items():
                if mask & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            self._stop.wait(0.02)

    def __enter__(self):
        if self.nv is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------- CPU baseline
def _cpu_numpy_frame(args):
    """One frame through the numpy restatement of blockwise.render (plan excluded,
    foveakit bench.py:80-85 convention).  Runs in a worker process."""
    seed, fix = args
    import numpy as np

    from oracle import fovea_oracle as fo

    img = np.random.default_rng(seed).integers(0, 256, (H, W, C), dtype=np.uint8)
    pl = fo.np_plan((W, H), fo.OracleParams(fragment_size=F, fixation=(float(fix[0]), float(fix[1]))))
    t0 = time.perf_counter()
    fo.np_render(img, F, pl["shift"], pl["length"])
    return time.perf_counter() - t0


def cpu_numpy_step(pool, cores, fixes, step):
    """One bounded step: `cores` frames, one per worker process.  Returns (frames, seconds)."""
    jobs = [(1000 * step + i, fixes[(step * cores + i) % len(fixes)]) for i in range(cores)]
    t0 = time.perf_counter()
    pool.map(_cpu_numpy_frame, jobs)
    return cores, time.perf_counter() - t0


def make_pool(cores):
    import multiprocessing as mp

    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    return mp.get_context("fork").Pool(cores)


def cpu_baseline_leg(fixes):
    """Bounded CPU baseline for the default arm: numpy port (the reference's arithmetic and
    speed) plus the C/OpenMP port, both on all host cores."""
    import numpy as np

    from oracle import fovea_oracle as fo

    cores = os.cpu_count() or 1
    with make_pool(cores) as pool:
        cpu_numpy_step(pool, cores, fixes, 0)              # warm-up (imports, page-in)
        n, sec = cpu_numpy_step(pool, cores, fixes, 1)
    numpy_fps = n / sec
    # C port: a few frames, OpenMP over fragments on all cores
    os.environ["OMP_NUM_THREADS"] = str(cores)
    img = np.random.default_rng(0).integers(0, 256, (H, W, C), dtype=np.uint8)
    pls = [fo.c_plan((W, H), fo.OracleParams(fragment_size=F, fixation=tuple(fixes[i * 32])))
           for i in range(4)]
    fo.c_render(img, F, pls[0]["shift"], pls[0]["length"], threads=cores)
    t0 = time.perf_counter()
    for pl in pls:
        fo.c_render(img, F, pl["shift"], pl["length"], threads=cores)
    c_fps = len(pls) / (time.perf_counter() - t0)
    return {"value": numpy_fps, "unit": "frames/s", "cores": cores, "kind": "port",
            "sample": (f"{n} of the workload's frames (1080p RGB, moving fixation), numpy "
                       "restatement of foveakit.blockwise.render over a prebuilt plan, one frame "
                       "per process on all cores"),
            "c_port": {"value": c_fps, "unit": "frames/s", "cores": cores,
                       "sample": "4 frames, fp64 C loops, OpenMP over fragments"}}


def run_reference(args):
    """--impl reference: the reference's CPU arithmetic (numpy port) on all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    fixes = moving_fixations(BATCH)
    cores = os.cpu_count() or 1
    frames, seconds = 0, 0.0
    with make_pool(cores) as pool:
        for s in range(args.warmup):
            cpu_numpy_step(pool, cores, fixes, s)
        for s in range(args.steps):
            n, sec = cpu_numpy_step(pool, cores, fixes, args.warmup + s)
            frames += n
            seconds += sec
    fps = frames / seconds
    sample = (f"each step = {cores} frames of the workload (one per process, {cores} cores), "
              "numpy restatement of foveakit.blockwise.render over a prebuilt plan")
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * seconds / max(args.steps, 1), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": headline_config(args.gpus, args.scaling),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------ GPU arm
class Bench:
    """Device-resident measurement of plan -> render on one GPU (CUDA events on the launching
    stream), with the roofline bookkeeping of SURVEY.md 8(d)."""

    def __init__(self, eng, local):
        import json as _json

        self.eng, self.local = eng, local
        peaks = {}
        try:
            peaks = _json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        except Exception:
            pass
        self.hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        self.hbm_src = ("measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks
                        else "fallback 6650 GB/s")
        self.clock_khz = eng.info["clock_khz"]
        self.fp32_nominal = 2.0 * eng.info["sm_count"] * 128 * self.clock_khz * 1e3 / 1e12
        self.probe_tf = None
        self._flush = None

    def flush_l2(self):
        import torch

        if self._flush is None:
            self._flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        self._flush.fill_(1)

    def measure(self, frames, fixes, params, steps, warmup, out=None, replan=True,
                flush=False, min_ms=0.0):
        """Times `steps` passes.  replan=False: the plan is built once and only the render
        is repeated (foveakit bench.py:80-85 convention for a single image); flush=True:
        L2 is overwritten between passes (inputs smaller than L2)."""
        import numpy as np
        import torch

        from paper_2012_08655_b200 import costs

        eng = self.eng
        n, h, w, c = frames.shape
        Fs = params.fragment_size
        if out is None:
            out = torch.empty_like(frames)
        fix_dev = torch.from_numpy(np.ascontiguousarray(fixes)).cuda()
        plan = eng.plan_for((w, h), Fs, n)
        stream = torch.cuda.current_stream()
        plan.model(params, fix_dev)

        def one(e0=None, e1=None, e2=None):
            if flush:
                self.flush_l2()
            if e0 is not None:
                e0.record(stream)
            if replan:
                plan.model(params, fix_dev)
            if e1 is not None:
                e1.record(stream)
            eng.render(frames, plan, out=out)
            if e2 is not None:
                e2.record(stream)

        for _ in range(max(warmup, 1)):
            one()
        if min_ms > 0:  # short steps: enough of them for the clock sampler to see the load
            a, b = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            a.record(stream)
            one()
            b.record(stream)
            torch.cuda.synchronize()
            est = max(a.elapsed_time(b), 1e-3)
            steps = int(min(max(steps, math.ceil(min_ms / est)), 400))
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        launches0 = eng.launch_count()
        torch.cuda.synchronize()
        with ClockSampler(self.local) as clocks:
            for k in range(steps):
                one(*ev[k])
            torch.cuda.synchronize()
            clocks.sample()
        launches = eng.launch_count() - launches0
        blur_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ev)
        plan_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
        if flush:   # the flush sits before e0: a step is plan + render
            total_ms = sum(e[0].elapsed_time(e[2]) for e in ev)
        else:
            total_ms = ev[0][0].elapsed_time(ev[-1][2])
        lengths, meta = plan.read_lengths()
        flops = costs.batch_flops((w, h), Fs, c, lengths, meta)
        executed = costs.executed_flops(plan.read_items()[:-1], c)
        bytes_alg = n * costs.frame_bytes((w, h), c, frames.element_size())
        return dict(out=out, plan=plan, steps=steps, launches=int(launches), total_ms=total_ms,
                    ms_per_step=total_ms / steps, blur_ms=blur_ms, plan_ms=plan_ms, flops=flops,
                    executed=executed, bytes=bytes_alg, clocks=clocks.summary(),
                    max_taps=int(meta[:, 6].max()))

    def roofline(self, m, kernel):
        achieved_tf = m["flops"] / (m["blur_ms"] * 1e-3) / 1e12
        achieved_gbs = m["bytes"] / (m["blur_ms"] * 1e-3) / 1e9
        t_fp32 = m["flops"] / (self.fp32_nominal * 1e12)
        t_hbm = m["bytes"] / (self.hbm_peak * 1e9)
        r = {
            "bound": "fp32" if t_fp32 >= t_hbm else "hbm", "kernel": kernel,
            "achieved": achieved_tf, "peak": self.fp32_nominal, "unit": "TFLOP/s",
            "frac": achieved_tf / self.fp32_nominal,
            "flops_per_launch": m["flops"], "executed_flops": m["executed"],
            "executed_over_algorithmic": m["executed"] / m["flops"] if m["flops"] else None,
            "executed_tflops": m["executed"] / (m["blur_ms"] * 1e-3) / 1e12,
            "kernel_ms": m["blur_ms"], "plan_kernel_ms": m["plan_ms"],
            "hbm": {"achieved": achieved_gbs, "peak": self.hbm_peak, "unit": "GB/s",
                    "frac": achieved_gbs / self.hbm_peak, "bytes_per_launch": m["bytes"],
                    "peak_source": self.hbm_src},
            "roofline_ms_per_launch": max(t_fp32, t_hbm) * 1e3,
        }
        if self.probe_tf:
            r["ffma_probe_tflops"] = self.probe_tf
            r["frac_of_ffma_probe"] = achieved_tf / self.probe_tf
        return r

    def leg(self, name, workload, frames, fixes, params, steps, warmup, **kw):
        """One entry of `configs`: a bounded measurement of another BASELINE config."""
        m = self.measure(frames, fixes, params, steps, warmup, min_ms=150.0, **kw)
        n = frames.shape[0]
        r = self.roofline(m, "")
        entry = {
            "name": name, "workload": workload, "frames": int(n), "steps": m["steps"],
            "value": n * m["steps"] / (m["total_ms"] * 1e-3), "unit": "frames/s",
            "ms_per_step": m["ms_per_step"], "kernel_ms": m["blur_ms"],
            "dtype": "u8" if frames.element_size() == 1 else "f32", "max_taps": m["max_taps"],
            "roofline": {k: r[k] for k in ("bound", "achieved", "peak", "unit", "frac",
                                           "flops_per_launch", "executed_flops",
                                           "executed_over_algorithmic", "executed_tflops")},
            "hbm_frac": r["hbm"]["frac"], "clocks": m["clocks"],
            "l2_policy": ("L2 overwritten between passes (256 MB fill)" if kw.get("flush") else
                          "inputs larger than L2"),
        }
        return entry, m


def config_legs(bench, args, rank, world):
    """Bounded measurements of the other BASELINE configs at their named shapes."""
    import numpy as np
    import torch

    import paper_2012_08655_b200 as fk

    legs = []
    W5, H5 = 1920, 1080

    def rand_u8(shape, seed):
        g = torch.Generator(device="cuda").manual_seed(seed)
        return torch.randint(0, 256, shape, dtype=torch.uint8, device="cuda", generator=g)

    def rand_f32(shape, seed):
        g = torch.Generator(device="cuda").manual_seed(seed)
        return torch.rand(shape, dtype=torch.float32, device="cuda", generator=g)

    def done():
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    if world == 1:
        # C1: one 1080p frame, centre fixation; `render` over a prebuilt plan
        # (foveakit bench.py:80-85), L2 overwritten between passes
        fr = rand_u8((1, H5, W5, 3), 11)
        e, _ = bench.leg("C1", "single 1920x1080 RGB uint8 image, centre fixation, 32x32 fragments; "
                         "render over a prebuilt plan (foveakit bench.py:80-85)", fr,
                         np.asarray([[W5 / 2.0, H5 / 2.0]]), fk.FoveationParams(), 20, 5,
                         replan=False, flush=True)
        # the call a foveakit user makes: host image in, host image out
        img = fk.RasterImage.from_array(fr[0].cpu().numpy())
        grid, bank = fk.plan(img.size, fk.FoveationParams())
        for _ in range(3):
            fk.render(img, grid, bank)
        t0 = time.perf_counter()
        for _ in range(10):
            fk.render(img, grid, bank)
        e["e2e_value"] = 10 / (time.perf_counter() - t0)
        e["e2e_api"] = "paper_2012_08655_b200.render(RasterImage, grid, bank) -- host image in and out"
        # the streaming request (fk_request_*): the image stays in HBM, one graph launch takes a
        # fixation and returns the frame and its plan summary in pinned host memory
        from paper_2012_08655_b200.engine import DevicePlan, FrameRequest, get_engine, pinned_empty
        host = pinned_empty((H5, W5, 3), np.uint8)
        rplan = DevicePlan(get_engine(torch.cuda.current_device()), (W5, H5), 32, 1)
        rstream = torch.cuda.Stream()
        rout = torch.empty_like(fr[0])
        req = FrameRequest(rplan.engine, rplan, fk.FoveationParams(), fr[0], rout, host, rstream)
        lat = []
        for k in range(60):
            t0 = time.perf_counter()
            req.launch(W5 / 2.0 + 3 * (k % 7), H5 / 2.0)
            rstream.synchronize()
            lat.append(time.perf_counter() - t0)
        req.close()
        rplan.close()
        e["request_ms_median"] = float(np.median(lat[10:]) * 1e3)
        e["request_api"] = ("FrameRequest.launch(x, y) + stream sync: fixation up, plan, render, "
                            "frame + plan summary down to pinned host memory, one CUDA graph")
        legs.append(e)
        del rout, host
        del fr
        done()
        # the per-GPU share of the headline batch at 8 GPUs, on this one GPU
        fr = rand_u8((32, H5, W5, 3), 12)
        e, _ = bench.leg("C2/8", "32 of the headline batch's frames (256 / 8: the per-GPU share of the "
                         "strong-scaling split at 8 GPUs), moving fixation, 32x32 fragments", fr,
                         moving_fixations(256)[::8].copy(), fk.FoveationParams(), 10, 3)
        legs.append(e)
        del fr
        done()
        # C3: 3840x2160, 16x16 fragments, centre and corner fixation
        fr = rand_u8((16, 2160, 3840, 3), 13)
        for fx, label in (((1920.0, 1080.0), "centre"), ((0.0, 0.0), "corner (0, 0)")):
            e, _ = bench.leg(f"C3 {label.split()[0]}", f"16 x 3840x2160 RGB uint8 frames, 16x16 fragments, "
                             f"{label} fixation", fr, np.tile(np.asarray([fx]), (16, 1)),
                             fk.FoveationParams(fragment_size=16), 5, 3)
            legs.append(e)
        del fr
        done()
    # C4: 65 536 x 256x256, random fixations (seed 1), 32x32 fragments; N / g frames per GPU
    n4 = args.c4_frames
    a, b = fk.shard_range(n4, rank, world)
    rng = np.random.default_rng(1)
    fix4 = np.stack([rng.integers(0, 256, n4), rng.integers(0, 256, n4)], axis=1).astype(np.float64)
    fr = rand_u8((b - a, 256, 256, 3), 14 + rank)
    e, _ = bench.leg("C4", f"RL-style batch of {n4} synthetic 256x256 RGB uint8 frames, random "
                     f"fixations, 32x32 fragments ({b - a} frames on this GPU of {world})", fr,
                     fix4[a:b], fk.FoveationParams(), 3, 3)
    legs.append(e)
    del fr
    done()
    if world == 1:
        # C5: float32 1080p frames, centre fixation, block sizes 8..64, default and steeper fit
        fr = rand_f32((args.c5_frames, H5, W5, 3), 15)
        out = torch.empty_like(fr)
        fix5 = np.tile(np.asarray([[W5 / 2.0, H5 / 2.0]]), (fr.shape[0], 1))
        for e2 in (2.3, 1.5):
            for Fs in (8, 16, 32, 64):
                e, _ = bench.leg(f"C5 F={Fs} e2={e2}", f"{fr.shape[0]} x 1920x1080 RGB float32 frames, "
                                 f"{Fs}x{Fs} fragments, centre fixation, CSF fit e2={e2}"
                                 + (" (steeper sigma-vs-eccentricity)" if e2 != 2.3 else " (default)"),
                                 fr, fix5, fk.FoveationParams(fragment_size=Fs, e2=e2), 5, 3, out=out)
                legs.append(e)
        del fr, out
        done()
    return legs


def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2012_08655_b200 as fk

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # FK_BENCH_ONE_GPU=1 (dry runs of the multi-rank path on a one-GPU box): every rank on
    # cuda:0, rendezvous and reductions over gloo -- the numbers of such a run mean nothing
    one_gpu = world > 1 and os.environ.get("FK_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    red_dev = "cpu" if one_gpu else "cuda"
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    global W, H, F
    W, H, F = args.width, args.height, args.fragment
    explore = (W, H, F, args.dtype, args.e2, args.variant, args.fixation, args.frames) != \
        (1920, 1080, 32, "u8", 2.3, 0, "moving", BATCH)
    eng = fk.get_engine(local)
    if args.variant:
        eng.set_kernel_variant(args.variant)
    params = fk.FoveationParams(fragment_size=F, e2=args.e2)
    total = args.frames * (world if args.scaling == "weak" else 1)
    first, last = fk.shard_range(total, rank, world)      # this rank's slice of the job
    n = last - first
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    if args.dtype == "u8":
        frames = torch.randint(0, 256, (n, H, W, C), dtype=torch.uint8, device="cuda", generator=gen)
    else:
        frames = torch.rand((n, H, W, C), dtype=torch.float32, device="cuda", generator=gen)
    out = torch.empty_like(frames)
    fixes_all = moving_fixations(total, W, H)
    if args.fixation == "centre":       # exploration only; the reported workload is "moving"
        fixes_all[:] = (W / 2.0, H / 2.0)
    elif args.fixation == "corner":
        fixes_all[:] = (0.0, 0.0)
    fixes = np.ascontiguousarray(fixes_all[first:last])
    fix_dev = fixes if args.fix_host else torch.from_numpy(fixes).cuda()
    plan = eng.plan_for((W, H), F, n)
    stream = torch.cuda.current_stream()
    bench = Bench(eng, local)

    def step():
        plan.model(params, fix_dev)
        eng.render(frames, plan, out=out)

    for _ in range(args.warmup):
        step()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    launches0 = eng.launch_count()
    barrier()
    with ClockSampler(local) as clocks:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for k in range(args.steps):
            ev[k][0].record(stream)
            plan.model(params, fix_dev)
            ev[k][1].record(stream)
            eng.render(frames, plan, out=out)
            ev[k][2].record(stream)
        t_end.record(stream)
        barrier()
    launches = eng.launch_count() - launches0
    total_ms = max_over_ranks(t_start.elapsed_time(t_end))
    blur_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ev)
    plan_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    ms_per_step = total_ms / args.steps
    value = total * args.steps / (total_ms * 1e-3)

    # roofline of the blur kernel: algorithmic FLOPs of this rank's plans / its duration
    from paper_2012_08655_b200 import costs

    lengths, meta = plan.read_lengths()
    m = dict(flops=costs.batch_flops((W, H), F, C, lengths, meta),
             executed=costs.executed_flops(plan.read_items()[:-1], C),
             bytes=n * costs.frame_bytes((W, H), C, frames.element_size()),
             blur_ms=blur_ms, plan_ms=plan_ms)
    bench.probe_tf, _ = eng.measure_fp32_peak()
    kernel = ("fk_blur_tma<" + ("uint8" if args.dtype == "u8" else "float") + "> (render of the "
              "batch: one persistent launch per tap-count class, up to 5 per step, side by side on "
              "forked streams; timed together)")
    roofline = bench.roofline(m, kernel)
    roofline["peak_source"] = (f"nominal FP32 = 2 x {eng.info['sm_count']} SMs x 128 lanes x "
                               f"{bench.clock_khz / 1e6:.3f} GHz (BASELINE.md s3; "
                               "MEASURED_PEAKS.json has no FP32 entry); ffma_probe_tflops is the "
                               "FFMA loop measured in this run")
    roofline["traffic"] = None
    try:  # ncu dram__bytes_read.sum + dram__bytes_write.sum of the render launches
        tr = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        if not explore and world == 1:
            roofline["traffic"] = tr["dram_bytes_per_frame"] * n
            roofline["traffic_source"] = ("static: " + tr.get("source", "profiles/traffic.json") +
                                          " (ncu capture of this workload, not measured in this run)")
    except Exception:
        pass

    # end to end: pinned host frames -> public API -> pinned host frames
    e2e_n = min(args.e2e_frames, n)
    np_dtype = np.uint8 if args.dtype == "u8" else np.float32
    h_in = fk.pinned_empty((e2e_n, H, W, C), np_dtype)
    h_out = fk.pinned_empty((e2e_n, H, W, C), np_dtype)
    h_in[...] = frames[:e2e_n].cpu().numpy()
    fix_host = fixes[:e2e_n]
    for _ in range(max(1, min(args.warmup, 3))):
        fk.foveate_batch(h_in, fix_host, params, out=h_out, devices=[local])
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        fk.foveate_batch(h_in, fix_host, params, out=h_out, devices=[local])
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e_frames_all = sum_over_ranks(float(e2e_n))
    e2e_value = e2e_frames_all * args.e2e_steps / e2e_s
    same = bool(torch.equal(torch.from_numpy(h_out).cuda(), out[:e2e_n]))
    e2e = {"value": e2e_value, "unit": "frames/s",
           "h2d_bytes_per_step": int(h_in.nbytes + fix_host.nbytes),
           "d2h_bytes_per_step": int(h_out.nbytes), "frames_per_step": int(e2e_frames_all),
           "steps": args.e2e_steps, "ms_per_step": 1000.0 * e2e_s / args.e2e_steps,
           "api": "paper_2012_08655_b200.foveate_batch(numpy pinned) -> fk_foveate_host_"
                  + ("u8" if args.dtype == "u8" else "f32"),
           "matches_device_path": same}
    del h_in, h_out

    legs = None
    if not explore and not args.no_configs:
        del frames, out
        torch.cuda.empty_cache()
        legs = config_legs(bench, args, rank, world)
        if world > 1:   # C4 is sharded: whole-job value = sum of the ranks' frames / slowest rank
            for e in legs:
                ms = max_over_ranks(e["ms_per_step"])
                e["value"] = args.c4_frames / (ms * 1e-3)
                e["ms_per_step"] = ms
                e["n_gpus"] = world

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not explore:
        cpu = cpu_baseline_leg(moving_fixations(BATCH))

    if rank == 0:
        if explore:
            config = {"workload": f"exploration: {n} x {W}x{H} RGB {args.dtype} frames, "
                                  f"{args.fixation} fixation, {F}x{F} fragments, e2={args.e2}",
                      "frames_per_step": total, "fragment_size": F, "l2_policy": "inputs larger than L2"}
        else:
            config = headline_config(world, args.scaling)
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": args.scaling if world > 1 else "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
            "clocks": clocks.summary(), "e2e": e2e, "gpu_launches": int(launches),
            "roofline": roofline, "cpu_baseline": cpu, "configs": legs,
            "paper_gtx1060": {"kernel_only_fps": 606, "end_to_end_fps": 165},
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: split the 256-frame batch over the ranks (default) or give "
                         "every rank its own 256 frames")
    ap.add_argument("--frames", type=int, default=BATCH, help="frames per step (whole job)")
    ap.add_argument("--e2e-frames", type=int, default=BATCH)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the bounded measurements of the other BASELINE configs")
    ap.add_argument("--c4-frames", type=int, default=65536)
    ap.add_argument("--c5-frames", type=int, default=64)
    ap.add_argument("--fixation", default="moving", choices=["moving", "centre", "corner"],
                    help="exploration only; BASELINE configs[1] is 'moving'")
    ap.add_argument("--width", type=int, default=1920, help="exploration only")
    ap.add_argument("--height", type=int, default=1080, help="exploration only")
    ap.add_argument("--fragment", type=int, default=32, help="exploration only")
    ap.add_argument("--dtype", default="u8", choices=["u8", "f32"], help="exploration only")
    ap.add_argument("--e2", type=float, default=2.3, help="exploration only (CSF fit)")
    ap.add_argument("--variant", type=int, default=0,
                    help="exploration only: fk_set_kernel_variant (0 = default kernels)")
    ap.add_argument("--fix-host", action="store_true",
                    help="exploration only: pass fixations from host memory each step")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
