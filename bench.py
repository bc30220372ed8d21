"""Benchmark of the blockwise foveation hot path (BASELINE.json metric).

    python bench.py --gpus N --steps K --warmup W            # this repo's CUDA path
    python bench.py --impl reference --gpus N --steps K ...  # reference CPU arithmetic

Workload (BASELINE.json configs[1]): a batch of 256 synthetic 1920x1080 RGB uint8 frames
with a per-frame moving fixation, 32x32 fragments, default CSF parameters.  A "step" is one
pass of plan -> render over the batch.  With N > 1 (torchrun, one rank per GPU) every rank
owns its own 256-frame batch -- frames are independent, there is no collective on the data
path -- so scaling is weak and `value` is the whole-job frames/s.

Prints ONE JSON line on rank 0.  `value` is device-resident throughput (CUDA events, max
over ranks); `e2e` is the same metric through the public host API (pinned host frames in,
pinned host frames out, copies inside the timed region); `roofline` describes the blur
kernel; `cpu_baseline` is the CPU oracle timed on this host (N = 1 only).
"""

from __future__ import annotations

import argparse
import json
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


def moving_fixations(n, w=1920, h=1080):
    """fx = floor(960 + 768 cos(2 pi i / n)), fy = floor(540 + 432 sin)
    (scaled with the frame size for the exploration workloads)."""
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

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.dev, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.dev)
                for name, bit in {**self.BAD, **self.NOTED}.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.05)

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
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "frames_per_step": cores, "fragment_size": F},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------ GPU arm
def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2012_08655_b200 as fk
    from paper_2012_08655_b200 import costs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    global W, H, F
    W, H, F = args.width, args.height, args.fragment
    explore = (W, H, F, args.dtype, args.e2, args.variant) != (1920, 1080, 32, "u8", 2.3, 0)
    eng = fk.get_engine(local)
    if args.variant:
        eng.set_kernel_variant(args.variant)
    params = fk.FoveationParams(fragment_size=F, e2=args.e2)
    n = args.frames
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    if args.dtype == "u8":
        frames = torch.randint(0, 256, (n, H, W, C), dtype=torch.uint8, device="cuda", generator=gen)
    else:
        frames = torch.rand((n, H, W, C), dtype=torch.float32, device="cuda", generator=gen)
    out = torch.empty_like(frames)
    fixes = moving_fixations(n, W, H)
    if args.fixation == "centre":       # exploration only; the reported workload is "moving"
        fixes[:] = (W / 2.0, H / 2.0)
    elif args.fixation == "corner":
        fixes[:] = (0.0, 0.0)
    fix_dev = fixes if args.fix_host else torch.from_numpy(fixes).cuda()
    plan = eng.plan_for((W, H), F, n)
    stream = torch.cuda.current_stream()

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
    value = world * n * args.steps / (total_ms * 1e-3)

    # roofline of the blur kernel: algorithmic FLOPs of this batch's plans / its duration
    lengths, meta = plan.read_lengths()
    flops = costs.batch_flops((W, H), F, C, lengths, meta)
    bytes_alg = n * costs.frame_bytes((W, H), C, frames.element_size())
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    clock_khz = eng.info["clock_khz"]
    fp32_nominal = 2.0 * eng.info["sm_count"] * 128 * clock_khz * 1e3 / 1e12
    probe_tf, _ = eng.measure_fp32_peak()
    achieved_tf = flops / (blur_ms * 1e-3) / 1e12
    achieved_gbs = bytes_alg / (blur_ms * 1e-3) / 1e9
    t_fp32 = flops / (fp32_nominal * 1e12)
    t_hbm = bytes_alg / (hbm_peak * 1e9)
    traffic = None
    try:  # ncu dram__bytes_read.sum + dram__bytes_write.sum of the render launches, per frame
        per_frame = json.loads((ROOT / "profiles" / "traffic.json").read_text()).get(
            "dram_bytes_per_frame")
        traffic = per_frame * n if per_frame else None
    except Exception:
        pass
    roofline = {
        "bound": "fp32" if t_fp32 >= t_hbm else "hbm",
        "kernel": (("fk_blur_bytes" if args.dtype == "u8" else "fk_blur_cols") +
                   " (render of the whole batch: one persistent launch per tap-count class, up "
                   "to 5 per step, side by side on forked streams; timed together)"),
        "achieved": achieved_tf, "peak": fp32_nominal, "unit": "TFLOP/s",
        "frac": achieved_tf / fp32_nominal,
        "peak_source": (f"nominal FP32 = 2 x {eng.info['sm_count']} SMs x 128 lanes x "
                        f"{clock_khz / 1e6:.3f} GHz (BASELINE.md s3; MEASURED_PEAKS.json has no "
                        "FP32 entry)"),
        "ffma_probe_tflops": probe_tf, "frac_of_ffma_probe": achieved_tf / probe_tf,
        "flops_per_launch": flops, "kernel_ms": blur_ms, "plan_kernel_ms": plan_ms,
        "hbm": {"achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved_gbs / hbm_peak, "bytes_per_launch": bytes_alg,
                "peak_source": hbm_src},
        "roofline_ms_per_launch": max(t_fp32, t_hbm) * 1e3,
        "traffic": traffic,
    }

    # end to end: pinned host frames -> public API -> pinned host frames
    e2e_n = args.e2e_frames
    e2e_n = min(e2e_n, n)
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
    e2e_value = world * e2e_n * args.e2e_steps / e2e_s
    same = bool(torch.equal(torch.from_numpy(h_out).cuda(), out[:e2e_n]))
    e2e = {"value": e2e_value, "unit": "frames/s",
           "h2d_bytes_per_step": int(h_in.nbytes + fix_host.nbytes),
           "d2h_bytes_per_step": int(h_out.nbytes), "frames_per_step": e2e_n,
           "steps": args.e2e_steps, "ms_per_step": 1000.0 * e2e_s / args.e2e_steps,
           "api": "paper_2012_08655_b200.foveate_batch(numpy pinned) -> fk_foveate_host_u8",
           "matches_device_path": same}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not explore:
        del h_in, h_out
        cpu = cpu_baseline_leg(fixes)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD if not explore else
                       f"exploration: {n} x {W}x{H} RGB {args.dtype} frames, moving fixation, "
                       f"{F}x{F} fragments, e2={args.e2}",
                       "frames_per_gpu": n, "fragment_size": F,
                       "l2_policy": "inputs larger than L2 (1.59 GB in + 1.59 GB out per step)",
                       "step": "fk_plan_model + fk_render_u8 over the whole batch"},
            "clocks": clocks.summary(), "e2e": e2e, "gpu_launches": int(launches),
            "roofline": roofline, "cpu_baseline": cpu,
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
    ap.add_argument("--frames", type=int, default=BATCH, help="frames per GPU per step")
    ap.add_argument("--e2e-frames", type=int, default=BATCH)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
