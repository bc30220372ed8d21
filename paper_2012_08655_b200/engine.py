"""Per-GPU engine: owns a libfovea handle, caches device plans, and runs the batch path.

This is the layer between the reference-shaped Python API (blockwise.py, retinal.py,
filters.py in this package) and the C ABI.  PyTorch is used only for device memory and
stream handles; all arithmetic happens in the CUDA kernels of csrc/.
"""

from __future__ import annotations

import ctypes as C
import math
import threading
import weakref

import numpy as np
import torch

from . import _native
from ._native import FkParams, FkPlanView, FkDeviceInfo, META_WORDS, check


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def native_params(params, size, use_shift=True, shift=None) -> FkParams:
    """FoveationParams -> fk_params, with the host scalars of SURVEY.md Appendix A."""
    w, h = size
    mode = 1 if use_shift else 0
    sx = sy = 0
    if shift is not None:
        mode, (sx, sy) = 2, (int(shift[0]), int(shift[1]))
    return FkParams(
        alpha=float(params.alpha), e2=float(params.e2), ct0=float(params.ct0),
        e_corner=float(params.e_corner), strength=float(params.strength),
        log_inv_ct0=math.log(1.0 / params.ct0),       # retinal.py:129
        two_pi=2.0 * math.pi,                         # retinal.py:155
        fmax=float(params.max_cpd()),                 # retinal.py:63-65
        d_corner=math.hypot(w / 2.0, h / 2.0),        # retinal.py:111
        fragment_size=int(params.fragment_size), use_shift=mode, shift_x=sx, shift_y=sy)


class DevicePlan:
    """Device-resident plans (sigma, tap counts, order) for up to max_frames frames."""

    def __init__(self, engine: "Engine", size, fragment_size: int, max_frames: int):
        self.engine = engine
        self.size = (int(size[0]), int(size[1]))
        self.fragment_size = int(fragment_size)
        self.max_frames = int(max_frames)
        self.n_frames = 0
        self.fix_on_device = False
        ptr = C.c_void_p()
        check(engine._lib.fk_plan_create(engine._h, self.size[0], self.size[1],
                                         self.fragment_size, self.max_frames, C.byref(ptr)),
              engine._h)
        self._p = ptr
        self.cap = engine._lib.fk_plan_cell_capacity(ptr)

    def close(self):
        if self._p:
            self.engine._lib.fk_plan_destroy(self._p)
            self._p = None

    def __del__(self):  # best effort; the engine also closes cached plans
        try:
            self.close()
        except Exception:
            pass

    def model(self, params, fixations, use_shift=True, shift=None, stream=None):
        """Run the plan kernel for len(fixations) frames (fk_plan_model)."""
        eng = self.engine
        prm = native_params(params, self.size, use_shift, shift)
        if isinstance(fixations, torch.Tensor) and fixations.is_cuda:
            fix = fixations
            if fix.dtype != torch.float64 or not fix.is_contiguous() or fix.ndim != 2:
                raise ValueError("device fixations must be a contiguous float64 [N, 2] tensor")
            n, ptr, on_dev = fix.shape[0], C.c_void_p(fix.data_ptr()), 1
        else:
            fix = np.ascontiguousarray(np.asarray(fixations, dtype=np.float64).reshape(-1, 2))
            n, ptr, on_dev = fix.shape[0], _np_ptr(fix), 0
        with eng._lock:
            check(eng._lib.fk_plan_model(self._p, C.byref(prm), n, ptr, on_dev,
                                         eng._stream(stream)), eng._h)
        self.n_frames = n
        self.fix_on_device = bool(on_dev)
        return self

    def density(self, density_map, sigma_max, fragment_size, fixations, use_shift=True,
                shift=None, stream=None):
        """Plan from a 1-channel density map shared by all frames (fk_plan_density)."""
        eng = self.engine
        dm = np.ascontiguousarray(density_map, dtype=np.uint8)
        if dm.ndim != 2:
            raise ValueError("density map must be a 2-D uint8 array")
        mode, sx, sy = (1 if use_shift else 0), 0, 0
        if shift is not None:
            mode, (sx, sy) = 2, (int(shift[0]), int(shift[1]))
        prm = FkParams(fragment_size=int(fragment_size), use_shift=mode, shift_x=sx, shift_y=sy)
        fix = np.ascontiguousarray(np.asarray(fixations, dtype=np.float64).reshape(-1, 2))
        with eng._lock:
            check(eng._lib.fk_plan_density(self._p, C.byref(prm), fix.shape[0], _np_ptr(fix), 0,
                                           _np_ptr(dm), dm.shape[1], dm.shape[0],
                                           C.c_double(float(sigma_max)), eng._stream(stream)),
                  eng._h)
        self.n_frames = fix.shape[0]
        self.fix_on_device = False
        return self

    def set_grid(self, shift, lengths, offsets, coeffs, stream=None):
        """Install a caller-supplied (grid, bank) pair for one frame (fk_plan_set_grid)."""
        eng = self.engine
        lengths = np.ascontiguousarray(lengths, dtype=np.int32)
        offsets = np.ascontiguousarray(offsets, dtype=np.int32)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        gh, gw = lengths.shape
        with eng._lock:
            check(eng._lib.fk_plan_set_grid(self._p, int(shift[0]), int(shift[1]), gw, gh,
                                            _np_ptr(lengths), _np_ptr(offsets), _np_ptr(coeffs),
                                            int(coeffs.size), eng._stream(stream)), eng._h)
        self.n_frames = 1
        self.fix_on_device = False
        return self

    def read_items(self, stream=None) -> list:
        """The render kernels' work lists of the last plan (fk_plan_read_items): one uint32
        [n, 4] array per tap-count class -- frame, x0 | y0 << 16, width | taps << 8 |
        height << 21, tap offset.  For accounting (costs.items_macs); synchronises."""
        eng = self.engine
        out = []
        with eng._lock:
            for k in range(eng._lib.fk_plan_item_classes()):
                n = C.c_int(0)
                check(eng._lib.fk_plan_read_items(self._p, k, None, 0, C.byref(n),
                                                  eng._stream(stream)), eng._h)
                items = np.empty((max(n.value, 0), 4), np.uint32)
                if n.value > 0:
                    check(eng._lib.fk_plan_read_items(self._p, k, _np_ptr(items), n.value,
                                                      C.byref(n), eng._stream(stream)), eng._h)
                out.append(items)
        return out

    def bad_fixations(self, stream=None) -> int:
        """Frames of the last plan whose fixation was outside the image (fk_plan_status;
        synchronises).  Host fixations never get that far: fk_plan_model rejects them."""
        eng = self.engine
        bad = C.c_int(0)
        with eng._lock:
            check(eng._lib.fk_plan_status(self._p, C.byref(bad), eng._stream(stream)), eng._h)
        return int(bad.value)

    def read(self, frame=0, stream=None) -> dict:
        """Synchronising read-back of one frame's plan."""
        eng = self.engine
        sigma = np.empty(self.cap, np.float64)
        raw = np.empty(self.cap, np.int32)
        length = np.empty(self.cap, np.int32)
        view = FkPlanView(sigma=sigma.ctypes.data, raw_length=raw.ctypes.data,
                          length=length.ctypes.data)
        with eng._lock:
            check(eng._lib.fk_plan_read(self._p, int(frame), C.byref(view), eng._stream(stream)),
                  eng._h)
        if view.status != 0:
            raise ValueError("fixation outside image")
        gw, gh = view.grid_w, view.grid_h
        n = gw * gh
        return dict(shift=(view.shift_x, view.shift_y), grid=(gw, gh),
                    foveal=(view.foveal_gy, view.foveal_gx), max_length=view.max_length,
                    sigma=sigma[:n].reshape(gh, gw).copy(),
                    raw_length=raw[:n].reshape(gh, gw).astype(np.int64),
                    length=length[:n].reshape(gh, gw).astype(np.int64))

    def read_lengths(self, first=0, count=None, stream=None):
        """(lengths [count, cap] int32, meta [count, 8] int32) for a frame range."""
        eng = self.engine
        count = self.n_frames - first if count is None else count
        lengths = np.empty((count, self.cap), np.int32)
        meta = np.empty((count, META_WORDS), np.int32)
        with eng._lock:
            check(eng._lib.fk_plan_read_lengths(self._p, int(first), int(count), _np_ptr(lengths),
                                                _np_ptr(meta), eng._stream(stream)), eng._h)
        return lengths, meta


class FrameRequest:
    """One gaze-contingent frame as one CUDA-graph launch (fk_request_*): fixation upload ->
    plan -> render -> frame and plan summary in pinned host memory, captured for fixed
    parameters and buffers.  `launch(x, y)` queues a request on the stream the graph was
    captured on; after that stream has been synchronised `info()` describes the frame.
    Requests of one object (and of objects sharing a plan) must not be in flight together."""

    def __init__(self, engine: "Engine", plan: DevicePlan, params, src: torch.Tensor,
                 out: torch.Tensor, host: np.ndarray | None, stream):
        if not (src.is_cuda and out.is_cuda and src.is_contiguous() and out.is_contiguous()
                and src.shape == out.shape and src.dtype == out.dtype):
            raise ValueError("src and out must be matching contiguous CUDA tensors")
        if src.dtype not in (torch.uint8, torch.float32):
            raise ValueError(f"frames must be uint8 or float32, got {src.dtype}")
        h, w, c = src.shape[-3:]
        if (w, h) != plan.size or src.numel() != h * w * c:
            raise ValueError(f"grid does not match image {(w, h)}")
        if host is not None and (host.nbytes != src.numel() * src.element_size()
                                 or not host.flags.c_contiguous):
            raise ValueError("host buffer must be C-contiguous and as large as the frame")
        self.engine, self.plan, self.stream = engine, plan, stream
        self._keep = (src, out, host)
        prm = native_params(params, plan.size, True)
        ptr = C.c_void_p()
        with engine._lock:
            check(engine._lib.fk_request_create(
                engine._h, plan._p, C.byref(prm), C.c_void_p(src.data_ptr()),
                C.c_void_p(out.data_ptr()), _np_ptr(host) if host is not None else None,
                int(c), int(src.dtype == torch.float32), engine._stream(stream), C.byref(ptr)),
                engine._h)
        self._r = ptr
        plan.n_frames = 1
        plan.fix_on_device = True
        info = engine._lib.fk_request_info(ptr)
        self._info = np.ctypeslib.as_array(info, shape=(16 + plan.cap,))

    def launch(self, x: float, y: float) -> None:
        eng = self.engine
        with eng._lock:
            check(eng._lib.fk_request_launch(self._r, float(x), float(y),
                                             eng._stream(self.stream)), eng._h)

    def info(self) -> dict:
        """Plan summary of the last request (valid after the stream has been synchronised)."""
        m = self._info
        if m[7] != 0 or m[8] != 0:
            raise ValueError("fixation outside image")
        gw, gh = int(m[2]), int(m[3])
        return dict(shift=(int(m[0]), int(m[1])), grid=(gw, gh), foveal=(int(m[4]), int(m[5])),
                    max_length=int(m[6]),
                    length=m[16:16 + gw * gh].reshape(gh, gw).astype(np.int64))

    def close(self):
        if self._r:
            self.engine._lib.fk_request_destroy(self._r)
            self._r = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Engine:
    """One GPU.  Thread-safe: the (short, asynchronous) C calls on the handle are serialised by
    a lock; the GPU work they queue runs on the caller's stream, and callers on different
    streams get plans of their own (plan_for), so their kernels overlap."""

    def __init__(self, device: int = 0):
        self._lib = _native.lib()
        self.device = int(device)
        h = C.c_void_p()
        check(self._lib.fk_create(self.device, C.byref(h)))
        self._h = h
        self._lock = threading.RLock()
        self._plans: dict = {}
        info = FkDeviceInfo()
        check(self._lib.fk_get_device_info(self._h, C.byref(info)), self._h)
        self.info = dict(name=info.name.decode(), sm_count=info.sm_count,
                         cc=(info.cc_major, info.cc_minor), clock_khz=info.clock_khz,
                         l2_bytes=info.l2_bytes, global_mem_bytes=info.global_mem_bytes,
                         max_smem_optin=info.max_smem_optin)

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        with self._lock:
            for p in self._plans.values():
                p.close()
            self._plans.clear()
            if self._h:
                self._lib.fk_destroy(self._h)
                self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self, stream=None):
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        return C.c_void_p(int(stream))

    # ---------------------------------------------------------------------- plans
    def plan_for(self, size, fragment_size, n_frames, stream=None) -> DevicePlan:
        """A cached DevicePlan able to hold n_frames frames of this geometry, for work queued
        on `stream` (default: the current stream).  Plans are cached per (geometry, stream): a
        plan's buffers are rewritten by every call, so callers on different streams -- two
        service connections on one image size, the shards of a batch -- must not share one."""
        sid = int(self._stream(stream).value or 0)
        key = (int(size[0]), int(size[1]), int(fragment_size), sid)
        with self._lock:
            p = self._plans.get(key)
            if p is None or p.max_frames < n_frames:
                if p is not None:
                    torch.cuda.synchronize(self.device)
                    p.close()
                p = DevicePlan(self, size, fragment_size, max(int(n_frames), 1))
                self._plans[key] = p
            return p

    def lut_taps(self, length: int) -> np.ndarray:
        """fp64 taps of one odd length from the device LUT (fk_lut_read)."""
        out = np.empty(int(length), np.float64)
        with self._lock:
            check(self._lib.fk_lut_read(self._h, int(length), _np_ptr(out)), self._h)
        return out

    # --------------------------------------------------------------------- render
    def render(self, frames: torch.Tensor, plan: DevicePlan, out=None, stream=None):
        """Blur device frames [N, H, W, C] (uint8 or float32) with a prepared plan."""
        if not (isinstance(frames, torch.Tensor) and frames.is_cuda):
            raise ValueError("Engine.render takes a CUDA tensor")
        if frames.device.index != self.device:
            raise ValueError(f"frames live on {frames.device}, engine on cuda:{self.device}")
        if frames.ndim != 4 or not frames.is_contiguous():
            raise ValueError("frames must be a contiguous [N, H, W, C] tensor")
        n, h, w, c = frames.shape
        if (w, h) != plan.size:
            raise ValueError(f"grid does not match image {(w, h)}")
        if n != plan.n_frames:
            raise ValueError(f"{n} frames but {plan.n_frames} fixations planned")
        if out is None:
            out = torch.empty_like(frames)
        elif out.shape != frames.shape or out.dtype != frames.dtype or not out.is_contiguous() \
                or out.device != frames.device:
            raise ValueError("out must match frames in shape, dtype and device")
        if frames.dtype == torch.uint8:
            fn = self._lib.fk_render_u8
        elif frames.dtype == torch.float32:
            fn = self._lib.fk_render_f32
        else:
            raise ValueError(f"frames must be uint8 or float32, got {frames.dtype}")
        with self._lock:
            check(fn(self._h, plan._p, C.c_void_p(frames.data_ptr()),
                     C.c_void_p(out.data_ptr()), int(n), int(c), self._stream(stream)), self._h)
        return out

    def foveate_device(self, frames: torch.Tensor, fixations, params, use_shift=True,
                       out=None, stream=None, validate=True):
        """plan + render for frames already resident on this GPU; returns (out, plan).

        Fixations that live on the device cannot be range-checked on the host; with
        ``validate`` (default) the plan kernel's count of out-of-image fixations is read
        back after the render has been queued (one 4-byte copy, synchronises the stream)
        and ValueError is raised as the reference does (retinal.py:73-74).  Pass
        ``validate=False`` to keep the call asynchronous: such frames are then copied
        through unchanged."""
        n, h, w, _ = frames.shape
        nfix = fixations.shape[0] if hasattr(fixations, "shape") else len(fixations)
        if nfix != n:
            raise ValueError(f"{n} frames but {nfix} fixations")
        with self._lock:
            plan = self.plan_for((w, h), params.fragment_size, n, stream=stream)
            plan.model(params, fixations, use_shift=use_shift, stream=stream)
            out = self.render(frames, plan, out=out, stream=stream)
            if validate and plan.fix_on_device:
                bad = plan.bad_fixations(stream=stream)
                if bad:
                    raise ValueError(f"fixation of {bad} frame(s) outside {w}x{h} image")
        return out, plan

    def foveate_host(self, frames: np.ndarray, fixations: np.ndarray, params, out=None,
                     use_shift=True, chunk_frames=0):
        """Host frames in, host frames out through the pipelined C entry point."""
        frames = np.asarray(frames)
        if frames.ndim != 4 or not frames.flags.c_contiguous:
            raise ValueError("frames must be a C-contiguous [N, H, W, C] array")
        n, h, w, c = frames.shape
        fix = np.ascontiguousarray(np.asarray(fixations, dtype=np.float64).reshape(-1, 2))
        if fix.shape[0] != n:
            raise ValueError(f"{n} frames but {fix.shape[0]} fixations")
        if out is None:
            out = np.empty_like(frames)
        elif out.shape != frames.shape or out.dtype != frames.dtype or not out.flags.c_contiguous:
            raise ValueError("out must match frames in shape and dtype")
        if frames.dtype == np.uint8:
            fn = self._lib.fk_foveate_host_u8
        elif frames.dtype == np.float32:
            fn = self._lib.fk_foveate_host_f32
        else:
            raise ValueError(f"frames must be uint8 or float32, got {frames.dtype}")
        prm = native_params(params, (w, h), use_shift)
        with self._lock:
            check(fn(self._h, C.byref(prm), w, h, c, n, _np_ptr(fix), _np_ptr(frames),
                     _np_ptr(out), int(chunk_frames)), self._h)
        return out

    # ---------------------------------------------------------------- measurement
    # ----------------------------------------------------------------------- SSIM
    def ssim_values(self, ref: torch.Tensor, test: torch.Tensor, window: np.ndarray, c1: float,
                    c2: float, values=None, accumulate=False, stream=None) -> torch.Tensor:
        """fk_ssim_u8: the SSIM map of two device images [H, W, C] as a float64 CUDA tensor
        (optionally accumulated onto `values`)."""
        for t in (ref, test):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.uint8
                    and t.ndim == 3 and t.is_contiguous() and t.device.index == self.device):
                raise ValueError("ssim_values takes contiguous uint8 CUDA tensors [H, W, C]")
        h, w, c = ref.shape
        win = np.ascontiguousarray(window, dtype=np.float64)
        n = int(win.shape[0])
        if values is None:
            if accumulate:
                raise ValueError("accumulate needs a map to add onto")
            values = torch.empty((max(h - n + 1, 1), max(w - n + 1, 1)), dtype=torch.float64,
                                 device=ref.device)
        with self._lock:
            check(self._lib.fk_ssim_u8(self._h, C.c_void_p(ref.data_ptr()),
                                       C.c_void_p(test.data_ptr()), int(w), int(h), int(c),
                                       _np_ptr(win), n, float(c1), float(c2),
                                       C.c_void_p(values.data_ptr()), int(bool(accumulate)),
                                       self._stream(stream)), self._h)
        return values

    def ssim_stats(self, values: torch.Tensor, divisor: float = 1.0, stream=None):
        """fk_ssim_stats: (mean, min, flat argmin) of a device map, after values /= divisor."""
        out = np.empty(3, np.float64)
        with self._lock:
            check(self._lib.fk_ssim_stats(self._h, C.c_void_p(values.data_ptr()),
                                          int(values.numel()), float(divisor), _np_ptr(out),
                                          self._stream(stream)), self._h)
        return float(out[0]), float(out[1]), int(out[2])

    def set_kernel_variant(self, variant: int) -> int:
        return int(self._lib.fk_set_kernel_variant(self._h, int(variant)))

    def launch_count(self) -> int:
        return int(self._lib.fk_launch_count(self._h))

    def measure_fp32_peak(self):
        tf, ms = C.c_double(), C.c_double()
        with self._lock:
            check(self._lib.fk_measure_fp32_peak(self._h, C.byref(tf), C.byref(ms)), self._h)
        return tf.value, ms.value


def pinned_empty(shape, dtype) -> np.ndarray:
    """A numpy array backed by pinned host memory (fk_host_alloc); freed with the array."""
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    ptr = C.c_void_p()
    check(_native.lib().fk_host_alloc(max(nbytes, 1), C.byref(ptr)))
    buf = (C.c_char * max(nbytes, 1)).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
    weakref.finalize(buf, _native.lib().fk_host_free, ptr)
    return arr


_engines: dict = {}
_engines_lock = threading.Lock()


def get_engine(device: int = 0) -> Engine:
    """Process-wide engine for a device (created on first use)."""
    device = int(device)
    with _engines_lock:
        eng = _engines.get(device)
        if eng is None or eng._h is None:
            eng = Engine(device)
            _engines[device] = eng
        return eng


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [first, last) slice of n frames owned by `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    base, extra = divmod(int(n), world)
    first = rank * base + min(rank, extra)
    return first, first + base + (1 if rank < extra else 0)
