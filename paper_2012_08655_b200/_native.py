"""ctypes binding of libfovea.so (include/fovea.h).  No torch types cross this boundary.

Loading never falls back to a CPU implementation: if the shared object cannot be built or
loaded the import fails, and on a box without a CUDA device ``fk_create`` reports
FK_ECUDA which surfaces here as ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import _build

FK_OK, FK_EINVAL, FK_ECUDA, FK_ENOMEM = 0, 1, 2, 3
META_WORDS = 8

#: every symbol include/fovea.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "fk_abi_version", "fk_device_count", "fk_create", "fk_destroy", "fk_last_error",
    "fk_get_device_info", "fk_build_lut", "fk_lut_max_length", "fk_lut_read",
    "fk_plan_create", "fk_plan_destroy", "fk_plan_cell_capacity", "fk_plan_model",
    "fk_plan_density", "fk_plan_set_grid", "fk_plan_read", "fk_plan_read_lengths",
    "fk_plan_status", "fk_plan_item_classes", "fk_plan_read_items", "fk_render_u8",
    "fk_render_f32", "fk_set_kernel_variant", "fk_launch_count", "fk_foveate_host_u8",
    "fk_foveate_host_f32", "fk_request_create", "fk_request_launch", "fk_request_info",
    "fk_request_destroy", "fk_host_alloc", "fk_host_free", "fk_measure_fp32_peak", "fk_ssim_u8", "fk_ssim_stats",
]


class FkParams(C.Structure):
    _fields_ = [
        ("alpha", C.c_double), ("e2", C.c_double), ("ct0", C.c_double),
        ("e_corner", C.c_double), ("strength", C.c_double), ("log_inv_ct0", C.c_double),
        ("two_pi", C.c_double), ("fmax", C.c_double), ("d_corner", C.c_double),
        ("fragment_size", C.c_int32), ("use_shift", C.c_int32),
        ("shift_x", C.c_int32), ("shift_y", C.c_int32),
    ]


class FkPlanView(C.Structure):
    _fields_ = [
        ("shift_x", C.c_int32), ("shift_y", C.c_int32), ("grid_w", C.c_int32),
        ("grid_h", C.c_int32), ("foveal_gy", C.c_int32), ("foveal_gx", C.c_int32),
        ("max_length", C.c_int32), ("status", C.c_int32),
        ("sigma", C.c_void_p), ("raw_length", C.c_void_p), ("length", C.c_void_p),
    ]


class FkDeviceInfo(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("sm_count", C.c_int32), ("cc_major", C.c_int32),
        ("cc_minor", C.c_int32), ("clock_khz", C.c_int32), ("l2_bytes", C.c_int32),
        ("global_mem_bytes", C.c_int64), ("max_smem_optin", C.c_int32), ("name", C.c_char * 64),
    ]


_lib = None
_lock = threading.Lock()


def _declare(lib):
    vp, i32, i64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_double
    P = C.POINTER
    sig = {
        "fk_abi_version": (i32, []),
        "fk_device_count": (i32, [P(C.c_int)]),
        "fk_create": (i32, [i32, P(vp)]),
        "fk_destroy": (i32, [vp]),
        "fk_last_error": (C.c_char_p, [vp]),
        "fk_get_device_info": (i32, [vp, P(FkDeviceInfo)]),
        "fk_build_lut": (i32, [vp, i32, vp]),
        "fk_lut_max_length": (i32, [vp, P(C.c_int)]),
        "fk_lut_read": (i32, [vp, i32, vp]),
        "fk_plan_create": (i32, [vp, i32, i32, i32, i32, P(vp)]),
        "fk_plan_destroy": (i32, [vp]),
        "fk_plan_cell_capacity": (i32, [vp]),
        "fk_plan_model": (i32, [vp, P(FkParams), i32, vp, i32, vp]),
        "fk_plan_density": (i32, [vp, P(FkParams), i32, vp, i32, vp, i32, i32, dbl, vp]),
        "fk_plan_set_grid": (i32, [vp, i32, i32, i32, i32, vp, vp, vp, i32, vp]),
        "fk_plan_read": (i32, [vp, i32, P(FkPlanView), vp]),
        "fk_plan_read_lengths": (i32, [vp, i32, i32, vp, vp, vp]),
        "fk_plan_status": (i32, [vp, P(C.c_int), vp]),
        "fk_plan_item_classes": (i32, []),
        "fk_plan_read_items": (i32, [vp, i32, vp, i32, P(C.c_int), vp]),
        "fk_render_u8": (i32, [vp, vp, vp, vp, i32, i32, vp]),
        "fk_render_f32": (i32, [vp, vp, vp, vp, i32, i32, vp]),
        "fk_set_kernel_variant": (i32, [vp, i32]),
        "fk_launch_count": (i64, [vp]),
        "fk_foveate_host_u8": (i32, [vp, P(FkParams), i32, i32, i32, i32, vp, vp, vp, i32]),
        "fk_foveate_host_f32": (i32, [vp, P(FkParams), i32, i32, i32, i32, vp, vp, vp, i32]),
        "fk_request_create": (i32, [vp, vp, P(FkParams), vp, vp, vp, i32, i32, vp, P(vp)]),
        "fk_request_launch": (i32, [vp, dbl, dbl, vp]),
        "fk_request_info": (P(C.c_int32), [vp]),
        "fk_request_destroy": (i32, [vp]),
        "fk_host_alloc": (i32, [C.c_size_t, P(vp)]),
        "fk_host_free": (i32, [vp]),
        "fk_measure_fp32_peak": (i32, [vp, P(dbl), P(dbl)]),
        "fk_ssim_u8": (i32, [vp, vp, vp, i32, i32, i32, vp, i32, dbl, dbl, vp, i32, vp]),
        "fk_ssim_stats": (i32, [vp, vp, i64, dbl, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded libfovea.so (built in-tree on first use if missing or stale)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                # FK_LIB_PATH (tuning runs): load an alternative build of libfovea.so as it is
                path = os.environ.get("FK_LIB_PATH") or _build.build_native()
                loaded = C.CDLL(str(path))
                _declare(loaded)
                if loaded.fk_abi_version() != 1:
                    raise RuntimeError("libfovea.so ABI version mismatch")
                _lib = loaded
    return _lib


def last_error(handle=None) -> str:
    msg = lib().fk_last_error(handle)
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, handle=None) -> None:
    """Map a libfovea status to the exception the reference API would raise."""
    if rc == FK_OK:
        return
    msg = last_error(handle) or last_error(None) or f"libfovea error {rc}"
    if rc == FK_EINVAL:
        raise ValueError(msg)
    if rc == FK_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)
