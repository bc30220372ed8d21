"""Gaze-contingent streaming of one resident image.

The reference streams frames from a websocket handler (service.py:192-238): a reader task
overwrites a one-slot mailbox with the newest message ("latest wins"), a render loop takes
whatever is in the slot, applies it to the per-connection parameters
(`_ConnectionState.apply`, service.py:121-146 -- overrides persist, the fixation is clamped
into the image and the clamp is reported) and renders with `blockwise.foveate`.  Its frame
time is dominated by the host<->device traffic the paper measures.

`FoveationStream` is that loop for the B200 path, without the web plumbing: the source image
is uploaded ONCE and stays in HBM; a worker thread owns a CUDA stream, a one-frame device
plan and a ring of pinned host buffers.  A request is ONE CUDA-graph launch
(`engine.FrameRequest`, fk_request_*): 16 bytes of fixation up, plan -> render on the device,
the frame and its plan summary down to pinned memory -- no per-kernel launch calls and no
synchronising read-back after the frame.  Graphs are captured per (parameters other than the
fixation, output slot) the first time a combination is requested.  Requests that arrive while
a frame is in flight overwrite each other; only the newest is rendered.
"""

from __future__ import annotations

import queue
import threading
import time
from dataclasses import replace

import numpy as np
import torch

from .engine import DevicePlan, FrameRequest, get_engine, pinned_empty
from .imaging import RasterImage
from .retinal import FoveationParams


def clamp_fixation(x: float, y: float, size) -> tuple[float, float, bool]:
    """service.py:58-63: clamp into [0, w-1] x [0, h-1]; True when the point moved."""
    w, h = size
    cx = min(max(float(x), 0.0), w - 1.0)
    cy = min(max(float(y), 0.0), h - 1.0)
    return cx, cy, (cx != x or cy != y)


class FoveationStream:
    """Latest-wins foveation of one device-resident image.

    submit(x, y, e_corner=..., strength=..., fragment=...) never blocks; frames() / get()
    yield (image uint8[H, W, C] in pinned memory, stats dict) for the requests that were
    actually rendered.  A returned array belongs to the caller until `depth - 1` further
    frames have been taken."""

    def __init__(self, source, params: FoveationParams | None = None, device: int = 0,
                 depth: int = 3):
        img = source.data if isinstance(source, RasterImage) else np.asarray(source)
        if img.ndim == 2:
            img = img[:, :, None]
        if img.dtype != np.uint8 or img.ndim != 3 or img.shape[2] not in (1, 3):
            raise ValueError("source must be a uint8 image with 1 or 3 channels")
        if depth < 2:
            raise ValueError(f"depth must be >= 2, got {depth}")
        self.size = (img.shape[1], img.shape[0])
        self.params = params if params is not None else FoveationParams()
        self._eng = get_engine(device)
        self._device = int(device)
        self._stream = torch.cuda.Stream(device=device)
        with torch.cuda.device(device):
            self._src = torch.from_numpy(np.ascontiguousarray(img)[None]).cuda()
            self._dev = [torch.empty_like(self._src) for _ in range(depth)]
        self._host = [pinned_empty(img.shape, np.uint8) for _ in range(depth)]
        self._plans: dict[int, DevicePlan] = {}
        self._requests: dict = {}
        self._slot = 0
        self._pending = None            # the mailbox: newest request, or None
        self._cv = threading.Condition()
        self._closed = False
        self._out: queue.Queue = queue.Queue()
        self.submitted = 0
        self.rendered = 0
        self._worker = threading.Thread(target=self._run, name="foveation-stream", daemon=True)
        self._worker.start()

    # ------------------------------------------------------------------ client side
    def submit(self, x: float, y: float, **overrides) -> None:
        """Post a request (service.py:213 `pending[0] = msg  # latest wins`)."""
        unknown = set(overrides) - {"e_corner", "strength", "fragment"}
        if unknown:
            raise ValueError(f"unknown fields {sorted(unknown)}")
        with self._cv:
            if self._closed:
                raise RuntimeError("stream is closed")
            self._pending = (float(x), float(y), dict(overrides))
            self.submitted += 1
            self._cv.notify()

    def get(self, timeout: float | None = None):
        """Next rendered (image, stats); raises queue.Empty on timeout, ValueError for a
        request the reference would have answered with an error message."""
        item = self._out.get(timeout=timeout)
        if isinstance(item, Exception):
            raise item
        return item

    def close(self) -> None:
        with self._cv:
            self._closed = True
            self._cv.notify()
        self._worker.join()
        for r in self._requests.values():
            r.close()
        self._requests.clear()
        for p in self._plans.values():
            p.close()
        self._plans.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------------ worker side
    def _apply(self, x, y, overrides):
        """_ConnectionState.apply (service.py:121-146): overrides persist."""
        updates = {}
        if "e_corner" in overrides:
            updates["e_corner"] = float(overrides["e_corner"])
        if "strength" in overrides:
            updates["strength"] = float(overrides["strength"])
        if "fragment" in overrides:
            updates["fragment_size"] = int(overrides["fragment"])
        cx, cy, clamped = clamp_fixation(x, y, self.size)
        updates["fixation"] = (cx, cy)
        self.params = replace(self.params, **updates)
        return self.params, clamped

    def _plan(self, fragment_size: int) -> DevicePlan:
        p = self._plans.get(fragment_size)
        if p is None:
            p = DevicePlan(self._eng, self.size, fragment_size, 1)
            self._plans[fragment_size] = p
        return p

    def _request(self, params: FoveationParams, slot: int) -> FrameRequest:
        """The captured graph for these parameters and this output slot."""
        key = (replace(params, fixation=None), slot)
        r = self._requests.get(key)
        if r is None:
            if len(self._requests) >= 8 * len(self._dev):   # parameters keep changing: start over
                self._stream.synchronize()
                for old in self._requests.values():
                    old.close()
                self._requests.clear()
            r = FrameRequest(self._eng, self._plan(params.fragment_size), params, self._src[0],
                             self._dev[slot][0], self._host[slot], self._stream)
            self._requests[key] = r
        return r

    def _run(self):
        torch.cuda.set_device(self._device)
        while True:
            with self._cv:
                while self._pending is None and not self._closed:
                    self._cv.wait()
                if self._closed:
                    return
                x, y, overrides = self._pending
                self._pending = None
            try:
                params, clamped = self._apply(x, y, overrides)
                slot = self._slot
                self._slot = (slot + 1) % len(self._dev)
                req = self._request(params, slot)
                t0 = time.perf_counter()
                req.launch(*params.fixation)
                self._stream.synchronize()
                ms = (time.perf_counter() - t0) * 1000.0
                info = req.info()
                stats = {
                    "render_ms": round(ms, 3),
                    "regions": int(len(np.unique(info["length"]))),
                    "fragment": params.fragment_size,
                    "method": "blockwise",
                    "shift": [int(info["shift"][0]), int(info["shift"][1])],
                    "x": params.fixation[0],
                    "y": params.fixation[1],
                }
                if clamped:
                    stats["warning"] = "fixation clamped to image bounds"
                self.rendered += 1
                self._out.put((self._host[slot], stats))
            except (ValueError, RuntimeError) as exc:   # the reference sends {"error": ...}
                self._out.put(exc)
