"""SSIM maps on the GPU -- mirror of foveakit.quality (quality.py:1-114), the tool the
reference uses to validate the block-wise renderer.

Same names, arguments and error messages as the reference; the arithmetic (BT.601 luma, five
separable windowed means over fully-valid windows, SSIM formula, fp64) runs in
``csrc/fk_ssim.cu`` behind ``fk_ssim_u8`` / ``fk_ssim_stats``.  There is no CPU path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .engine import get_engine
from .imaging import RasterImage

WINDOW_SIZE = 11
WINDOW_SIGMA = 1.5
K1 = 0.01
K2 = 0.03
DYNAMIC_RANGE = 255.0


def _window() -> np.ndarray:
    """quality.py:38-42, the reference's own expression (host scalars, like the LUT inputs)."""
    r = WINDOW_SIZE // 2
    k = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-(k * k) / (2.0 * WINDOW_SIGMA * WINDOW_SIGMA))
    return w / w.sum()


@dataclass(frozen=True)
class SSIMMap:
    """Dense per-window SSIM plus its summary statistics (quality.py:51-67)."""

    values: np.ndarray  # float64, (h - 10, w - 10), in [-1, 1]
    mean: float
    min: float
    argmin: tuple[int, int]  # image coordinates (y, x) of the worst window center

    def to_image(self) -> RasterImage:
        """8-bit rendering of the map: round(255 * clamp(ssim, 0, 1)) (convolve.py:15)."""
        v = np.clip(self.values, 0.0, 1.0) * 255.0
        return RasterImage.from_array(np.clip(np.floor(v + 0.5), 0, 255).astype(np.uint8))

    def stats_text(self) -> str:
        return (
            f"mean {self.mean:.6f}\n"
            f"min {self.min:.6f}\n"
            f"argmin {self.argmin[1]} {self.argmin[0]}\n"
        )


def _check_pair(reference: RasterImage, test: RasterImage) -> None:
    if reference.size != test.size or reference.channels != test.channels:
        raise ValueError(
            f"dimension mismatch: {reference.size}x{reference.channels} vs "
            f"{test.size}x{test.channels}"
        )
    if reference.width < WINDOW_SIZE or reference.height < WINDOW_SIZE:
        raise ValueError(f"images must be at least {WINDOW_SIZE}px per side")


def _finish(eng, values: torch.Tensor, divisor: float) -> SSIMMap:
    """_map_from_values (quality.py:70-79) on the device map."""
    mean, mn, flat = eng.ssim_stats(values, divisor)
    my, mx = divmod(flat, values.shape[1])
    offset = WINDOW_SIZE // 2
    return SSIMMap(values=values.cpu().numpy(), mean=mean, min=mn,
                   argmin=(int(my) + offset, int(mx) + offset))


def _constants():
    return (K1 * DYNAMIC_RANGE) ** 2, (K2 * DYNAMIC_RANGE) ** 2


def ssim_map(reference: RasterImage, test: RasterImage, device: int = 0) -> SSIMMap:
    """quality.py:82-103."""
    _check_pair(reference, test)
    eng = get_engine(device)
    dev = torch.device("cuda", device)
    c1, c2 = _constants()
    x = torch.from_numpy(np.ascontiguousarray(reference.data)).to(dev)
    y = torch.from_numpy(np.ascontiguousarray(test.data)).to(dev)
    values = eng.ssim_values(x, y, _window(), c1, c2)
    return _finish(eng, values, 1.0)


def mean_ssim_map(pairs, device: int = 0) -> SSIMMap:
    """Pixel-wise arithmetic mean of the SSIM maps of (reference, test) pairs
    (quality.py:106-114): the maps are summed on the device in the order given."""
    pairs = list(pairs)
    if not pairs:
        raise ValueError("mean_ssim_map needs at least one pair")
    eng = get_engine(device)
    dev = torch.device("cuda", device)
    c1, c2 = _constants()
    win = _window()
    values = None
    for ref, test in pairs:
        _check_pair(ref, test)
        shape = (ref.height - WINDOW_SIZE + 1, ref.width - WINDOW_SIZE + 1)
        if values is not None and tuple(values.shape) != shape:
            raise ValueError("all pairs must share the same dimensions")
        x = torch.from_numpy(np.ascontiguousarray(ref.data)).to(dev)
        y = torch.from_numpy(np.ascontiguousarray(test.data)).to(dev)
        values = eng.ssim_values(x, y, win, c1, c2, values=values, accumulate=values is not None)
    return _finish(eng, values, float(len(pairs)))
