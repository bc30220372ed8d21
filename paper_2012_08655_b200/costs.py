"""Algorithmic work of the blur per frame -- the numerators of the roofline.

MACs per channel = sum over non-identity fragments of L * (fw * (fh + 2r) + fw * fh),
r = (L - 1) / 2: the per-fragment count of foveakit.costs.ops_per_output_pixel
(costs.py:32-35, G * (2 + (G - 1) / F) MAC per pixel) on the true clipped fragment sizes.
Bytes per frame = read once + write once."""

from __future__ import annotations

import numpy as np

from .tiling import fragment_spans


def frame_macs(size, fragment_size: int, shift, lengths) -> int:
    """Per-channel multiply-accumulates for one frame's (gh, gw) tap-count grid."""
    w, h = size
    spx = fragment_spans(w, fragment_size, int(shift[0]))
    spy = fragment_spans(h, fragment_size, int(shift[1]))
    fw = (spx[:, 1] - spx[:, 0])[None, :]
    fh = (spy[:, 1] - spy[:, 0])[:, None]
    L = np.asarray(lengths, dtype=np.int64).reshape(len(spy), len(spx))
    r = (L - 1) // 2
    return int(np.where(L > 1, L * (fw * (fh + 2 * r) + fw * fh), 0).sum())


def batch_flops(size, fragment_size: int, channels: int, lengths, meta) -> float:
    """Total algorithmic FLOPs (2 per MAC, all channels) of a planned batch, from
    DevicePlan.read_lengths() output."""
    total = 0
    for i in range(len(meta)):
        sx, sy, gw, gh = (int(v) for v in meta[i, :4])
        total += frame_macs(size, fragment_size, (sx, sy), lengths[i, : gw * gh])
    return 2.0 * channels * total


def frame_bytes(size, channels: int, itemsize: int) -> int:
    """Algorithmic HBM bytes per frame: every sample read once and written once."""
    return 2 * size[0] * size[1] * channels * itemsize
