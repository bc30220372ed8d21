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
    DevicePlan.read_lengths() output.  Frames that share a tiling shift share their fragment
    sizes, so the batch is summed shift by shift (at most fragment_size^2 groups)."""
    w, h = size
    meta = np.asarray(meta)
    lengths = np.asarray(lengths)
    key = meta[:, 0].astype(np.int64) * 65536 + meta[:, 1]
    total = 0
    for k in np.unique(key):
        rows = np.nonzero(key == k)[0]
        sx, sy, gw, gh = (int(v) for v in meta[rows[0], :4])
        spx = fragment_spans(w, fragment_size, sx)
        spy = fragment_spans(h, fragment_size, sy)
        fw = (spx[:, 1] - spx[:, 0])[None, None, :]
        fh = (spy[:, 1] - spy[:, 0])[None, :, None]
        L = lengths[rows, : gw * gh].astype(np.int64).reshape(len(rows), gh, gw)
        r = (L - 1) // 2
        total += int(np.where(L > 1, L * (fw * (fh + 2 * r) + fw * fh), 0).sum())
    return 2.0 * channels * total


def frame_bytes(size, channels: int, itemsize: int) -> int:
    """Algorithmic HBM bytes per frame: every sample read once and written once."""
    return 2 * size[0] * size[1] * channels * itemsize


def items_macs(items) -> int:
    """Per-channel multiply-accumulates the render kernels execute for one work list
    (DevicePlan.read_items): L * (w * (h + 2r) + w * h) per strip.  Merged strips run the
    horizontal pass over the 2r halo rows between their fragments once, so this is below
    the algorithmic count of frame_macs, which charges every fragment its own halo.  A mixed
    item (bit 31 of its last word: a filter per 8-pixel column, radii packed 6 bits each) is
    the sum over its columns."""
    it = np.asarray(items, dtype=np.int64).reshape(-1, 4)
    if it.size == 0:
        return 0
    w = it[:, 2] & 0xFF
    L = (it[:, 2] >> 8) & 0x1FFF
    h = it[:, 2] >> 21
    mixed = (it[:, 3] >> 31) & 1
    r = (L - 1) // 2
    total = int(np.where((L > 1) & (mixed == 0), L * (w * (h + 2 * r) + w * h), 0).sum())
    for k in range(4):
        rk = (it[:, 3] >> (6 * k)) & 63
        wk = np.clip(w - 8 * k, 0, 8)
        Lk = 2 * rk + 1
        total += int(np.where((mixed == 1) & (wk > 0), Lk * (wk * (h + 2 * rk) + wk * h), 0).sum())
    return total


def executed_flops(item_lists, channels: int) -> float:
    """FLOPs the strips of a planned batch execute (2 per MAC, all channels)."""
    return 2.0 * channels * sum(items_macs(it) for it in item_lists)
