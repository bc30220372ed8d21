"""Host model of the plan kernel's strip emission (csrc/fk_plan.cu, fk_emit_items) and of the
lane slots the render kernel spends on the strips.  Design tool: runs without a GPU (plans
come from the numpy oracle) and answers, per workload, where FLOPs go:

  algorithmic  2 C sum_cells L (fw (fh + 2r) + fw fh)           (the roofline numerator)
  executed     the same sum over the merged strips (halo rows between merged fragments once)
  slots        what the kernel's partition pays for them: a strip occupies all four warps
               whatever its width (96 float columns), the H pass one lane per tile row in
               blocks of 32 rows (short first block), the V pass rounds of 32 (pixel, group)
               tasks per warp.

usage: python tools/strip_model.py W H F [e2] [fixation: centre|corner|moving|random] [frames]
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import fovea_oracle as fo  # noqa: E402

RECT = 32


def spans(extent, F, off):
    return fo.np_fragment_spans(extent, F, off)


def emit_strips(size, F, shift, length, strip_rows=1024, hsplit=False, vmerge_wide=False):
    """(x0, y0, fw, fh, L) strips as fk_emit_items produces them.  hsplit: cut a group of
    cells that do not share their taps into runs of equal cells instead of single cells;
    vmerge_wide: merge vertically for F > 32 as well."""
    w, h = size
    sx, sy = shift
    spx, spy = spans(w, F, sx), spans(h, F, sy)
    gh, gw = length.shape
    merge = F <= RECT
    mgrp = RECT // F if merge else 1
    lead = 1 if sx > 0 else 0
    vm = merge or vmerge_wide
    maxc = max(strip_rows // F, 1) if vm else 1
    units = []  # per grid row: list of (g0, g1)
    for gy in range(gh):
        row = []
        gx = 0
        while gx < gw:
            if mgrp <= 1 or (lead and gx == 0):
                row.append((gx, gx + 1))
                gx += 1
                continue
            g0 = lead + ((gx - lead) // mgrp) * mgrp
            g1 = min(g0 + mgrp, gw)
            Ls = length[gy, g0:g1]
            if g1 - g0 >= 2 and Ls[0] > 1 and np.all(Ls == Ls[0]):
                row.append((g0, g1))
            elif hsplit:
                a = g0
                while a < g1:
                    b = a + 1
                    while b < g1 and length[gy, b] == length[gy, a] and length[gy, a] > 1:
                        b += 1
                    row.append((a, b))
                    a = b
            else:
                row.extend((x, x + 1) for x in range(g0, g1))
            gx = g1
        units.append(row)
    out = []
    # vertical greedy merging per unit column key (g0, g1)
    open_ = {}  # (g0, g1) -> [gy0, n, L]
    for gy in range(gh):
        seen = set()
        for (g0, g1) in units[gy]:
            L = int(length[gy, g0])
            key = (g0, g1)
            seen.add(key)
            cur = open_.get(key)
            if cur and vm and L > 1 and cur[2] == L and cur[0] + cur[1] == gy and cur[1] < maxc:
                cur[1] += 1
            else:
                if cur:
                    out.append((key, *cur))
                open_[key] = [gy, 1, L]
        for key in list(open_):
            if key not in seen:
                out.append((key, *open_.pop(key)))
    for key, cur in open_.items():
        out.append((key, *cur))
    strips = []
    for (g0, g1), gy0, n, L in out:
        x0, x1 = int(spx[g0, 0]), int(spx[g1 - 1, 1])
        y0, y1 = int(spy[gy0, 0]), int(spy[gy0 + n - 1, 1])
        for xs in range(x0, x1, RECT):
            strips.append((xs, y0, min(RECT, x1 - xs), y1 - y0, L))
    return strips


def account(size, F, shift, length, strips, C=3):
    w, h = size
    spx, spy = spans(w, F, shift[0]), spans(h, F, shift[1])
    fw = (spx[:, 1] - spx[:, 0])[None, :]
    fh = (spy[:, 1] - spy[:, 0])[:, None]
    L = length.astype(np.int64)
    r = (L - 1) // 2
    alg = int(np.where(L > 1, L * (fw * (fh + 2 * r) + fw * fh), 0).sum())
    ex = slots = hs = vs = 0
    for (x0, y0, sw, sh, l) in strips:
        if l <= 1:
            continue
        rr = (l - 1) // 2
        th = sh + 2 * rr
        ex += l * (sw * th + sw * sh)
        # H pass: blocks of 32 rows after a short first block; every block costs 32 lane rows
        lead = (2 * rr) & 31
        n_first = min(th, 32) if lead == 0 or lead > th else lead
        nblocks = 1 + -(-(th - n_first) // 32)
        hslot = l * RECT * 32 * nblocks
        # V pass: rounds of 32 tasks (8 pixels x groups of 8 rows) per warp, 8 rows per task
        groups = -(-sh // 8)
        # per block the V pass runs over the groups it released; approximate by total rounds
        vrounds = -(-(groups * 8) // 32)
        vslot = l * RECT * vrounds * 32
        slots += hslot + vslot
        hs += hslot
        vs += vslot
    return alg, ex, slots, hs, vs


def fixations(kind, n, w, h, seed=1):
    if kind == "centre":
        return np.tile([[w / 2.0, h / 2.0]], (n, 1))
    if kind == "corner":
        return np.zeros((n, 2))
    if kind == "random":
        rng = np.random.default_rng(seed)
        return np.stack([rng.integers(0, w, n), rng.integers(0, h, n)], axis=1).astype(float)
    i = np.arange(n, dtype=np.float64)
    return np.stack([np.floor(w / 2 + 0.4 * w * np.cos(2 * np.pi * i / n)),
                     np.floor(h / 2 + 0.4 * h * np.sin(2 * np.pi * i / n))], axis=1)


def main():
    w, h, F = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    e2 = float(sys.argv[4]) if len(sys.argv) > 4 else 2.3
    kind = sys.argv[5] if len(sys.argv) > 5 else "centre"
    n = int(sys.argv[6]) if len(sys.argv) > 6 else (1 if kind in ("centre", "corner") else 8)
    for label, kw in (("current", {}), ("hsplit", dict(hsplit=True)),
                      ("vmerge_wide", dict(vmerge_wide=True)),
                      ("both", dict(hsplit=True, vmerge_wide=True))):
        tot = np.zeros(5)
        nstrips = 0
        for fx in fixations(kind, n, w, h):
            pl = fo.np_plan((w, h), fo.OracleParams(fragment_size=F, e2=e2, fixation=(float(fx[0]), float(fx[1]))))
            st = emit_strips((w, h), F, pl["shift"], pl["length"], **kw)
            nstrips += len(st)
            tot += account((w, h), F, pl["shift"], pl["length"], st)
        alg, ex, slots, hs, vs = tot
        print(f"{label:12s} strips/frame {nstrips / n:8.0f}  executed/alg {ex / alg:.3f}  "
              f"slots/alg {slots / alg:.3f} (H {hs / alg:.3f} V {vs / alg:.3f})  useful/slots {ex / slots:.3f}")


if __name__ == "__main__":
    main()
