/*
 * fk_plan.cu -- device-side planning for blockwise foveation (sm_100a).
 *
 *   fk_plan_kernel   one CTA per frame: tiling shift, grid geometry, per-fragment
 *                    eccentricity -> sigma (fp64, bit-identical to the reference),
 *                    tap count, foveal-fragment forcing, and the render kernels' work
 *                    items (same-filter strips, one list per tap-count class).
 *   fk_lut_kernel    Gaussian taps for every odd length (fp64 and fp32 copies).
 *
 * Reference arithmetic restated here (paths under /root/reference/pkg/src/foveakit/):
 * blockwise.py:39-51, tiling.py:15-39, retinal.py:97-177, filters.py:20-38,77-85,
 * blockwise.py:107-133.  The operation order of SURVEY.md Appendix A is kept, and every
 * fp64 operation is an explicitly rounded intrinsic so nothing is fused.
 */
#include <cstdlib>

#include "fk_hypot.h"
#include "fk_internal.h"

namespace {

__device__ __forceinline__ void fk_span(int extent, int F, int off, int g, int &a, int &b)
{
    /* tiling.py:21-27: starts = {0 if off > 0} U {off, off+F, ... < extent} */
    const int lead = off > 0 ? 1 : 0;
    if (lead && g == 0) {
        a = 0;
        b = off < extent ? off : extent;
    } else {
        a = off + (g - lead) * F;
        b = a + F < extent ? a + F : extent;
    }
}

__device__ __forceinline__ int fk_span_count_dev(int extent, int F, int off)
{
    int n = extent > off ? (extent - off + F - 1) / F : 0;
    return n + (off > 0 ? 1 : 0);
}

/* tiling.py:36-39: searchsorted(starts, coord, side="right") - 1, clamped.
 * starts are integers, so start <= coord  <=>  start <= floor(coord). */
__device__ __forceinline__ int fk_cell_of(int extent, int F, int off, int n, long long ic)
{
    int count = off > 0 ? 1 : 0;
    if (extent > off && ic >= off) {
        long long k = (ic - off) / F + 1;
        int n_main = (extent - off + F - 1) / F;
        count += (int)(k < n_main ? k : n_main);
    }
    int idx = count - 1;
    idx = idx < 0 ? 0 : idx;
    return idx > n - 1 ? n - 1 : idx;
}

/*
 * Turn the cells of frame f into strips and append them to the per-class work lists.
 * Called by all threads of the CTA that owns the frame; `length`, `offset` and the frame's
 * meta words must have been written by this CTA.
 *
 * Fragments up to FK_RECT wide are merged in two steps, both exact (an output pixel depends
 * only on the image and its filter):
 *   across  m = FK_RECT / F neighbouring cells of a grid row (aligned groups after the
 *           leading partial cell) become one unit FK_RECT wide: one filter when they share
 *           their taps, else a mixed item with a filter per cell (pd.mixed, fk_internal.h);
 *   down    a vertical run of equal units (same cells, same taps) is cut from its top into
 *           strips of at most pd.strip_rows / F grid rows, which lets the fragments of a
 *           strip share the horizontal pass over the 2r halo rows between them.
 * Wider fragments are cut into columns FK_RECT wide; those merge down the grid in the same
 * way (a 64-pixel fragment is two columns, each the head of its own strips), and only
 * fragments taller than FK_STRIP_ROWS are cut into pieces without merging.
 */
template <typename CT>
__device__ void fk_emit_items(const fk_plan_dev &pd, int f, int ncells, const CT *len,
                              const int32_t *off_global, CT *strip)
{
    /* len / strip: the frame's cell arrays -- 16-bit copies in the CTA's shared memory when they
     * fit (the walks below are chains of dependent loads), else the plan's global arrays.
     * off_global: the tap offsets of a caller's bank (fk_plan_set_grid), nullptr for the
     * canonical table, where the taps of radius r start at r * r. */
    auto off_of = [&](int c) -> int {
        if (off_global) return off_global[c];
        const int r = ((int)len[c] - 1) >> 1;
        return r * r;
    };
    __shared__ int ccount[2 * FK_NCLASS]; /* [0, N): front of the class lists, [N, 2N): back */
    __shared__ int cbase[2 * FK_NCLASS];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int32_t *meta = pd.meta + (size_t)f * FK_META_WORDS;
    const int sx = meta[FK_META_SX], sy = meta[FK_META_SY];
    const int gw = meta[FK_META_GW], gh = meta[FK_META_GH];
    const int F = pd.fragment;
    const bool merge = F <= FK_RECT;      /* cells of a grid row may merge across */
    const bool vmerge = pd.nsub_y == 1;   /* ... and units down the grid (always, today) */
    const int maxc = vmerge ? (pd.strip_rows / F > 1 ? pd.strip_rows / F : 1) : 1;
    const int mgrp = merge ? FK_RECT / F : 1; /* cells per horizontal unit */
    const int lead = sx > 0 ? 1 : 0;
    const int per_cell = pd.nsub_x * pd.nsub_y; /* FK_RECT-wide columns of a wider fragment */
    if (tid < 2 * FK_NCLASS) ccount[tid] = 0;
    __syncthreads();

    /* The unit [u0, u1) of grid row gy that contains cell gx, and its kind -- 0: the cell
     * alone; 1: its aligned group of mgrp cells, all with one filter; 2: the group with a filter
     * per cell (a mixed item, fk_internal.h: every cell blurred, nothing longer than the fast
     * kernels take, canonical taps). */
    auto unit_of = [&](int gy, int gx, int &u0, int &u1) -> int {
        u0 = gx;
        u1 = gx + 1;
        if (mgrp <= 1 || (lead && gx == 0)) return 0;
        const int g0 = lead + ((gx - lead) / mgrp) * mgrp;
        const int g1 = g0 + mgrp < gw ? g0 + mgrp : gw;
        if (g1 - g0 < 2) return 0;
        const CT *lr = len + gy * gw;
        const int L0 = lr[g0], o0 = off_of(gy * gw + g0);
        bool same = true;
        int lmax = 0;
        for (int x = g0; x < g1; x++) {
            if (lr[x] <= 1) return 0;
            same = same && lr[x] == L0 && off_of(gy * gw + x) == o0;
            lmax = lr[x] > lmax ? (int)lr[x] : lmax;
        }
        /* a warp's 8 pixel columns must lie in one cell: F = 8 or 16 */
        if (!same && (!pd.mixed || (F & 7) != 0 || lmax > FK_CLASS_L4)) return 0;
        u0 = g0;
        u1 = g1;
        return same ? 1 : 2;
    };
    /* Vertical runs of equal units are cut greedily from their top into strips of at most maxc
     * cells.  One thread per grid column walks its column once and records, for every cell,
     * the number of grid rows of the strip it heads (0: headed further up). */
    for (int gx = tid; gx < gw; gx += nt) {
        int head = -1, hu0 = 0, hu1 = 0, hkind = 0;
        for (int gy = 0; gy < gh; gy++) {
            const int c = gy * gw + gx;
            int u0 = gx, u1 = gx + 1, kind = 0;
            const bool mergeable = vmerge && len[c] != 1;
            if (mergeable) kind = unit_of(gy, gx, u0, u1);
            if (gx != u0) { /* inside a unit headed by the cell to its left */
                strip[c] = 0;
                head = -1;
                continue;
            }
            bool joins = mergeable && head >= 0 && gy - head < maxc && u0 == hu0 && u1 == hu1 &&
                         kind == hkind;
            for (int x = u0; joins && x < u1; x++) /* the same filter(s) as the head row */
                joins = len[gy * gw + x] == len[head * gw + x] && off_of(gy * gw + x) == off_of(head * gw + x);
            if (joins) {
                strip[c] = 0;
                strip[head * gw + gx] += 1;
            } else {
                strip[c] = 1;
                head = mergeable ? gy : -1;
                hu0 = u0;
                hu1 = u1;
                hkind = kind;
            }
        }
    }
    __syncthreads();
    /* Cell c heads a strip of n grid rows of the unit [u0, u1) of the given kind; n = 0 when the
     * cell belongs to a strip headed by another cell. */
    auto strip_of = [&](int c, int &u0, int &u1, int &kind) {
        const int gy = c / gw, gx = c - gy * gw;
        u0 = gx;
        u1 = gx + 1;
        kind = 0;
        const int n = strip[c];
        if (n > 0 && merge && len[c] != 1) kind = unit_of(gy, gx, u0, u1);
        return n;
    };
    /* longest filter of a unit, and the packed radii of a mixed one: pixel column 8 w of the
     * unit lies in cell u0 + 8 w / F (every cell of a group but the last is F wide) */
    auto unit_filters = [&](int c, int u0, int u1, int kind, int &lmax, uint32_t &toff) {
        lmax = len[c];
        toff = (uint32_t)off_of(c);
        if (kind != 2) return;
        const int gy = c / gw;
        toff = FK_ITEM_MIXED;
        for (int w = 0; w < FK_RECT / 8; w++) {
            const int x = u0 + (8 * w) / F;
            if (x >= u1) break;
            const int L = len[gy * gw + x];
            lmax = L > lmax ? L : lmax;
            toff |= (uint32_t)((L - 1) >> 1) << (6 * w);
        }
    };
    /* rectangle s of the strip headed by cell c; false when it is empty, which happens for
     * clipped fragments wider than FK_RECT */
    auto sub_rect = [&](int c, int n, int u1, int s, int &rx0, int &ry0, int &fw, int &fh) {
        const int gy = c / gw, gx = c - gy * gw;
        int x0, x1, y0, y1, t0, t1;
        fk_span(pd.width, F, sx, gx, x0, x1);
        fk_span(pd.width, F, sx, u1 - 1, t0, x1);
        fk_span(pd.height, F, sy, gy, y0, y1);
        fk_span(pd.height, F, sy, gy + n - 1, t1, y1);
        (void)t0;
        (void)t1;
        const int sby = s / pd.nsub_x, sbx = s - sby * pd.nsub_x;
        rx0 = x0 + sbx * FK_RECT;
        ry0 = y0 + sby * FK_STRIP_ROWS;
        fw = x1 - rx0;
        fh = y1 - ry0;
        fw = fw > FK_RECT ? FK_RECT : fw;
        fh = fh > FK_STRIP_ROWS ? FK_STRIP_ROWS : fh;
        return fw > 0 && fh > 0 && ry0 >= pd.y_lo && ry0 < pd.y_hi;
    };

    /* which end of its class list a strip goes to (fk_class_list, fk_internal.h): tall strips to
     * the front, so that the items the persistent CTAs draw last are short ones */
    auto list_end = [&](int L, int fh) { return L > 1 && fh <= FK_TALL_ROWS(L) ? FK_NCLASS : 0; };
    for (int c = tid; c < ncells; c += nt) {
        int u0, u1, kind, lmax;
        uint32_t toff;
        const int n = strip_of(c, u0, u1, kind);
        if (n == 0) continue;
        unit_filters(c, u0, u1, kind, lmax, toff);
        int cnt = 0, a, b2, w, h2 = 0, hh = 0;
        for (int s = 0; s < per_cell; s++)
            if (sub_rect(c, n, u1, s, a, b2, w, h2)) {
                cnt++;
                hh = h2;
            }
        if (cnt) atomicAdd(&ccount[list_end(lmax, hh) + fk_class_of(lmax)], cnt);
    }
    __syncthreads();
    if (tid < 2 * FK_NCLASS) { /* one reservation per class and end keeps a frame's items together */
        const int k = tid < FK_NCLASS ? tid : FK_COUNTER_BACK + tid - FK_NCLASS;
        cbase[tid] = ccount[tid] ? atomicAdd(&pd.counters[k], ccount[tid]) : 0;
        ccount[tid] = 0; /* becomes the running slot inside the reservation */
    }
    __syncthreads();
    for (int c = tid; c < ncells; c += nt) {
        int u0, u1, kind, L;
        uint32_t toff;
        const int n = strip_of(c, u0, u1, kind);
        if (n == 0) continue;
        unit_filters(c, u0, u1, kind, L, toff);
        const int k = fk_class_of(L);
        int cnt = 0, rx0, ry0, fw, fh = 0, hh = 0;
        for (int s = 0; s < per_cell; s++)
            if (sub_rect(c, n, u1, s, rx0, ry0, fw, fh)) {
                cnt++;
                hh = fh;
            }
        if (cnt == 0) continue;
        const int end = list_end(L, hh);
        const int slot = cbase[end + k] + atomicAdd(&ccount[end + k], cnt);
        fk_item *base = pd.items + (size_t)k * pd.items_cap;
        /* front: upwards from 0; back: downwards from items_cap - 1 */
        fk_item *dst = end ? base + (pd.items_cap - 1 - (size_t)slot) : base + slot;
        for (int s = 0; s < per_cell; s++) {
            if (!sub_rect(c, n, u1, s, rx0, ry0, fw, fh)) continue;
            fk_item it;
            it.frame = (uint32_t)f;
            it.xy = (uint32_t)rx0 | ((uint32_t)ry0 << 16);
            it.geom = (uint32_t)fw | ((uint32_t)L << 8) | ((uint32_t)fh << 21);
            it.taps_off = toff;
            *dst = it;
            dst += end ? -1 : 1;
        }
    }
}

/* Frame f as plain copies (a frame whose fixation lies outside the image). */
__device__ void fk_emit_copy_through(const fk_plan_dev &pd, int f, bool count_bad)
{
    const int W = pd.width, H = pd.height, tid = threadIdx.x;
    if (pd.y_lo > 0) return; /* the plan of a request's lower band: the upper band's plan copies the frame */
    const int ncx = (W + 254) / 255, ncy = (H + 2046) / 2047;
    if (ncx * ncy <= pd.cap) {
        __shared__ int s_base;
        if (tid == 0) {
            if (count_bad) atomicAdd(&pd.counters[FK_COUNTER_BAD], 1);
            s_base = atomicAdd(&pd.counters[FK_CLASS_COPY], ncx * ncy);
        }
        __syncthreads();
        fk_item *dst = pd.items + (size_t)FK_CLASS_COPY * pd.items_cap + s_base;
        for (int i = tid; i < ncx * ncy; i += blockDim.x) {
            const int cy = i / ncx, cx = i - cy * ncx;
            const int x0 = cx * 255, y0 = cy * 2047;
            const int fw = W - x0 < 255 ? W - x0 : 255, fh = H - y0 < 2047 ? H - y0 : 2047;
            fk_item it;
            it.frame = (uint32_t)f;
            it.xy = (uint32_t)x0 | ((uint32_t)y0 << 16);
            it.geom = (uint32_t)fw | (1u << 8) | ((uint32_t)fh << 21);
            it.taps_off = 0;
            dst[i] = it;
        }
    } else if (tid == 0 && count_bad) {
        atomicAdd(&pd.counters[FK_COUNTER_BAD], 1);
    }
}

__global__ void __launch_bounds__(FK_PLAN_THREADS_MAX)
fk_plan_kernel(fk_plan_dev pd, fk_params prm, const double *__restrict__ fix, int n_frames,
               fk_density_dev den, int cells_in_smem)
{
    extern __shared__ int16_t sm_cells[]; /* [2][cap]: length, strip (cells_in_smem) */
    __shared__ int s_lmax;
    const int f = blockIdx.x;
    if (f >= n_frames) return;
    const int tid = threadIdx.x;
    const int W = pd.width, H = pd.height, F = pd.fragment;
    const double fx = fix[2 * f], fy = fix[2 * f + 1];
    int32_t *meta = pd.meta + (size_t)f * FK_META_WORDS;
    if (pd.self_zero) { /* a one-frame plan: this CTA is the only writer of the counters */
        if (tid < FK_COUNTER_WORDS) pd.counters[tid] = 0;
        __syncthreads();
    }

    /* retinal.py:73: fixation must satisfy 0 <= fx < w and 0 <= fy < h (NaN fails) */
    if (!(fx >= 0.0 && fx < (double)W && fy >= 0.0 && fy < (double)H)) {
        /* the host raises ValueError (fk_plan_status); the frame is copied through so that
         * the output buffer is defined whatever the caller does with the error */
        if (tid < FK_META_WORDS) meta[tid] = tid == FK_META_STATUS ? 1 : 0;
        if (pd.info_out && f == 0 && tid < 9) pd.info_out[tid] = tid >= FK_META_STATUS ? 1 : 0;
        fk_emit_copy_through(pd, f, true);
        return;
    }
    const long long ifx = (long long)floor(fx), ify = (long long)floor(fy);
    int sx = 0, sy = 0;
    if (prm.use_shift == 1) { /* blockwise.py:49-51, Python's non-negative modulo */
        long long dx = (ifx - F / 2) % F, dy = (ify - F / 2) % F;
        sx = (int)(dx < 0 ? dx + F : dx);
        sy = (int)(dy < 0 ? dy + F : dy);
    } else if (prm.use_shift == 2) { /* caller-chosen tiling origin (retinal.py:159-161) */
        sx = prm.shift_x;
        sy = prm.shift_y;
    }
    const int gw = fk_span_count_dev(W, F, sx), gh = fk_span_count_dev(H, F, sy);
    const int fgx = fk_cell_of(W, F, sx, gw, ifx), fgy = fk_cell_of(H, F, sy, gh, ify);
    const int ncells = gw * gh;
    if (tid == 0) s_lmax = 1;
    __syncthreads();

    double *sigma = pd.sigma + (size_t)f * pd.cap;
    int32_t *raw = pd.raw_length + (size_t)f * pd.cap;
    int32_t *len = pd.length + (size_t)f * pd.cap;
    int32_t *off = pd.offset + (size_t)f * pd.cap;
    int lmax = 1;
    for (int c = tid; c < ncells; c += blockDim.x) {
        const int gy = c / gw, gx = c - gy * gw;
        int x0, x1, y0, y1;
        fk_span(W, F, sx, gx, x0, x1);
        fk_span(H, F, sy, gy, y0, y1);
        const double mx = __ddiv_rn((double)(x0 + x1), 2.0);          /* tiling.py:33 */
        const double my = __ddiv_rn((double)(y0 + y1), 2.0);
        double s;
        if (den.map != nullptr) {
            /* retinal.py:180-231: _map_coords, _bilinear, _density_to_sigma */
            const double mw = (double)den.map_w, mh = (double)den.map_h;
            double u = __dsub_rn(__dmul_rn(__dadd_rn(mx, 0.5), __ddiv_rn(mw, (double)W)), 0.5);
            double v = __dsub_rn(__dmul_rn(__dadd_rn(my, 0.5), __ddiv_rn(mh, (double)H)), 0.5);
            u = fmin(fmax(u, 0.0), __dsub_rn(mw, 1.0));
            v = fmin(fmax(v, 0.0), __dsub_rn(mh, 1.0));
            const int u0 = (int)floor(u), v0 = (int)floor(v);
            const int u1 = u0 + 1 < den.map_w - 1 ? u0 + 1 : den.map_w - 1;
            const int v1 = v0 + 1 < den.map_h - 1 ? v0 + 1 : den.map_h - 1;
            const double fu = __dsub_rn(u, (double)u0), fv = __dsub_rn(v, (double)v0);
            const double m00 = (double)den.map[(size_t)v0 * den.map_w + u0];
            const double m01 = (double)den.map[(size_t)v0 * den.map_w + u1];
            const double m10 = (double)den.map[(size_t)v1 * den.map_w + u0];
            const double m11 = (double)den.map[(size_t)v1 * den.map_w + u1];
            const double top = __dadd_rn(__dmul_rn(m00, __dsub_rn(1.0, fu)), __dmul_rn(m01, fu));
            const double bot = __dadd_rn(__dmul_rn(m10, __dsub_rn(1.0, fu)), __dmul_rn(m11, fu));
            const double smp = __dadd_rn(__dmul_rn(top, __dsub_rn(1.0, fv)), __dmul_rn(bot, fv));
            s = __dmul_rn(den.sigma_max, __dsub_rn(1.0, __ddiv_rn(smp, 255.0)));
        } else {
            const double d = fk_hypot(__dsub_rn(mx, fx), __dsub_rn(my, fy)); /* retinal.py:110 */
            const double e = __dmul_rn(__ddiv_rn(d, prm.d_corner), prm.e_corner); /* :112 */
            const double fdeg = __dmul_rn(                                  /* retinal.py:129 */
                __ddiv_rn(prm.e2, __dmul_rn(prm.alpha, __dadd_rn(e, prm.e2))), prm.log_inv_ct0);
            const double fpix = __ddiv_rn(__dmul_rn(0.5, fdeg), prm.fmax);  /* retinal.py:140 */
            s = __ddiv_rn(prm.strength, __dmul_rn(prm.two_pi, fpix));       /* retinal.py:155 */
        }
        sigma[c] = s;
        /* filters.py:25-26.  Non-finite or huge sigma saturates; the host rejects such
         * parameter sets before launching (SigmaField validation, retinal.py:93-94). */
        double n6 = ceil(__dmul_rn(6.0, s));
        int n = (n6 >= 1.0 && n6 < 1.0e9) ? (int)n6 : (n6 >= 1.0e9 ? 1000000001 : 1);
        if ((n & 1) == 0) n += 1;
        raw[c] = n;
        const int L = (gy == fgy && gx == fgx) ? 1 : n;                 /* blockwise.py:129 */
        len[c] = L;
        const int r = (L - 1) >> 1;
        off[c] = r * r;
        if (cells_in_smem) sm_cells[c] = (int16_t)(L < 32767 ? L : 32767);
        lmax = L > lmax ? L : lmax;
    }
    atomicMax(&s_lmax, lmax);
    __syncthreads();
    if (tid == 0) {
        meta[FK_META_SX] = sx;
        meta[FK_META_SY] = sy;
        meta[FK_META_GW] = gw;
        meta[FK_META_GH] = gh;
        meta[FK_META_FGY] = fgy;
        meta[FK_META_FGX] = fgx;
        meta[FK_META_LMAX] = s_lmax;
        meta[FK_META_STATUS] = 0;
    }
    __syncthreads();
    if (pd.info_out && f == 0) { /* the request's plan summary, straight into pinned host memory */
        if (tid < FK_META_WORDS) pd.info_out[tid] = meta[tid];
        if (tid == FK_META_WORDS) pd.info_out[tid] = 0;
        for (int c = tid; c < ncells; c += blockDim.x) pd.info_out[16 + c] = len[c];
    }
    /* filters the fast kernels cannot take anyway (> 8191 taps are rejected by the host) never
     * reach 16 bits; the model's offsets are the canonical r * r */
    if (cells_in_smem)
        fk_emit_items<int16_t>(pd, f, ncells, sm_cells, nullptr, sm_cells + pd.cap);
    else
        fk_emit_items<int32_t>(pd, f, ncells, len, nullptr, pd.strip + (size_t)f * pd.cap);
}

/* Item emission from the cell arrays of a plan: a caller-supplied grid (fk_plan_set_grid), or
 * the work lists of a planned batch once more with other settings (pd.mixed). */
__global__ void __launch_bounds__(FK_PLAN_THREADS_MAX)
fk_order_kernel(fk_plan_dev pd, int n_frames, int cells_in_smem)
{
    extern __shared__ int16_t sm_cells[];
    const int f = blockIdx.x;
    if (f >= n_frames) return;
    const int32_t *meta = pd.meta + (size_t)f * FK_META_WORDS;
    if (meta[FK_META_STATUS] != 0) {
        fk_emit_copy_through(pd, f, false);
        return;
    }
    const int ncells = meta[FK_META_GW] * meta[FK_META_GH];
    const int32_t *len = pd.length + (size_t)f * pd.cap;
    const int32_t *off = pd.canonical ? nullptr : pd.offset + (size_t)f * pd.cap;
    if (cells_in_smem) {
        for (int c = threadIdx.x; c < ncells; c += blockDim.x)
            sm_cells[c] = (int16_t)(len[c] < 32767 ? len[c] : 32767);
        __syncthreads();
        fk_emit_items<int16_t>(pd, f, ncells, sm_cells, off, sm_cells + pd.cap);
    } else {
        fk_emit_items<int32_t>(pd, f, ncells, len, off, pd.strip + (size_t)f * pd.cap);
    }
}

/* filters.py:30-38 at sigma = L/6 (filters.py:78): one CTA per odd length. */
__global__ void __launch_bounds__(128)
fk_lut_kernel(double *__restrict__ lut64, float *__restrict__ lut32, int max_length)
{
    __shared__ double part[128];
    const int r = blockIdx.x;
    const int L = 2 * r + 1;
    if (L > max_length) return;
    const int base = r * r;
    if (L == 1) {
        if (threadIdx.x == 0) { lut64[0] = 1.0; lut32[0] = 1.0f; }
        return;
    }
    const double sigma = __ddiv_rn((double)L, 6.0);
    const double denom = __dmul_rn(__dmul_rn(2.0, sigma), sigma);
    double local = 0.0;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        const double k = (double)(i - r);
        const double w = exp(-__ddiv_rn(__dmul_rn(k, k), denom));
        lut64[base + i] = w;
        local += w;
    }
    part[threadIdx.x] = local;
    __syncthreads();
    for (int s = 64; s > 0; s >>= 1) {
        if (threadIdx.x < s) part[threadIdx.x] += part[threadIdx.x + s];
        __syncthreads();
    }
    const double sum = part[0];
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        const double w = __ddiv_rn(lut64[base + i], sum);
        lut64[base + i] = w;
        lut32[base + i] = (float)w;
    }
}

} // namespace

cudaError_t fk_launch_build_lut(double *lut64, float *lut32, int max_length, cudaStream_t s)
{
    const int nr = (max_length - 1) / 2 + 1;
    fk_lut_kernel<<<nr, 128, 0, s>>>(lut64, lut32, max_length);
    return cudaGetLastError();
}

/* One CTA per frame: large CTAs while all frames fit the device in one wave (a streaming request
 * plans one frame, the headline batch 256: the cell loop is a chain of fp64 divisions per cell
 * and the emission walks are short, so threads are what shortens it), small ones for big
 * batches. */
static int plan_threads(int n_frames)
{
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            sms = 1;
    }
    static const int force = getenv("FK_PLAN_THREADS") ? atoi(getenv("FK_PLAN_THREADS")) : 0;
    if (force) return force;
    return n_frames <= 2 * sms ? FK_PLAN_THREADS_MAX : FK_PLAN_THREADS;
}

/* Dynamic shared memory for a frame's cell arrays (length, offset, strip), 0 when they do not
 * fit: the kernels then walk the plan's global arrays. */
static size_t cell_smem_bytes(const fk_plan_dev &pd)
{
    const size_t need = 2 * (size_t)pd.cap * sizeof(int16_t); /* tap counts and strip heights */
    return need <= 200 * 1024 ? need : 0;
}

cudaError_t fk_launch_plan(const fk_plan_dev &pd, const fk_params &prm, int n_frames,
                           const double *fix_dev, const fk_density_dev &den, cudaStream_t s)
{
    const size_t smem = cell_smem_bytes(pd);
    if (smem > 40 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fk_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int threads = plan_threads(n_frames);
    fk_plan_kernel<<<n_frames, threads, smem, s>>>(pd, prm, fix_dev, n_frames, den, smem != 0);
    return cudaGetLastError();
}

cudaError_t fk_launch_order(const fk_plan_dev &pd, int n_frames, cudaStream_t s)
{
    const size_t smem = cell_smem_bytes(pd);
    if (smem > 40 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fk_order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    fk_order_kernel<<<n_frames, plan_threads(n_frames), smem, s>>>(pd, n_frames, smem != 0);
    return cudaGetLastError();
}
