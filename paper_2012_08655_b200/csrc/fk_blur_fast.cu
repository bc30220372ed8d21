/*
 * fk_blur_fast.cu -- register-blocked separable blur for sm_100a (the hot kernel).
 *
 * Same arithmetic as blockwise.py:136-153 (_render_cell): clamp-to-edge tile, horizontal
 * pass over every tile row into a real-valued intermediate, vertical pass, one rounding
 * (convolve.py:15).  What differs from fk_blur_generic is only how the work is laid out:
 *
 *   work items  strips at most 32 pixels wide and 256 tall with one filter each (vertical
 *               runs of same-filter fragments share the horizontal pass over the halo rows
 *               between them), taken from the plan's per-class lists (fk_internal.h) by
 *               persistent CTAs of 128 threads,
 *               item i of the list going to CTA i mod grid; the launch for a class sizes
 *               its shared memory for that class's longest filter, so short filters get
 *               more CTAs per SM.  Descriptors are prefetched two items ahead.
 *   staging     uint8 frames: the tile (rectangle + halo) is fetched 32 rows at a time by
 *               TMA (cp.async.bulk.tensor, 128-byte x 32-row boxes starting on a 16-byte
 *               boundary, zero fill outside the image) into a raw byte buffer.  Each warp
 *               converts ITS OWN 8 rows to fp32 (funnel shift + PRMT/FADD + I2F) into its
 *               private rows of the working tile and then filters them, so the 32-row
 *               blocks need no CTA-wide barrier; the last warp to leave the raw buffer
 *               issues the TMA for the next block (or for the first block of the next
 *               item), which lands while the H and V passes run.  float32 frames and
 *               buffers TMA cannot describe are staged with plain loads through a column
 *               map.  Tile row pitch = 4 (mod 8) floats so LDS.128 from 8 different rows
 *               hits 8 different bank groups.
 *   H pass      one task = 8 pixels x C channels of one tile row (8C accumulators).  The
 *               taps are walked in chunks of 4; the input window lives in 16C registers
 *               used as a four-slot ring with compile-time indices, one slot refilled by
 *               LDS.128 a whole chunk before it is read, so the inner loop is 32C FFMA
 *               per (C + 1) LDS.128 -- the FP32 pipe, not the LSU, is the limiter.
 *   V pass      one task = 8 output rows x one RGB pixel (or 4 adjacent floats for gray),
 *               same ring scheme over rows of the intermediate.  The intermediate itself
 *               is a ring of 2r + 72 rows in shared memory: the output groups whose 8 + 2r
 *               rows are complete after block b are rendered after the H pass of block
 *               b + 1, ordered by two pairs of mbarriers instead of CTA barriers, so a
 *               strip of any height needs no more shared memory than a single fragment
 *               and warps only meet at a CTA barrier once per strip.
 *
 * Taps are zero-padded to a multiple of 4; every shared-memory word a padded tap can
 * touch holds a finite value so 0 * garbage never produces a NaN.
 */
#include "fk_stage.cuh"

namespace {

/*
 * TMA = true : T is uint8_t and `tmap` describes the input batch as a 3-D byte tensor
 *              (W*C, H, N) with 128 x 32 x 1 boxes.
 * TMA = false: plain-load staging (float32 frames, or buffers TMA cannot describe).
 */
template <typename T, int C, bool TMA>
__global__ void __launch_bounds__(kThreads, 2)
fk_blur_fast(const __grid_constant__ CUtensorMap tmap, fk_plan_dev pd,
             const T *__restrict__ in, T *__restrict__ out, int klass, int wts_floats, int twp,
             int npanel_max, int icap)
{
    constexpr int SEG = 8 * C;
    constexpr int NSEG_MAX = (kSub * C + SEG - 1) / SEG; /* 4 */
    constexpr int IWP = NSEG_MAX * SEG;                   /* ring row pitch: 96 or 32 floats */
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    /* layout: [raw panels][barriers, 64 B][colmap][per-warp taps x 3][tile][ring] */
    unsigned char *raw = smem_raw;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + (TMA ? npanel_max * kPanelBytes : 0));
    int *raw_done = reinterpret_cast<int *>(bar + 1);
    uint64_t *hbar = bar + 2; /* [2] H pass of a block done by all warps (block parity) */
    uint64_t *vbar = bar + 4; /* [2] V pass of a block done by all warps */
    int *colmap = reinterpret_cast<int *>(reinterpret_cast<unsigned char *>(bar) + 64);
    float *wts = reinterpret_cast<float *>(colmap + twp);
    float *tile = wts + kWarps * 3 * wts_floats;
    float *interm = tile + kTB * twp;

    const int W = pd.width, H = pd.height;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const fk_class_list list = fk_list_of(pd, klass);
    const int n_items = list.n_items;
    const int stride = (int)gridDim.x;
    const uint4 none = make_uint4(0u, 0u, 0u, 0u);
    auto load_item = [&](int i) {
        return i < n_items ? __ldg(reinterpret_cast<const uint4 *>(list.at(i))) : none;
    };

    /* One 32-row block of an item: the box origin is clamped into the image so that every
     * clamped source row / column of the block lies inside the box. */
    auto issue = [&](const item_geo &g, int rb) {
        const int c0a = (g.xs_c * C) & ~15;
        const int ys_c = fast_clamp(g.y0 - g.r + rb, 0, H - 1);
        mbar_expect_tx(bar, (uint32_t)(g.npanel * kPanelBytes));
        for (int p = 0; p < g.npanel; p++)
            tma_load_3d(raw + p * kPanelBytes, &tmap, bar, c0a + p * kPanelB, ys_c, g.f);
    };
    /* Zero-padded taps of an item into one of THIS WARP's three tap buffers, with cp.async
     * so nobody waits for the loads (src-size 0 writes the zero padding).  Per-warp copies
     * mean no other warp has to be waited for before the taps are used. */
    auto fill_taps = [&](const uint4 q, int slot) {
        const int L = (int)((q.z >> 8) & 0x1fffu);
        const int n = 4 * ((L + 3) >> 2) + 4;
        const float *taps = pd.taps + q.w;
        float *dst = wts + (warp * 3 + slot) * wts_floats;
        for (int i = lane; i < n; i += 32) {
            const int in_range = i < L;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst + i)),
                         "l"(taps + (in_range ? i : 0)), "r"(in_range ? 4 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    int idx = (int)blockIdx.x;
    uint4 q_cur = load_item(idx);
    uint4 q_nxt = load_item(idx + stride);
    if (tid == 0) {
        if (TMA) mbar_init(bar, 1);
        mbar_init(&hbar[0], kWarps);
        mbar_init(&hbar[1], kWarps);
        mbar_init(&vbar[0], kWarps);
        mbar_init(&vbar[1], kWarps);
        *raw_done = 0;
    }
    /* the intermediate is a ring of icap rows; rows a padded tap can reach before they
     * have been produced must hold finite values, so start from zeros */
    for (int i = tid; i < icap * (IWP / 4); i += kThreads)
        reinterpret_cast<float4 *>(interm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (idx < n_items) fill_taps(q_cur, 0);
    __syncthreads();
    if (TMA && tid == 0 && idx < n_items) issue(decode_item<C>(q_cur, W), 0);

    uint32_t phase = 0;
    int wslot = 0;   /* tap buffer of the current item (0..2) */
    int nblocks = 0; /* 32-row blocks processed so far by this CTA (indexes hbar / vbar) */
    int rpos = 0;    /* ring row where the current item's first tile row goes (multiple of 4) */
    uint4 q_nn = none;
    /*
     * The items of this CTA form one stream of 32-row blocks.  Inside and across items:
     *   block B:  convert own rows -> wait vbar(B-2) -> H into the ring -> arrive hbar(B)
     *             -> wait hbar(B-1) -> V over the groups block B-1 released -> arrive vbar(B-1)
     * The ring holds 2r + 80 rows and continues across items, so H of block B only overwrites
     * rows that V of block B-2 and older were reading, a warp never waits for work it has
     * just finished itself, and there is no CTA-wide barrier on the vector path.
     */
    for (; idx < n_items; idx += stride, q_cur = q_nxt, q_nxt = q_nn, wslot = wslot == 2 ? 0 : wslot + 1) {
        q_nn = load_item(idx + 2 * stride); /* descriptor prefetch, two items ahead */
        const bool have_next = idx + stride < n_items;
        const float *w_cur = wts + (warp * 3 + wslot) * wts_floats;
        /* this item's taps were requested one item ago by this warp */
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        /* request the next item's; that buffer was last read by this warp two items ago */
        if (have_next) fill_taps(q_nxt, wslot == 2 ? 0 : wslot + 1);

        const item_geo g = decode_item<C>(q_cur, W);
        const int x0 = g.x0, y0 = g.y0, fw = g.fw, fh = g.fh, r = g.r;
        const int nchunk = g.nchunk, th = g.th, nseg = g.nseg, tw = g.tw, twz = g.twz;
        const size_t frame_off = (size_t)g.f * H * W * C;
        const T *src = in + frame_off;
        T *dst = out + frame_off;
        const bool vec = TMA && g.xin; /* vector converter, no column map */

        if (vec) {
            /* the vector converter writes whole quads up to tw only; the tile columns
             * beyond, which only padded taps and discarded outputs touch, are zeroed
             * once per item by the warp that owns the rows */
            const int q0 = (tw + 3) >> 2, nq = (twz >> 2) - q0;
            for (int i = lane; i < nq * kWR; i += 32) {
                const int row = i / nq, q = i - row * nq;
                reinterpret_cast<float4 *>(tile + (warp * kWR + row) * twp)[q0 + q] =
                    make_float4(0.f, 0.f, 0.f, 0.f);
            }
            __syncwarp();
        } else {
            /* clamp-to-edge by index.  TMA: tile column -> byte offset inside the box;
             * plain loads: tile column -> element offset inside the image row.  The map is
             * shared by the CTA: one barrier so nobody still reads the previous one, one so
             * everybody sees the new one. */
            __syncthreads();
            for (int j = tid; j < twz; j += kThreads) {
                int m = -1;
                if (j < tw) {
                    const int px = j / C, c = j - px * C;
                    const int xx = fast_clamp(x0 - r + px, 0, W - 1);
                    if (TMA) {
                        m = g.skew + (xx - g.xs_c) * C + c;
                        m = (m >> 7) * kPanelBytes + (m & (kPanelB - 1));
                    } else {
                        m = xx * C + c;
                    }
                }
                colmap[j] = m;
            }
            __syncthreads();
        }

        const int ngroups = (fh + kRV - 1) / kRV; /* groups of 8 output rows */
        const int ncg = (fw * C + 3) >> 2;        /* quads of output floats per row */
        const bool wide = (fw * C) % 4 == 0;
        int jdone = 0, rbm = rpos;                /* groups released; ring row of block start */
        int pend_b = 0, pend_e = 0;               /* groups released by the previous block */
        auto ring_row = [&](int k) { /* ring position of this item's tile row k */
            int p = rpos + k;
            while (p >= icap) p -= icap;
            return p;
        };
        /* vertical pass (blockwise.py:152) + rounding (convolve.py:15) over output groups
         * [jb, je): 8 output rows each, read from the ring */
        auto v_groups = [&](int jb, int je) {
            if (C == 3) {
                /* one task = one RGB pixel x 8 rows: a warp per group, a lane per pixel */
                const int ntask = (je - jb) * 32;
                for (int task = tid; task < ntask; task += kThreads) {
                    const int rg = jb + (task >> 5), px = task & 31;
                    if (px < fw) {
                        float acc[kRV][3];
                        v_task<3>(interm + px * 3, IWP, ring_row(rg * kRV), icap, w_cur, nchunk, acc);
                        T *orow = dst + ((size_t)(y0 + rg * kRV) * W + x0 + px) * 3;
#pragma unroll
                        for (int j = 0; j < kRV; j++) {
                            if (rg * kRV + j < fh) {
#pragma unroll
                                for (int i = 0; i < 3; i++) orow[i] = fast_px<T>::store(acc[j][i]);
                            }
                            orow += (size_t)W * 3;
                        }
                    }
                }
            } else {
                const int ntask = (je - jb) * ncg;
                for (int task = tid; task < ntask; task += kThreads) {
                    const int rg = jb + task / ncg, cg = task % ncg;
                    float acc[kRV][4];
                    v_task<4>(interm + cg * 4, IWP, ring_row(rg * kRV), icap, w_cur, nchunk, acc);
                    T *orow = dst + ((size_t)(y0 + rg * kRV) * W + x0) * C + cg * 4;
#pragma unroll
                    for (int j = 0; j < kRV; j++) {
                        if (rg * kRV + j < fh) {
#pragma unroll
                            for (int i = 0; i < 4; i++)
                                if (wide || cg * 4 + i < fw * C)
                                    orow[i] = fast_px<T>::store(acc[j][i]);
                        }
                        orow += (size_t)W * C;
                    }
                }
            }
        };
        const int nblk = (th + kTB - 1) / kTB;
        for (int b = 0; b <= nblk; b++) { /* iteration nblk only drains the last V groups */
            const int rb = b * kTB;
            int new_b = jdone, new_e = jdone;
            if (b < nblk) {
            const int nrows = th - rb < kTB ? th - rb : kTB;
            const int ys = y0 - r + rb;
            const bool mine = warp * kWR < nrows; /* this warp owns rows of this block */
            if (TMA) {
                mbar_wait(bar, phase);
                phase ^= 1;
                if (mine) {
                    const int ys_c = fast_clamp(ys, 0, H - 1);
                    if (vec) {
                        const uint32_t *raw32 = reinterpret_cast<const uint32_t *>(raw);
                        const int bsh = (g.skew & 3) * 8;
                        const int w0 = lane + (g.skew >> 2), w1 = w0 + 1;
                        const int i0 = (w0 >> 5) * kPanelWords + (w0 & 31);
                        const int i1 = (w1 >> 5) * kPanelWords + (w1 & 31);
                        const int nw = (tw + 3) >> 2;
                        const int np = (nw + 31) >> 5;
                        bool pred[kMaxPanels - 1];
#pragma unroll
                        for (int p = 0; p < kMaxPanels - 1; p++) pred[p] = lane + 32 * p < nw;
                        float4 *tp = reinterpret_cast<float4 *>(tile + warp * kWR * twp) + lane;
                        if (ys >= 0 && ys + kTB <= H) {
                            const uint32_t *rp0 = raw32 + warp * kWR * (kPanelB / 4) + i0;
                            const uint32_t *rp1 = raw32 + warp * kWR * (kPanelB / 4) + i1;
                            switch (np) {
                            case 1: convert_rows_vec<1>(rp0, rp1, tp, twp / 4, bsh, pred); break;
                            case 2: convert_rows_vec<2>(rp0, rp1, tp, twp / 4, bsh, pred); break;
                            case 3: convert_rows_vec<3>(rp0, rp1, tp, twp / 4, bsh, pred); break;
                            default: convert_rows_vec<4>(rp0, rp1, tp, twp / 4, bsh, pred); break;
                            }
                        } else { /* rows clamp at the top / bottom edge of the image */
                            for (int i = 0; i < kWR; i++) {
                                const int rr = fast_clamp(ys + warp * kWR + i, 0, H - 1) - ys_c;
                                const uint32_t *rp = raw32 + rr * (kPanelB / 4);
#pragma unroll
                                for (int p = 0; p < kMaxPanels - 1; p++) {
                                    if (pred[p]) {
                                        const uint32_t lo = rp[i0 + p * kPanelWords];
                                        const uint32_t hi = rp[i1 + p * kPanelWords];
                                        tp[32 * p] = bytes_to_float4(__funnelshift_r(lo, hi, bsh));
                                    }
                                }
                                tp += twp / 4;
                            }
                        }
                    } else {
                        for (int i = 0; i < kWR; i++) {
                            const int rr = fast_clamp(ys + warp * kWR + i, 0, H - 1) - ys_c;
                            const unsigned char *rp = raw + rr * kPanelB;
                            float *tp = tile + (warp * kWR + i) * twp;
                            for (int j = lane; j < twz; j += 32) {
                                const int m = colmap[j];
                                tp[j] = m >= 0 ? (float)rp[m] : 0.0f;
                            }
                        }
                    }
                }
                __syncwarp();
                /* this warp is done with the raw bytes; the last one out refills them with
                 * the next 32 rows, or with the first rows of the next item */
                if (lane == 0) {
                    if (atomicAdd(raw_done, 1) == kWarps - 1) {
                        *raw_done = 0;
                        if (rb + kTB < th)
                            issue(g, rb + kTB);
                        else if (have_next)
                            issue(decode_item<C>(q_nxt, W), 0);
                    }
                }
            } else if (mine) {
                /* plain loads, eight rows in flight per lane */
                const T *grow[kWR];
#pragma unroll
                for (int i = 0; i < kWR; i++)
                    grow[i] = src + (size_t)fast_clamp(ys + warp * kWR + i, 0, H - 1) * W * C;
                float *tp = tile + warp * kWR * twp;
                for (int j = lane; j < twz; j += 32) {
                    const int m = colmap[j];
                    float v[kWR];
#pragma unroll
                    for (int i = 0; i < kWR; i++) v[i] = m >= 0 ? fast_px<T>::load(grow[i] + m) : 0.0f;
#pragma unroll
                    for (int i = 0; i < kWR; i++) tp[i * twp + j] = v[i];
                }
                __syncwarp();
            }
            /* H of this block overwrites ring rows last read by V of block B-2 */
            if (nblocks + b >= 2)
                mbar_wait(&vbar[(nblocks + b - 2) & 1], ((nblocks + b - 2) >> 1) & 1);
            /* horizontal pass over this warp's rows (blockwise.py:151) into the ring */
            if (mine) {
                for (int task = lane; task < kWR * nseg; task += 32) {
                    const int row = warp * kWR + (nseg == 4 ? task >> 2 : task / nseg);
                    const int seg = nseg == 4 ? task & 3 : task % nseg;
                    if (row < nrows) {
                        int rr = rbm + row;
                        rr = rr >= icap ? rr - icap : rr;
                        h_task<C>(tile + row * twp + seg * SEG, w_cur, nchunk,
                                  interm + (size_t)rr * IWP + seg * SEG);
                    }
                }
            }
            __syncwarp(); /* the next block's conversion overwrites this warp's tile rows */
            if (lane == 0) mbar_arrive(&hbar[(nblocks + b) & 1]);
            rbm += kTB;
            rbm = rbm >= icap ? rbm - icap : rbm;

            /* groups of 8 output rows whose 8 + 2r intermediate rows exist after this block */
            const int produced = rb + nrows;
            int jend = ngroups;
            if (produced < th) {
                const int avail = produced - 2 * r - kRV;
                jend = avail >= 0 ? avail / kRV + 1 : 0;
                jend = jend < ngroups ? jend : ngroups;
            }
            new_e = jend;
            jdone = jend;
            } /* b < nblk */
            if (b >= 1) { /* render what the PREVIOUS block released */
                mbar_wait(&hbar[(nblocks + b - 1) & 1], ((nblocks + b - 1) >> 1) & 1);
                v_groups(pend_b, pend_e);
                __syncwarp();
                if (lane == 0) mbar_arrive(&vbar[(nblocks + b - 1) & 1]);
            }
            pend_b = new_b;
            pend_e = new_e;
        }
        nblocks += nblk;
        rpos = (ring_row(th) + 3) & ~3; /* the next item continues the ring */
        rpos = rpos >= icap ? rpos - icap : rpos;
    }
}

struct fast_layout {
    int wts_floats, twp, irows, npanel;
    size_t smem;
};

template <int C> fast_layout fast_layout_for(int max_length, bool tma)
{
    constexpr int SEG = 8 * C;
    constexpr int NSEG = (kSub * C + SEG - 1) / SEG;
    constexpr int IWP = NSEG * SEG;
    fast_layout l;
    const int nchunk = (max_length + 3) / 4;
    l.wts_floats = 4 * nchunk + 4; /* one zero quad after the last chunk (tap prefetch) */
    const int twz = C * (8 * NSEG + 4 + 4 * nchunk);
    int twp = (twz + 3) & ~3;
    if ((twp & 7) != 4) twp += 4; /* pitch = 4 (mod 8) floats */
    l.twp = twp;
    /* ring of intermediate rows: 2r + 80 lets a block of 32 new rows -- of this strip or of
     * the next one -- be written while the previous block's output groups are still being
     * rendered (multiple of 4) */
    l.irows = (2 * ((max_length - 1) / 2) + 80 + 3) & ~3;
    l.npanel = tma ? (15 + (kSub + 2 * ((max_length - 1) / 2)) * C + 4 + kPanelB - 1) / kPanelB : 0;
    l.smem = (size_t)l.npanel * kPanelBytes + 64 + (size_t)twp * sizeof(int) +
             ((size_t)kWarps * 3 * l.wts_floats + (size_t)kTB * twp + (size_t)l.irows * IWP) *
                 sizeof(float);
    return l;
}

template <typename T, int C, bool TMA>
cudaError_t launch_fast(fk_handle *h, const CUtensorMap &map, const fk_plan_dev &pd, int klass,
                        const void *in, void *out, int class_length, cudaStream_t s, bool *taken)
{
    const fast_layout l = fast_layout_for<C>(class_length, TMA);
    *taken = false;
    const size_t max_smem = h->prop.sharedMemPerBlockOptin;
    if (l.smem > max_smem || (TMA && l.npanel > kMaxPanels)) return cudaSuccess;
    auto kernel = fk_blur_fast<T, C, TMA>;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)l.smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, l.smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaSuccess;
    const int grid = h->prop.multiProcessorCount * occ;
    kernel<<<grid, kThreads, l.smem, s>>>(map, pd, (const T *)in, (T *)out, klass, l.wts_floats,
                                          l.twp, l.npanel, l.irows);
    *taken = true;
    return cudaGetLastError();
}

} // namespace

/* Renders the items of one class list.  Returns cudaSuccess with *taken = false when the
 * fast kernel cannot take the class (filters too long for its shared-memory layout).
 * h->variant: 0 auto, 2 = fast kernel with plain-load staging (no TMA). */
cudaError_t fk_launch_blur_fast(fk_handle *h, const fk_plan_dev &pd, int klass, const void *in,
                                void *out, int n_frames, int channels, int is_f32,
                                int class_length, cudaStream_t s, bool *taken)
{
    CUtensorMap map;
    memset(&map, 0, sizeof map);
    if (is_f32) {
        if (channels == 3)
            return launch_fast<float, 3, false>(h, map, pd, klass, in, out, class_length, s, taken);
        return launch_fast<float, 1, false>(h, map, pd, klass, in, out, class_length, s, taken);
    }
    const bool tma = h->variant != 2 &&
                     make_tensor_map(&map, in, pd.width, pd.height, channels, n_frames);
    if (channels == 3) {
        if (tma)
            return launch_fast<uint8_t, 3, true>(h, map, pd, klass, in, out, class_length, s, taken);
        return launch_fast<uint8_t, 3, false>(h, map, pd, klass, in, out, class_length, s, taken);
    }
    if (tma)
        return launch_fast<uint8_t, 1, true>(h, map, pd, klass, in, out, class_length, s, taken);
    return launch_fast<uint8_t, 1, false>(h, map, pd, klass, in, out, class_length, s, taken);
}
