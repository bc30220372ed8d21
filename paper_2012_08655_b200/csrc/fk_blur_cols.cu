/*
 * fk_blur_cols.cu -- column-partitioned separable blur for RGB frames on sm_100a: fk_blur_cols
 * (buffers TMA cannot describe) and, further down, fk_blur_tma -- the hot kernel of the render
 * path, uint8 and float32 frames staged by TMA -- which shares everything after the H pass
 * with it.
 *
 * Same arithmetic as blockwise.py:136-153 (_render_cell): clamp-to-edge tile, horizontal
 * pass over every tile row into a real-valued intermediate, vertical pass, one rounding
 * (convolve.py:15), taps accumulated in ascending order in fp32 -- bit-identical to
 * fk_blur_generic and to the row-partitioned fk_blur_fast it replaces for C = 3.
 *
 * What is different is who does what.  A work item is a strip at most 32 pixels (96 floats)
 * wide with one filter (fk_internal.h); a CTA of four warps walks its items 32 tile rows at
 * a time, and WARP w OWNS THE 24 FLOAT COLUMNS [24w, 24w + 24) OF THE STRIP in both passes:
 *
 *   stage    the 32 x (96 + 6r) byte block arrives by TMA (128-byte x 32-row boxes from a
 *            16-byte aligned origin); each warp converts 8 of its rows to fp32 in the shared
 *            working tile.  [CTA barrier A: the tile is complete]
 *   H pass   lane = tile row.  One task = the warp's 24 columns of that row: 24 accumulators,
 *            the input window in a four-slot register ring refilled a chunk ahead
 *            (h_part).  The row pitch of the tile is 4 (mod 8) floats, so
 *            the 32 rows of a warp read conflict-free.  Results go to the warp's columns of
 *            the intermediate, which is stored TRANSPOSED (ring[column][row]): consecutive
 *            lanes write consecutive words.  [split barrier B: a warp arrives here and waits
 *            only before the next conversion, so the V pass absorbs the skew between warps]
 *   V pass   one task = one RGB pixel (three columns) x 8 output rows, read from the
 *            transposed intermediate with one LDS.128 per column and four rows; the warp's
 *            8 pixels x the groups of 8 rows completed by the block (4 in the steady state)
 *            are exactly one round of its 32 lanes.  Column pitch 4 (mod 8) floats:
 *            conflict-free.
 *
 * Because a warp consumes in the V pass only what it produced itself in the H pass, the
 * intermediate needs no synchronisation at all and no slack for pipelining: it is a ring of
 * 2r + 32 rows per column.  The only CTA-wide synchronisation left are the two barriers
 * around the shared tile, and between them every warp has exactly the same amount of work.
 * The next block's TMA is issued right after barrier A and lands under the H and V passes.
 * The first block of an item is cut to 2r mod 32 rows, which makes every later block complete
 * exactly four groups of 8 output rows (a full V round); that short block's H pass is packed
 * four lanes per row so that the warps left without rows skip it.
 *
 * Long filters: the working tile is what limits the CTAs per SM, so for the classes with
 * long filters the taps are walked in up to four PANELS of `pc` chunks.  Panel p needs only
 * the tile columns [12 pc p, 12 pc (p + 1) + 96 + ...), so the tile is as wide as one panel;
 * the raw bytes of the block stay in shared memory and are converted panel by panel, the 24
 * accumulators of a lane's row stay in registers across panels (same taps, same order: the
 * result does not change), and each panel costs one more pair of barriers.
 *
 * Taps are zero-padded to a multiple of 4 -- in FRONT for the V pass and for the H pass of
 * fk_blur_tma, whose first chunk skips the zeros and starts from a plain product (see
 * v_task_px), at the end for h_part; every shared-memory word a padded tap can touch holds a
 * finite value so 0 * garbage never produces a NaN.
 */
#include <cstdlib>

#include "fk_stage.cuh"

/*
 * fk_blur_tma synchronises with mbarriers only ("bytes landed", "H pass done"), which
 * compute-sanitizer's racecheck does not model.  -DFK_DEBUG_CTA_BARRIERS (python -m
 * paper_2012_08655_b200._build --debug-barriers, tools/racecheck.sh) adds a CTA barrier next
 * to each of them -- the mbarriers stay -- so that racecheck can verify everything they order
 * between threads: the item slots thread 0 publishes, the taps, the intermediate.  (What TMA
 * writes is invisible to racecheck either way.)
 */
#ifdef FK_DEBUG_CTA_BARRIERS
#define FK_DEBUG_CTA_SYNC() __syncthreads()
#else
#define FK_DEBUG_CTA_SYNC()
#endif

namespace {

constexpr int kC = 3;
constexpr int kSegF = 8 * kC;        /* float columns owned by one warp: 24 */
constexpr int kRowF = kWarps * kSegF; /* floats per strip row: 96 */

__device__ __forceinline__ float4 lds128(uint32_t addr)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}

/*
 * uint8 frames: byte -> fp32 without an arithmetic instruction.  The word (b << 16) read as a
 * float IS b * 2^-133 for every b in [0, 255]: below 2^24 the float encoding is linear
 * (the denormals and the first normal binade share one spacing), so one PRMT per byte makes
 * an exact input value.  The horizontal taps are scaled by 2^120 when a warp fetches them,
 * which puts the intermediate at 2^-13 of its true value -- every FMA rounds exactly as the
 * unscaled one does (powers of two; nothing is near under- or overflow), so the result is
 * still bit-identical to fk_blur_generic -- and the 2^13 comes back for free in the FMA that
 * adds the rounding half before the store.  float32 frames use the values as they are.
 */
constexpr float kTapScaleH = 1.329227995784916e36f; /* 2^120 */
constexpr float kOutScale = 8192.0f;                /* 2^13 */

__device__ __forceinline__ float4 bytes_to_float4_s(uint32_t w)
{
    float4 f;
    f.x = __uint_as_float(__byte_perm(w, 0u, 0x4044));
    f.y = __uint_as_float(__byte_perm(w, 0u, 0x4144));
    f.z = __uint_as_float(__byte_perm(w, 0u, 0x4244));
    f.w = __uint_as_float(__byte_perm(w, 0u, 0x4344));
    return f;
}
template <typename T> struct cols_px;
template <> struct cols_px<uint8_t> {
    static __device__ __forceinline__ float load(const uint8_t *p)
    {
        return __uint_as_float((uint32_t)__ldg(p) << 16);
    }
    static __device__ __forceinline__ float from_byte(unsigned char b)
    {
        return __uint_as_float((uint32_t)b << 16);
    }
    static __device__ __forceinline__ uint8_t store(float v)
    {
        /* convolve.py:15: clip(floor(v + 0.5), 0, 255); cvt.rmi saturates to [0, 255] */
        uint32_t u;
        asm("cvt.rmi.sat.u8.f32 %0, %1;" : "=r"(u) : "f"(fmaf(v, kOutScale, 0.5f)));
        return (uint8_t)u;
    }
};
template <> struct cols_px<float> {
    static __device__ __forceinline__ float load(const float *p) { return __ldg(p); }
    static __device__ __forceinline__ float from_byte(unsigned char b) { return (float)b; }
    static __device__ __forceinline__ float store(float v) { return v; }
};

/* One RGB pixel of a V task to the output row, if the row exists: rounded unconditionally and
 * stored under a predicate -- as a branch around the nine instructions of a row the guard
 * cost three more per row (BSSY / BRA / BSYNC), eight rows per task. */
__device__ __forceinline__ void store_px_if(bool ok, uint8_t *p, const float (&v)[kC])
{
    uint32_t a, b, c; /* convolve.py:15, as cols_px<uint8_t>::store, kept as the 32-bit cvt results */
    asm("cvt.rmi.sat.u8.f32 %0, %1;" : "=r"(a) : "f"(fmaf(v[0], kOutScale, 0.5f)));
    asm("cvt.rmi.sat.u8.f32 %0, %1;" : "=r"(b) : "f"(fmaf(v[1], kOutScale, 0.5f)));
    asm("cvt.rmi.sat.u8.f32 %0, %1;" : "=r"(c) : "f"(fmaf(v[2], kOutScale, 0.5f)));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.global.u8 [%1], %2;\n\t"
                 "@p st.global.u8 [%1+1], %3;\n\t@p st.global.u8 [%1+2], %4;\n\t}" ::"r"((uint32_t)ok),
                 "l"(p), "r"(a), "r"(b), "r"(c)
                 : "memory");
}
__device__ __forceinline__ void store_px_if(bool ok, float *p, const float (&v)[kC])
{
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.global.f32 [%1], %2;\n\t"
                 "@p st.global.f32 [%1+4], %3;\n\t@p st.global.f32 [%1+8], %4;\n\t}" ::"r"((uint32_t)ok),
                 "l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2])
                 : "memory");
}

/* convert_rows_vec (fk_stage.cuh) with the scaled conversion */
template <int NP>
__device__ __forceinline__ void convert_rows_vec_s(const uint32_t *__restrict__ rp0,
                                                   const uint32_t *__restrict__ rp1,
                                                   float4 *__restrict__ tp, int tstride4, int bsh,
                                                   const bool (&pred)[kMaxPanels - 1])
{
#pragma unroll 1
    for (int i0 = 0; i0 < kWR; i0 += 4) {
        uint32_t lo[4][NP], hi[4][NP];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int p = 0; p < NP; p++) {
                lo[i][p] = rp0[(i0 + i) * (kPanelB / 4) + p * kPanelWords];
                hi[i][p] = rp1[(i0 + i) * (kPanelB / 4) + p * kPanelWords];
            }
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int p = 0; p < NP; p++) {
                const float4 v = bytes_to_float4_s(__funnelshift_r(lo[i][p], hi[i][p], bsh));
                if (pred[p]) tp[(i0 + i) * tstride4 + 32 * p] = v;
            }
    }
}

/*
 * Horizontal task, one panel of taps: acc[j] += sum_k g[k] * in[j + 3k], j in [0, 24), for
 * one tile row.  `trow` is the shared address of the first input float of the warp's
 * columns for this panel (16-byte aligned), `wts` of the panel's first tap; nchunk chunks of
 * four taps.  Ring of four slots of 12 input values: a chunk reads slots p, p+1, p+2 and
 * refills slot p+3 -- dead since the previous chunk -- with the values the NEXT chunk needs.
 */
__device__ __forceinline__ void h_part(uint32_t trow, uint32_t wts, int nchunk,
                                       float (&acc)[kSegF])
{
    constexpr int C = kC, NW = 16 * C;
    float win[NW];
#pragma unroll
    for (int v = 0; v < 3 * C; v++) {
        const float4 x = lds128(trow + 16 * v);
        win[4 * v + 0] = x.x;
        win[4 * v + 1] = x.y;
        win[4 * v + 2] = x.z;
        win[4 * v + 3] = x.w;
    }
    uint32_t nxt = trow + 16 * 3 * C;
    float4 g4 = lds128(wts);
    uint32_t wa = wts + 16;
    auto chunk = [&](const int p) {
        const float g[4] = {g4.x, g4.y, g4.z, g4.w};
        g4 = lds128(wa); /* next chunk's taps (a quad always follows: next panel or padding) */
        wa += 16;
#pragma unroll
        for (int v = 0; v < C; v++) {
            const float4 x = lds128(nxt + 16 * v);
            const int q = (((p + 3) % 4) * C + v) * 4;
            win[q + 0] = x.x;
            win[q + 1] = x.y;
            win[q + 2] = x.z;
            win[q + 3] = x.w;
        }
        nxt += 16 * C;
#pragma unroll
        for (int t = 0; t < 4; t++) {
#pragma unroll
            for (int j = 0; j < kSegF; j++)
                acc[j] = fmaf(g[t], win[(p * 4 * C + C * t + j) % NW], acc[j]);
        }
    };
    /* one copy of the four ring phases, left after the last chunk: the kernel is bound by
     * instruction fetch as soon as its loops outgrow the instruction cache */
    for (int c = 0; c < nchunk; c += 4) {
        chunk(0);
        if (c + 1 >= nchunk) break;
        chunk(1);
        if (c + 2 >= nchunk) break;
        chunk(2);
        if (c + 3 >= nchunk) break;
        chunk(3);
    }
}

/*
 * Vertical task on the transposed intermediate: acc[j][k] = sum_t g[t] * col_k[row0 + j + t],
 * j < 8 output rows, k < 3 adjacent columns (one RGB pixel).  `col` is the shared-memory
 * address of row 0 of the first column, `cpitch` the bytes between columns; a column is a
 * ring of `cap` rows; row0 and cap are multiples of 4, so a quad of rows never straddles the
 * wrap.  Four-slot register ring of four rows per column, one LDS.128 per column a chunk
 * ahead of its use.  The four load addresses of a turn of the ring are plain offsets unless
 * the ring wraps inside the turn.
 */
__device__ __forceinline__ void v_task_px(uint32_t col, uint32_t cpitch, int row0, int cap,
                                          uint32_t wts, int nchunk, int zpad, float (&acc)[kRV][kC])
{
    float win[kC][16];
    const uint32_t end = col + 4u * (uint32_t)cap;
    auto step = [&](uint32_t x) {
        x += 16;
        return x == end ? col : x;
    };
    uint32_t a = col + 4u * (uint32_t)row0;
#pragma unroll
    for (int v = 0; v < 3; v++) {
#pragma unroll
        for (int k = 0; k < kC; k++) {
            const float4 x = lds128(a + k * cpitch);
            win[k][4 * v + 0] = x.x;
            win[k][4 * v + 1] = x.y;
            win[k][4 * v + 2] = x.z;
            win[k][4 * v + 3] = x.w;
        }
        a = step(a);
    }
    float4 g4 = lds128(wts);
    uint32_t wa = wts + 16;
    auto refill = [&](const int p, const uint32_t la) { /* ring slot p + 3 <- the quad at la */
#pragma unroll
        for (int k = 0; k < kC; k++) {
            const float4 x = lds128(la + k * cpitch);
            win[k][(4 * (p + 3) + 0) % 16] = x.x;
            win[k][(4 * (p + 3) + 1) % 16] = x.y;
            win[k][(4 * (p + 3) + 2) % 16] = x.z;
            win[k][(4 * (p + 3) + 3) % 16] = x.w;
        }
    };
    /* one chunk of four taps at ring phase p; `la` = address of the quad of rows to load */
    auto chunk = [&](const int p, const uint32_t la) {
        const float g[4] = {g4.x, g4.y, g4.z, g4.w};
        g4 = lds128(wa); /* next chunk's taps (one padding quad follows the last) */
        wa += 16;
        refill(p, la);
#pragma unroll
        for (int t = 0; t < 4; t++) {
#pragma unroll
            for (int j = 0; j < kRV; j++)
#pragma unroll
                for (int k = 0; k < kC; k++)
                    acc[j][k] = fmaf(g[t], win[k][(4 * p + t + j) % 16], acc[j][k]);
        }
    };
    /* The first chunk (ring phase 0) holds the zpad zeros the taps are padded with in FRONT
     * (3 or 1: L is odd): their FMAs are skipped and the first real tap is a plain product,
     * which is what fmaf(g, x, 0) rounds to -- no accumulator is zeroed and no zero tap is
     * ever multiplied.  The window is unchanged: the intermediate is stored zpad rows down,
     * so that the padded filter still starts on a quad of rows. */
    {
        const float g[4] = {g4.x, g4.y, g4.z, g4.w};
        g4 = lds128(wa);
        wa += 16;
        refill(0, a);
        if (zpad == 3) {
#pragma unroll
            for (int j = 0; j < kRV; j++)
#pragma unroll
                for (int k = 0; k < kC; k++) acc[j][k] = g[3] * win[k][(3 + j) % 16];
        } else {
#pragma unroll
            for (int j = 0; j < kRV; j++)
#pragma unroll
                for (int k = 0; k < kC; k++) acc[j][k] = g[1] * win[k][(1 + j) % 16];
#pragma unroll
            for (int t = 2; t < 4; t++) {
#pragma unroll
                for (int j = 0; j < kRV; j++)
#pragma unroll
                    for (int k = 0; k < kC; k++)
                        acc[j][k] = fmaf(g[t], win[k][(t + j) % 16], acc[j][k]);
            }
        }
        a = step(a);
    }
    for (int c = 1; c < nchunk; c += 4) {
        /* the four load addresses of this turn: plain offsets unless the ring wraps in it */
        uint32_t a1 = a + 16, a2 = a + 32, a3 = a + 48, an = a + 64;
        if (an >= end) {
            a1 = step(a);
            a2 = step(a1);
            a3 = step(a2);
            an = step(a3);
        }
        chunk(1, a);
        if (c + 1 >= nchunk) break;
        chunk(2, a1);
        if (c + 2 >= nchunk) break;
        chunk(3, a2);
        if (c + 3 >= nchunk) break;
        chunk(0, a3);
        a = an;
    }
}

/*
 * Rare paths of the converter, kept out of line so that neither their code nor the index
 * arithmetic the compiler would hoist for them sits in the per-block path:
 * rows that clamp at the top / bottom edge of the image (the warp's 8 rows, one at a time) ...
 */
__device__ __noinline__ void convert_rows_clamped(const uint32_t *rl, const uint32_t *rh,
                                                  float4 *tp /* lane 0's */, int tstride4, int bsh,
                                                  int nw, int lane, int row_first, int box_first,
                                                  int H)
{
#pragma unroll 1
    for (int i0 = 0; i0 < kWR; i0 += 4) { /* four rows in flight */
        int ro[4]; /* offsets of the clamped source rows relative to the warp's first box row */
#pragma unroll
        for (int i = 0; i < 4; i++)
            ro[i] = (fast_clamp(row_first + i0 + i, 0, H - 1) - box_first) * (kPanelB / 4);
#pragma unroll 1
        for (int wj = lane, o = 0; wj < nw; wj += 32, o += kPanelWords) {
            uint32_t lo[4], hi[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                lo[i] = rl[ro[i] + o];
                hi[i] = rh[ro[i] + o];
            }
#pragma unroll
            for (int i = 0; i < 4; i++)
                tp[(i0 + i) * tstride4 + wj] = bytes_to_float4_s(__funnelshift_r(lo[i], hi[i], bsh));
        }
    }
}
/* ... and tile columns left / right of the image, which repeat the edge pixel (clamp-to-edge
 * in x, blockwise.py:147), read from the raw bytes of the same row.  `trow0` is the warp's
 * first tile row shifted by the panel's first float, el / er the raw bytes of pixel 0 / W-1.
 * Both runs start on a pixel, so the channel of a lane's element advances by 32 mod 3 = 2 per
 * step of its loop. */
__device__ __noinline__ void patch_x_edges(const unsigned char *raw, float *trow0, int twp,
                                           int lane, int row_first, int box_first, int H, int nl,
                                           int nr, int tw, int el, int er, int f0, int pwz)
{
    auto raw_at = [](const unsigned char *rp, int m) {
        return __uint_as_float((uint32_t)rp[(m >> 7) * kPanelBytes + (m & (kPanelB - 1))] << 16);
    };
    const int c0 = lane % kC;
    const int lo = f0, hi = f0 + pwz; /* tile floats this panel holds */
#pragma unroll 1
    for (int i = 0; i < kWR; i++) {
        const unsigned char *rp = raw + (fast_clamp(row_first + i, 0, H - 1) - box_first) * kPanelB;
        float *trow = trow0 + i * twp;
#pragma unroll 1
        for (int side = 0; side < 2; side++) {
            const int n = (side ? nr : nl) * kC;
            if (n == 0) continue;
            const int e = side ? er : el;
            const float v0 = raw_at(rp, e), v1 = raw_at(rp, e + 1), v2 = raw_at(rp, e + 2);
            const int base = side ? tw - n : 0;
            int c = c0;
#pragma unroll 1
            for (int j = lane; j < n; j += 32) {
                const int jg = base + j;
                if (jg >= lo && jg < hi) trow[jg] = c == 0 ? v0 : (c == 1 ? v1 : v2);
                c += 2;
                c = c >= kC ? c - kC : c;
            }
        }
    }
}

/*
 * float32 frames whose tile lies inside the image in x: the warp's 8 rows are staged with
 * 128-bit loads.  Tile quad q = image floats [s0 + 4q, +4) of the row, s0 = 3 (x0 - r): the
 * aligned quad at or below it and the next one, shifted by REM = s0 mod 4 floats (a
 * compile-time choice of registers).  `g0` points at the aligned quad of tile quad 0 in image
 * row 0, `row_first` is the warp's first source row (rows clamp in y), `last` the last aligned
 * quad of an image row that may be read.
 */
constexpr int kG = 8; /* rows a lane keeps in flight while staging float32 frames */
template <int REM>
__device__ __forceinline__ void stage_rows_f32(const float *__restrict__ g0, int row_first, int H,
                                               int rowstride, int aq0, int last,
                                               float *__restrict__ tp, int twp, int lane, int nw,
                                               int nq_all)
{
#pragma unroll 1
    for (int q = lane; q < nq_all; q += 32) {
        const bool ok = q < nw;
        const bool okb = REM != 0 && ok && aq0 + q + 1 <= last;
#pragma unroll 1
        for (int i0 = 0; i0 < kWR; i0 += kG) { /* kG rows in flight */
            float4 a[kG], b[kG];
#pragma unroll
            for (int i = 0; i < kG; i++) {
                const float4 *rp = reinterpret_cast<const float4 *>(
                                       g0 + (size_t)fast_clamp(row_first + i0 + i, 0, H - 1) * rowstride) + q;
                a[i] = ok ? __ldg(rp) : make_float4(0.f, 0.f, 0.f, 0.f);
                b[i] = okb ? __ldg(rp + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int i = 0; i < kG; i++) {
                float4 v;
                if (REM == 0) v = a[i];
                if (REM == 1) v = make_float4(a[i].y, a[i].z, a[i].w, b[i].x);
                if (REM == 2) v = make_float4(a[i].z, a[i].w, b[i].x, b[i].y);
                if (REM == 3) v = make_float4(a[i].w, b[i].x, b[i].y, b[i].z);
                reinterpret_cast<float4 *>(tp + (i0 + i) * twp)[q] = v;
            }
        }
    }
}

/*
 * TMA = true : T is uint8_t and `tmap` describes the input batch as a 3-D byte tensor
 *              (W*3, H, N) with 128 x 32 x 1 boxes.
 * TMA = false: plain-load staging (float32 frames, or buffers TMA cannot describe).
 */
template <typename T, bool TMA, int MINB> /* MINB: resident CTAs per SM the register budget allows */
__global__ void __launch_bounds__(kThreads, MINB)
fk_blur_cols(const __grid_constant__ CUtensorMap tmap, fk_plan_dev pd,
             const T *__restrict__ in, T *__restrict__ out, int klass, int wts_floats, int twp,
             int npanel_max, int icap, int ipitch, int cmw, int pc, int f32vec)
{
    /* twp: pitch of the working tile (one panel wide); cmw: ints in the column map (full
     * tile width); pc: chunks of four taps per panel */
    constexpr int C = kC;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    /* layout: [raw panels][TMA barrier, 64 B][colmap][per-warp taps x 3][tile][ring] */
    unsigned char *raw = smem_raw;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + (TMA ? npanel_max * kPanelBytes : 0));
    uint64_t *hbar = bar + 1;                           /* "H pass done": one arrival per warp */
    int *next_slot = reinterpret_cast<int *>(bar + 2); /* [2] item indices drawn by thread 0 */
    int *colmap = reinterpret_cast<int *>(reinterpret_cast<unsigned char *>(bar) + 64);
    float *wts = reinterpret_cast<float *>(colmap + cmw);
    float *tile = wts + kWarps * 3 * wts_floats;
    float *ring = tile + kTB * twp; /* [kRowF columns][ipitch], icap rows used */
    const uint32_t ring_s = smem_u32(ring), tile_s = smem_u32(tile);

    const int W = pd.width, H = pd.height;
    const uint32_t row_bytes = (uint32_t)(W * kC) * (uint32_t)sizeof(T); /* bytes between image rows */
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const fk_class_list list = fk_list_of(pd, klass);
    const int n_items = list.n_items;
    /* Items are dealt dynamically: a CTA starts with items blockIdx and blockIdx + grid and
     * draws every further one from the class's cursor (zeroed before the render launches)
     * when it starts an item, two items ahead of its use, so the draw, its hand-over through
     * shared memory and the descriptor load all hide behind an item's work. */
    int *cursor = pd.counters + FK_NCLASS + klass;
    const int stride = (int)gridDim.x;
    const uint4 none = make_uint4(0u, 0u, 0u, 0u);
    auto load_item = [&](int i) {
        return i < n_items ? __ldg(reinterpret_cast<const uint4 *>(list.at(i))) : none;
    };
    /* One 32-row block of an item.  Rows: the box origin is clamped into the image so that
     * every clamped source row of the block lies inside the box.  Columns: the box starts at
     * the 16-byte boundary at or below the tile's first byte even when that lies left of the
     * image (TMA takes negative coordinates and fills what is outside with zeros), so tile
     * float j is always raw byte skew + j; the columns outside the image are patched with the
     * edge pixel after the conversion. */
    auto issue = [&](const item_geo &g, int rb) {
        const int byte0 = (g.x0 - g.r) * C;
        const int c0a = byte0 & ~15;
        const int np = (byte0 - c0a + g.tw + 4 + kPanelB - 1) / kPanelB;
        const int ys_c = fast_clamp(g.y0 - g.r + rb, 0, H - 1);
        mbar_expect_tx(bar, (uint32_t)(np * kPanelBytes));
#pragma unroll 1
        for (int p = 0; p < np; p++)
            tma_load_3d(raw + p * kPanelBytes, &tmap, bar, c0a + p * kPanelB, ys_c, g.f);
    };
    /* Zero-padded taps of an item into one of THIS WARP's two tap buffers with cp.async
     * (src-size 0 writes the zero padding).  The padding to a multiple of four goes in FRONT
     * (v_task_px skips it in its first chunk). */
    auto fill_taps = [&](const uint4 q, int slot) {
        const int L = (int)((q.z >> 8) & 0x1fffu);
        const int n = 4 * ((L + 3) >> 2) + 4;
        const int z = n - 4 - L; /* zeros in front (3 or 1), one zero quad behind */
        const float *taps = pd.taps + q.w;
        float *dst = wts + (warp * 3 + slot) * wts_floats;
        for (int i = lane; i < n; i += 32) {
            const int in_range = i >= z && i < z + L;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst + i)),
                         "l"(taps + (in_range ? i - z : 0)), "r"(in_range ? 4 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    int idx = (int)blockIdx.x, idx_nxt = idx + stride;
    uint4 q_cur = load_item(idx);
    uint4 q_nxt = load_item(idx_nxt);
    if (tid == 0) {
        if (TMA) mbar_init(bar, 1);
        mbar_init(hbar, kWarps);
    }
    /* rows of the intermediate a padded tap can reach before they have been produced must
     * hold finite values, so start from zeros */
    for (int i = tid; i < kRowF * ipitch / 4; i += kThreads)
        reinterpret_cast<float4 *>(ring)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (idx < n_items) fill_taps(q_cur, 0);
    __syncthreads();
    if (TMA && tid == 0 && idx < n_items) issue(decode_item<C>(q_cur, W), 0);

    uint32_t phase = 0, hphase = 0;
    bool hpend = false; /* an "H pass done" phase has been arrived at and not yet waited for */
    int wslot = 0;
    uint4 q_nn = none;
    int idx_nn = n_items, par = 0;
    for (; idx < n_items; idx = idx_nxt, idx_nxt = idx_nn, q_cur = q_nxt, q_nxt = q_nn, wslot ^= 1, par ^= 1) {
        if (tid == 0) next_slot[par] = 2 * stride + atomicAdd(cursor, 1); /* read after barrier A */
        const bool have_next = idx_nxt < n_items;
        const float *w_cur = wts + (warp * 3 + wslot) * wts_floats; /* taps, V pass */
        float *w_h = wts + (warp * 3 + 2) * wts_floats;             /* taps, H pass */
        /* this item's taps were requested one item ago by this warp */
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        int zpad;
        { /* the H pass's copy: padded at the END (its window loads are tied to the tile's
             16-byte grid), scaled for uint8 frames (see bytes_to_float4_s) */
            const int L = (int)((q_cur.z >> 8) & 0x1fffu);
            const int n = 4 * ((L + 3) >> 2) + 4;
            zpad = n - 4 - L;
            const float sc = sizeof(T) == 1 ? kTapScaleH : 1.0f;
            for (int i = lane; i < n; i += 32) w_h[i] = i < L ? w_cur[i + zpad] * sc : 0.0f;
            __syncwarp();
        }
        /* request the next item's: that buffer held the previous item's taps */
        if (have_next) fill_taps(q_nxt, wslot ^ 1);

        const item_geo g = decode_item<C>(q_cur, W);
        const int x0 = g.x0, y0 = g.y0, fw = g.fw, fh = g.fh, r = g.r;
        const int nchunk = g.nchunk, th = g.th, tw = g.tw, twz = g.twz;
        const size_t frame_off = (size_t)g.f * H * W * C;
        const T *src = in + frame_off;
        T *dst = out + frame_off;
        const bool vec = TMA; /* vector converter; plain-load staging goes through a column map */
        const int skew = ((x0 - r) * C) & 15;                      /* tile float 0 = raw byte skew */
        const int nl = r - x0 > 0 ? r - x0 : 0;                    /* tile pixels left of the image */
        const int nr = x0 + fw + r - W > 0 ? x0 + fw + r - W : 0; /* ... and right of it */
        const int ncol = fw * C - kSegF * warp < kSegF ? fw * C - kSegF * warp : kSegF;
        const bool active = ncol > 0; /* this warp owns columns of this item */

        if (!TMA) {
            /* clamp-to-edge by index: tile column -> element offset inside the image row.
             * Everybody is past the last barrier of the previous item, so nobody reads the old
             * map any more. */
#pragma unroll 1
            for (int j = tid; j < twz; j += kThreads) {
                int m = -1;
                if (j < tw) {
                    const int px = j / C, c = j - px * C;
                    m = fast_clamp(x0 - r + px, 0, W - 1) * C + c;
                }
                colmap[j] = m;
            }
            __syncthreads();
        }

        const int ngroups = (fh + kRV - 1) / kRV; /* groups of 8 output rows */
        /* The first block of an item is cut short so that the 2r rows of lead are absorbed
         * there: from then on every block of 32 rows completes exactly four groups of 8 output
         * rows -- one full round of the warp's lanes in the V pass.  (It moves the partial
         * block of a strip from its end to its start.) */
        const int lead = (2 * r) & (kTB - 1);
        const int n_first = lead == 0 || lead > th ? (th < kTB ? th : kTB) : lead;
        const int npan = (nchunk + pc - 1) / pc;  /* tap panels of this item */
        int vdone = 0; /* output groups rendered so far */
        int rbm = 0;   /* ring row of the first tile row of the block */
        for (int rb = 0, nrows = n_first; rb < th; rb += nrows, nrows = th - rb < kTB ? th - rb : kTB) {
            const int ys = y0 - r + rb;
            const bool mine = warp * kWR < nrows; /* this warp converts rows of this block */
            float hacc[kSegF];
#pragma unroll
            for (int j = 0; j < kSegF; j++) hacc[j] = 0.0f;
            for (int pn = 0; pn < npan; pn++) {
                const int c0 = pn * pc;
                const int nch = nchunk - c0 < pc ? nchunk - c0 : pc;
                const int f0 = 4 * C * c0;                        /* first tile float of the panel */
                const int pwz = C * (8 * g.nseg + 4 + 4 * nch);   /* floats the H tasks may touch */
                const int pval = tw - f0 < pwz ? tw - f0 : pwz;   /* of which image data */
                /* The tile is free once every warp is through the previous H pass.  That
                 * barrier is split: a warp arrives right after its H pass and waits only here,
                 * so the V pass in between absorbs whatever skew the warps have. */
                if (hpend) {
                    mbar_wait(hbar, hphase);
                    hphase ^= 1;
                    hpend = false;
                }
                if (vec && rb == 0 && npan == 1) {
                    /* the columns beyond the image data once per item, in all eight rows the
                     * warp owns whether or not the (short) first block reaches them: shared
                     * memory starts out as whatever the previous kernel left there */
                    const int nw = (pval + 3) >> 2, nq = (pwz >> 2) - nw;
                    float4 *zp = reinterpret_cast<float4 *>(tile + (warp * kWR + (lane >> 2)) * twp) + nw;
#pragma unroll 1
                    for (int q = lane & 3; q < nq; q += 4) zp[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
                if (TMA) {
                    if (pn == 0) {
                        mbar_wait(bar, phase);
                        phase ^= 1;
                    }
                    if (mine) {
                        const int ys_c = fast_clamp(ys, 0, H - 1);
                        if (vec) {
                            /* tile word wj = raw bytes [sk + 4 wj, +4): two aligned words and a
                             * funnel shift.  One column of 32 words x the warp's 8 rows per
                             * iteration: 16 loads in flight, then 8 independent conversions.
                             * Rows clamp at the top / bottom edge of the image through their
                             * offsets inside the box (lanes past the tile read other shared
                             * memory of this CTA, harmlessly). */
                            const uint32_t *raw32 = reinterpret_cast<const uint32_t *>(raw);
                            const int sk = skew + f0; /* raw byte of the panel's first float */
                            const int bsh = (sk & 3) * 8;
                            const int nw = (pval + 3) >> 2; /* quads with image data */
                            const int w00 = lane + (sk >> 2), w01 = w00 + 1;
                            /* 32 words further along the row = same place in the next panel */
                            const uint32_t *rl = raw32 + warp * kWR * (kPanelB / 4) +
                                                 (w00 >> 5) * kPanelWords + (w00 & 31);
                            const uint32_t *rh = raw32 + warp * kWR * (kPanelB / 4) +
                                                 (w01 >> 5) * kPanelWords + (w01 & 31);
                            float4 *tp = reinterpret_cast<float4 *>(tile + warp * kWR * twp) + lane;
                            if (ys >= 0 && ys + kTB <= H) {
#pragma unroll 1
                                for (int wj = lane; wj < nw; wj += 32) {
                                    uint32_t lo[kWR], hi[kWR];
#pragma unroll
                                    for (int i = 0; i < kWR; i++) {
                                        lo[i] = rl[i * (kPanelB / 4)];
                                        hi[i] = rh[i * (kPanelB / 4)];
                                    }
#pragma unroll
                                    for (int i = 0; i < kWR; i++)
                                        tp[i * (twp / 4)] =
                                            bytes_to_float4_s(__funnelshift_r(lo[i], hi[i], bsh));
                                    rl += kPanelWords;
                                    rh += kPanelWords;
                                    tp += 32;
                                }
                            } else { /* rows clamp at the top / bottom edge of the image */
                                convert_rows_clamped(rl, rh, tp - lane, twp / 4, bsh, nw, lane,
                                                     ys + warp * kWR, ys_c + warp * kWR, H);
                            }
                            /* the vector converter writes whole quads of image data only; the
                             * columns beyond, which only padded taps and discarded outputs
                             * touch, are zeroed -- once per item (above), or every time when
                             * panels of different widths share the tile */
                            if (npan > 1) {
                                const int nq = (pwz >> 2) - nw;
                                float4 *zp =
                                    reinterpret_cast<float4 *>(tile + (warp * kWR + (lane >> 2)) * twp) + nw;
#pragma unroll 1
                                for (int q = lane & 3; q < nq; q += 4)
                                    zp[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                            }
                            if (nl | nr) {
                                __syncwarp();
                                patch_x_edges(raw, tile + warp * kWR * twp - f0, twp, lane,
                                              ys + warp * kWR, ys_c, H, nl, nr, tw, skew + nl * C,
                                              skew + (W - 1 - x0 + r) * C, f0, pwz);
                            }
                        }
                    }
                } else if (mine && sizeof(T) == 4 && f32vec && nl == 0 && nr == 0) {
                    /* float32 frames, tile inside the image in x: 128-bit loads */
                    const int s0 = (x0 - r) * C + f0; /* image float of the panel's first float */
                    const float *g0 = reinterpret_cast<const float *>(src) + (s0 & ~3);
                    float *tp = tile + warp * kWR * twp;
                    const int nw = (pval + 3) >> 2, nq_all = pwz >> 2;
                    const int aq0 = s0 >> 2, last = (W * C) / 4 - 1;
                    switch (s0 & 3) {
                    case 0: stage_rows_f32<0>(g0, ys + warp * kWR, H, W * C, aq0, last, tp, twp, lane, nw, nq_all); break;
                    case 1: stage_rows_f32<1>(g0, ys + warp * kWR, H, W * C, aq0, last, tp, twp, lane, nw, nq_all); break;
                    case 2: stage_rows_f32<2>(g0, ys + warp * kWR, H, W * C, aq0, last, tp, twp, lane, nw, nq_all); break;
                    default: stage_rows_f32<3>(g0, ys + warp * kWR, H, W * C, aq0, last, tp, twp, lane, nw, nq_all); break;
                    }
                } else if (mine) {
                    /* plain loads, eight rows in flight per lane */
                    const T *grow[kWR];
#pragma unroll
                    for (int i = 0; i < kWR; i++)
                        grow[i] = src + (size_t)fast_clamp(ys + warp * kWR + i, 0, H - 1) * W * C;
                    float *tp = tile + warp * kWR * twp;
                    for (int j = lane; j < pwz; j += 32) {
                        const int m = f0 + j < twz ? colmap[f0 + j] : -1;
                        float v[kWR];
#pragma unroll
                        for (int i = 0; i < kWR; i++)
                            v[i] = m >= 0 ? cols_px<T>::load(grow[i] + m) : 0.0f;
#pragma unroll
                        for (int i = 0; i < kWR; i++) tp[i * twp + j] = v[i];
                    }
                }
                __syncthreads(); /* A: the tile holds the panel */
                if (rb == 0 && pn == 0) { /* the item after the next: index, then descriptor */
                    idx_nn = next_slot[par];
                    q_nn = load_item(idx_nn);
                }
                if (TMA && tid == 0 && pn == npan - 1) { /* the raw bytes are free */
                    const bool more = rb + nrows < th; /* next block, else the next item's first */
                    if (more || have_next) issue(decode_item<C>(more ? q_cur : q_nxt, W), more ? rb + nrows : 0);
                }
                /* horizontal pass (blockwise.py:151): lane = tile row, the warp's 24 columns.
                 * The short first block of an item (at most 24 rows, more blocks to follow, so
                 * no V pass reads these rows before the next CTA barrier) is packed instead:
                 * four adjacent lanes take the four column sets of one row, and the warps
                 * left without rows skip the pass. */
                const bool packed = rb == 0 && nrows <= 24 && nrows < th;
                const int hrow = packed ? tid >> 2 : lane;
                const int hset = packed ? tid & 3 : warp;
                const bool hdo = hrow < nrows && kSegF * hset < fw * C;
                if (hdo)
                    h_part(tile_s + 4u * (uint32_t)(hrow * twp + kSegF * hset),
                           smem_u32(w_h) + 16u * (uint32_t)c0, nch, hacc);
                if (pn == npan - 1 && hdo) {
                    int rr = rbm + hrow + zpad; /* zpad rows down: see v_task_px */
                    rr = rr >= icap ? rr - icap : rr;
                    float *rp = ring + (size_t)(kSegF * hset) * ipitch + rr;
#pragma unroll
                    for (int j = 0; j < kSegF; j++) rp[j * ipitch] = hacc[j];
                }
                if (pn < npan - 1) {
                    __syncthreads(); /* B between panels: the next conversion follows at once */
                } else {
                    __syncwarp(); /* the warp's own rows of the intermediate, before its V pass */
                    if (lane == 0) mbar_arrive(hbar);
                    hpend = true;
                }
            }
            rbm += nrows;
            while (rbm >= icap) rbm -= icap;

            /* vertical pass (blockwise.py:152) + rounding (convolve.py:15) over the output
             * groups whose 8 + 2r intermediate rows exist now */
            const int produced = rb + nrows;
            int jend = ngroups;
            if (produced < th) {
                const int avail = produced - 2 * r - kRV;
                jend = avail >= 0 ? avail / kRV + 1 : 0;
                jend = jend < ngroups ? jend : ngroups;
            }
            if (active) {
                /* one task = one RGB pixel x 8 rows; the warp's 8 pixels x the groups released
                 * by this block (4 in the steady state) = one full round of its 32 lanes */
                const int npx = ncol / C;
                const int ntask = (jend - vdone) * 8;
                for (int t = lane; t < ntask; t += 32) {
                    const int gi = vdone + (t >> 3), px = t & 7;
                    if (px < npx) {
                        int r0 = gi * kRV;
                        while (r0 >= icap) r0 -= icap;
                        float acc[kRV][C];
                        v_task_px(ring_s + 4u * (uint32_t)((kSegF * warp + C * px) * ipitch),
                                  4u * (uint32_t)ipitch, r0, icap, smem_u32(w_cur), nchunk, zpad, acc);
                        const uint64_t ob = reinterpret_cast<uint64_t>(
                            dst + ((size_t)(y0 + gi * kRV) * W + x0) * C + kSegF * warp + C * px);
#pragma unroll
                        for (int j = 0; j < kRV; j++) /* row j: one 32 x 32 -> 64-bit multiply-add */
                            store_px_if(gi * kRV + j < fh,
                                        reinterpret_cast<T *>(ob + (uint64_t)row_bytes * (uint64_t)j), acc[j]);
                    }
                }
            }
            vdone = jend;
        }
    }
}

/* =====================================================================================
 * fk_blur_tma -- RGB frames staged by TMA: the H pass reads what landed directly (uint8 below;
 * float32: h_float).
 *
 * No working tile, no conversion pass, no CTA barrier.  The batch is seen as a 4-D tensor
 * (16 bytes, 16-byte units of a row, rows, frames) and a block of tile rows lands as
 * raw[row][nq units of 16 B]: the kernel gets
 * a family of tensor maps whose boxes are 32 rows of nq units for a few odd nq, and an item
 * picks the narrowest that holds its filter (one box shape per class launch, wide enough for
 * the class's longest filter, moves 20-30 % more bytes from the L2 on float32 frames, whose
 * blocks are four times the size; boxes of fewer rows for the short first and last blocks of
 * an item were measured as well: nothing).  The row pitch 16 nq with nq odd
 * spreads lane = row reads of 128 bits over all banks.  uint8: a lane walks its row as a stream
 * of aligned 32-bit words from one address register (immediate offsets over a turn of four
 * chunks): per chunk of four taps three new words, a funnel shift each to undo the byte
 * misalignment of the tile, and one PRMT per byte into the denormal-linear fp32 encoding
 * (bytes_to_float4_s) -- all on the integer pipe, under the 96 FFMAs of the chunk.  Rows clamp
 * in y by picking the box row; columns outside the image are patched in the raw bytes (edge
 * items only, with a CTA barrier).
 * Everything after the H pass (transposed intermediate, V pass, dealing of items, taps) is
 * fk_blur_cols.  Synchronisation: per raw buffer (one or two) a `bar` (TMA bytes landed, all
 * warps wait) and an `hbar` ("H pass done", one arrival per warp; thread 0 waits for it before
 * it requests the block that goes into that buffer next).
 * ===================================================================================== */
constexpr int kQB = 16;      /* bytes per unit of a row: a chunk of 16 bytes / a quad of floats */
constexpr int kMapWidths = 6; /* box widths per launch */
/* 16-byte units of a row that a lane's stream reads for a filter of `length` taps.  uint8: 15
 * bytes of skew + 96 + 12 per chunk of taps + what the window loads ahead; float32: the last
 * warp starts at quad 18 and reads 9 + 3 per chunk of taps but the last (what the last chunk
 * loads ahead is never used and may come from whatever follows the block in shared memory). */
template <typename T> __host__ __device__ __forceinline__ int tma_units_for(int length)
{
    return sizeof(T) == 1 ? (168 + 6 * ((length - 1) >> 1) + kQB - 1) / kQB
                          : 18 + 6 + 3 * ((length + 6) >> 2);
}
struct fk_tmaps {
    CUtensorMap m[kMapWidths]; /* boxes of kTB rows x (nq - (j << nq_shift)) units */
};

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c0, int c1, int c2, int c3)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

/*
 * Horizontal task on raw bytes: acc[j] += sum_k g[k] * byte[b0 + j + 3k], j in [0, 24), for one
 * row.  `row_s` is the shared address of the row's first byte in the raw block, b0 the byte
 * of the row that is input 0 of this task.
 */
__device__ __forceinline__ void h_bytes(uint32_t row_s, int b0, uint32_t wts, int nchunk, int zpad,
                                        float (&acc)[kSegF])
{
    constexpr int C = kC, NW = 16 * C;
    float win[NW];
    /* word i of the stream lies at a + 4 i; `a` advances by 12 words per turn of four chunks */
    uint32_t a = row_s + (uint32_t)((b0 >> 2) * 4);
    const uint32_t bsh = (uint32_t)(b0 & 3) * 8u;
    auto put = [&](const int slot4, uint32_t lo, uint32_t hi) { /* four floats from one shifted word */
        const float4 f = bytes_to_float4_s(__funnelshift_r(lo, hi, bsh));
        win[slot4 + 0] = f.x;
        win[slot4 + 1] = f.y;
        win[slot4 + 2] = f.z;
        win[slot4 + 3] = f.w;
    };
    /* words 0..9: inputs 0..35 (slots 0..2); word 9 is carried as the low half of the next */
    uint32_t carry = lds32(a);
#pragma unroll
    for (int k = 0; k < 9; k++) {
        const uint32_t nx = lds32(a + 4u * (uint32_t)(k + 1));
        put(4 * k, carry, nx);
        carry = nx;
    }
    /* words 10, 11, 12: loaded a chunk ahead of their conversion */
    uint32_t n0 = lds32(a + 40), n1 = lds32(a + 44), n2 = lds32(a + 48);
    float4 g4 = lds128(wts);
    uint32_t wa = wts + 16;
    /* slot p+3 <- the three words loaded during the previous chunk, then load the next three:
     * words 13 + 3c .. 15 + 3c of the stream for chunk c, i.e. 1 + 3p' .. 3 + 3p' past the
     * turn's first word with p' = p, or 4 for p = 0 (the last chunk of a turn) */
    auto refill = [&](const int p) {
        const int q = ((p + 3) % 4) * 4 * C;
        put(q + 0, carry, n0);
        put(q + 4, n0, n1);
        put(q + 8, n1, n2);
        carry = n2;
        const uint32_t o = 4u * (uint32_t)(1 + 3 * (p == 0 ? 4 : p));
        n0 = lds32(a + o);
        n1 = lds32(a + o + 4);
        n2 = lds32(a + o + 8);
    };
    auto chunk = [&](const int p) {
        const float g[4] = {g4.x, g4.y, g4.z, g4.w};
        g4 = lds128(wa); /* next chunk's taps (one padding quad follows the last) */
        wa += 16;
        refill(p);
#pragma unroll
        for (int t = 0; t < 4; t++) {
#pragma unroll
            for (int j = 0; j < kSegF; j++)
                acc[j] = fmaf(g[t], win[(p * 4 * C + C * t + j) % NW], acc[j]);
        }
    };
    /* first chunk: the taps are padded with zpad zeros in FRONT (the stream starts 3 zpad
     * bytes early); their FMAs are skipped and the first real tap is a plain product (what
     * fmaf(g, x, 0) rounds to), so no accumulator is zeroed -- see v_task_px */
    {
        const float g[4] = {g4.x, g4.y, g4.z, g4.w};
        g4 = lds128(wa);
        wa += 16;
        refill(0);
        if (zpad == 3) {
#pragma unroll
            for (int j = 0; j < kSegF; j++) acc[j] = g[3] * win[(C * 3 + j) % NW];
        } else {
#pragma unroll
            for (int j = 0; j < kSegF; j++) acc[j] = g[1] * win[(C * 1 + j) % NW];
#pragma unroll
            for (int t = 2; t < 4; t++) {
#pragma unroll
                for (int j = 0; j < kSegF; j++) acc[j] = fmaf(g[t], win[(C * t + j) % NW], acc[j]);
            }
        }
    }
    a += 48; /* the first chunk closed turn 0 */
    for (int c = 1; c < nchunk; c += 4) {
        chunk(1);
        if (c + 1 >= nchunk) break;
        chunk(2);
        if (c + 2 >= nchunk) break;
        chunk(3);
        if (c + 3 >= nchunk) break;
        chunk(0);
        a += 48;
    }
}

/*
 * Horizontal task on float32 frames.  TMA fetches whole 16-byte quads of a row only (the
 * global address of a box must be 16-byte aligned), and a tile starts on any float: its first
 * float is 3 (x0 - r).  The residue is absorbed by the TAPS: the stream starts zf = (x0 - r)
 * mod 4 pixels left of the tile, on a pixel that is a multiple of four (a float that is a
 * multiple of 12, quad-aligned), and the filter is padded with zf zeros in front and zb at
 * the end up to a multiple of four taps.  The block lands as raw[row][quads] with stream
 * float 0 at raw float 0, so a lane's stream is one LDS.128 per quad: no shift, no conversion
 * (the row pitch is an odd number of quads: conflict-free).  Zero taps are never multiplied -- the image may hold
 * anything beyond the filter's support, and a partial first / last chunk costs what its
 * real taps cost: the first and the last chunk of a task run a copy of the chunk whose four
 * tap groups are guarded (uniform branches), the chunks in between the plain one.
 * `row_s` is the shared address of the first quad of the warp's columns in the lane's row,
 * `wts` of the padded taps, nchunk = (zf + L + zb) / 4.
 */
__device__ __forceinline__ void h_float(uint32_t row_s, uint32_t wts, int nchunk, int zf, int zb,
                                        float (&acc)[kSegF])
{
    constexpr int C = kC, NW = 16 * C;
    float win[NW];
#pragma unroll
    for (int v = 0; v < 3 * C; v++) {
        const float4 x = lds128(row_s + (uint32_t)(v * kQB));
        win[4 * v + 0] = x.x;
        win[4 * v + 1] = x.y;
        win[4 * v + 2] = x.z;
        win[4 * v + 3] = x.w;
    }
#pragma unroll
    for (int j = 0; j < kSegF; j++) acc[j] = 0.0f;
    uint32_t nxt = row_s + 3 * C * kQB;
    float4 g4 = lds128(wts);
    uint32_t wa = wts + 16;
    auto refill = [&](const int p) { /* ring slot p + 3 <- the next three quads of the row */
#pragma unroll
        for (int v = 0; v < C; v++) {
            const float4 x = lds128(nxt + (uint32_t)(v * kQB));
            const int q = (((p + 3) % 4) * C + v) * 4;
            win[q + 0] = x.x;
            win[q + 1] = x.y;
            win[q + 2] = x.z;
            win[q + 3] = x.w;
        }
        nxt += C * kQB;
    };
    auto chunk = [&](const int p) {
        const float g[4] = {g4.x, g4.y, g4.z, g4.w};
        g4 = lds128(wa); /* next chunk's taps (one padding quad follows the last) */
        wa += 16;
        refill(p);
#pragma unroll
        for (int t = 0; t < 4; t++) {
#pragma unroll
            for (int j = 0; j < kSegF; j++)
                acc[j] = fmaf(g[t], win[(p * 4 * C + C * t + j) % NW], acc[j]);
        }
    };
    auto guarded = [&](const int p, const int tlo, const int thi) { /* taps [tlo, thi) only */
        const float g[4] = {g4.x, g4.y, g4.z, g4.w};
        g4 = lds128(wa);
        wa += 16;
        refill(p);
#pragma unroll
        for (int t = 0; t < 4; t++) {
            if (t >= tlo && t < thi) {
#pragma unroll
                for (int j = 0; j < kSegF; j++)
                    acc[j] = fmaf(g[t], win[(p * 4 * C + C * t + j) % NW], acc[j]);
            }
        }
    };
    guarded(0, zf, nchunk == 1 ? 4 - zb : 4);
    if (nchunk == 1) return;
    const int nmid = nchunk - 1; /* chunks [1, nmid) are whole */
    for (int c = 1; c < nmid; c += 4) {
        chunk(1);
        if (c + 1 >= nmid) break;
        chunk(2);
        if (c + 2 >= nmid) break;
        chunk(3);
        if (c + 3 >= nmid) break;
        chunk(0);
    }
    switch (nmid & 3) { /* the last chunk, at the phase the ring has reached */
    case 0: guarded(0, 0, 4 - zb); break;
    case 1: guarded(1, 0, 4 - zb); break;
    case 2: guarded(2, 0, 4 - zb); break;
    default: guarded(3, 0, 4 - zb); break;
    }
}

/*
 * float32 frames, items at the left / right image border: clamp-to-edge in x
 * (blockwise.py:147).  TMA fills the quads outside the row with zeros; the stream floats
 * left and right of the image, which repeat the edge pixel, are fetched from global memory
 * here.  Four threads per box row; `e0` is the image float of stream float 0 (a multiple of
 * 3, so the channel of stream float j is j mod 3), `n` the stream floats that meet taps.
 */
__device__ __noinline__ void patch_x_edges_f32(unsigned char *raw, int pitch,
                                               const float *__restrict__ src, int e0, int n, int WC,
                                               int ys_c, int H, int tid)
{
    const int row = tid >> 2;
    const int gy = ys_c + row < H - 1 ? ys_c + row : H - 1;
    const float *grow = src + (size_t)gy * WC;
    float *rrow = reinterpret_cast<float *>(raw + row * pitch);
    auto put = [&](int j, int gi) { rrow[j] = __ldg(grow + gi); };
    const int nl = e0 < 0 ? (-e0 < n ? -e0 : n) : 0;
#pragma unroll 1
    for (int j = tid & 3; j < nl; j += 4) put(j, j % kC);
    int j0 = WC - e0;
    j0 = j0 < nl ? nl : j0;
#pragma unroll 1
    for (int j = j0 + (tid & 3); j < n; j += 4) put(j, WC - kC + j % kC);
}

/*
 * Filters of an item, per warp (pixel columns [8 w, 8 w + 8) of the strip): a plain item has
 * one filter; a mixed item (fk_internal.h) one per warp, its radius packed in taps_off and
 * its taps at r * r of the canonical table.
 */
__device__ __forceinline__ int warp_radius(const uint4 q, int warp)
{
    return (q.w & FK_ITEM_MIXED) ? (int)((q.w >> (6 * warp)) & 63u)
                                 : (int)(((q.z >> 8) & 0x1fffu) - 1u) >> 1;
}
__device__ __forceinline__ int warp_length(const uint4 q, int warp)
{
    return 2 * warp_radius(q, warp) + 1;
}
__device__ __forceinline__ uint32_t warp_taps_off(const uint4 q, int warp)
{
    const uint32_t r = (uint32_t)warp_radius(q, warp);
    return (q.w & FK_ITEM_MIXED) ? r * r : q.w;
}
/* First 16-byte unit of a row that the TMA box of an item fetches (g.r: the longest filter).
 * uint8: the chunk that holds the stream's first byte, 3 zpad bytes left of the tile -- in a
 * plan that may hold mixed items, three pixels left of it: every warp's stream starts 3 zpad
 * <= 9 bytes left of ITS tile, which starts at or right of the item's; float32: the quad of
 * the pixel at or below the tile's first that is a multiple of four (h_float). */
template <typename T, bool MIXED> __device__ __forceinline__ int box_unit(const item_geo &g)
{
    if (sizeof(T) != 1) return (((g.x0 - g.r) & ~3) * kC) >> 2;
    const int lead_px = MIXED ? 3 : 4 * g.nchunk - g.L;
    return ((g.x0 - g.r - lead_px) * kC) >> 4;
}

/* Three resident CTAs per SM with 167 registers beat four with 127 (27.0 k against 26.8 k
 * frames/s on the bench, 19.4 k against 18.8 k with corner fixations): at 127 the compiler
 * rematerialises addresses and constants inside the task set-up. */
/* MIXED: the plan may hold mixed items (fragments of 8 or 16 pixels); without them the per-warp
 * geometry below folds into the item's at compile time. */
template <typename T, int MINB, bool MIXED>
__global__ void __launch_bounds__(kThreads, MINB)
fk_blur_tma(const __grid_constant__ fk_tmaps tmaps, fk_plan_dev pd, const T *__restrict__ in,
            T *__restrict__ out, int klass, int wts_floats, int nq, int nq_shift, int icap, int ipitch,
            int nbuf, uint32_t icap_rcp)
{
    constexpr int C = kC;
    constexpr bool kBytes = sizeof(T) == 1;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    /* layout: [raw x nbuf: 32 rows x nq units of 16 B at most][barriers + item slots, 128 B][per-warp taps x 3][ring]
     * nq: units per row of the widest box (the class's longest filter), 1 << nq_shift: units
     * between box widths.  nbuf = 2 where a second raw buffer does not cost a resident CTA: the TMA request then
     * runs two blocks ahead of the H pass instead of one, so the first blocks of an item --
     * which have no V pass yet to hide the fetch under -- do not wait for their bytes. */
    const int raw_bytes = nq * kQB * kTB;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + nbuf * raw_bytes); /* [2] bytes landed */
    uint64_t *hbar = bar + 2;                                                   /* [2] H pass done */
    int *slot_idx = reinterpret_cast<int *>(bar + 4);                 /* [2] */
    uint4 *slot_desc = reinterpret_cast<uint4 *>(bar + 6);            /* [2], 16-byte aligned */
    int4 *cur_state = reinterpret_cast<int4 *>(bar + 10);             /* the request cursor: tile row, item, valid, buffer */
    int4 *cur_rec = reinterpret_cast<int4 *>(bar + 12);               /* [2]: what its item's requests share */
    float *wts = reinterpret_cast<float *>(reinterpret_cast<unsigned char *>(bar) + 128);
    float *ring = wts + kWarps * 3 * wts_floats;
    const uint32_t ring_s = smem_u32(ring);

    const int W = pd.width, H = pd.height;
    const uint32_t row_bytes = (uint32_t)(W * kC) * (uint32_t)sizeof(T); /* bytes between image rows */
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const fk_class_list list = fk_list_of(pd, klass);
    const int n_items = list.n_items;
    int *cursor = pd.counters + FK_NCLASS + klass;
    const int stride = (int)gridDim.x;
    const uint4 none = make_uint4(0u, 0u, 0u, 0u);
    auto load_item = [&](int i) {
        return i < n_items ? __ldg(reinterpret_cast<const uint4 *>(list.at(i))) : none;
    };
    /* Box width of an item: index into the launch's widths (0 = widest) of the narrowest one
     * that holds the units a lane's stream reads (tma_units_for, evaluated by launch_tma for the
     * class's longest filter). */
    auto width_of = [&](const item_geo &g) {
        const int j = (nq - tma_units_for<T>(g.L)) >> nq_shift;
        return j < kMapWidths - 1 ? j : kMapWidths - 1;
    };
    auto fill_taps = [&](const uint4 q, int slot) {
        const int L = MIXED ? warp_length(q, warp) : (int)((q.z >> 8) & 0x1fffu);
        const int n = 4 * ((L + 3) >> 2) + 4;
        const int z = n - 4 - L; /* zeros in front (3 or 1), one zero quad behind */
        const float *taps = pd.taps + (MIXED ? warp_taps_off(q, warp) : q.w);
        float *dst = wts + (warp * 3 + slot) * wts_floats;
        for (int i = lane; i < n; i += 32) {
            const int in_range = i >= z && i < z + L;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst + i)),
                         "l"(taps + (in_range ? i - z : 0)), "r"(in_range ? 4 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    /* Items: the first two are blockIdx and blockIdx + grid; every further one is drawn by
     * thread 0 from the class's cursor, published (index and descriptor) in shared memory one
     * item after it was drawn -- its descriptor has long arrived by then -- and picked up by
     * everybody after the first "bytes landed" wait of the following item. */
    int idx = (int)blockIdx.x, idx_nxt = idx + stride;
    uint4 q_cur = load_item(idx);
    uint4 q_nxt = load_item(idx_nxt);
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        mbar_init(hbar, kWarps);
        mbar_init(hbar + 1, kWarps);
    }
    for (int i = tid; i < kRowF * ipitch / 4; i += kThreads)
        reinterpret_cast<float4 *>(ring)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (idx < n_items) fill_taps(q_cur, 0);
    __syncthreads();

    /* The request cursor: the block to fetch next -- tile row `crb` of item number `citem` of this
     * CTA -- runs nbuf blocks ahead of the H pass, at most two items ahead of the block that is
     * handed over (every item has at least two blocks).  It lives in shared memory, because the
     * hand-over of a raw buffer ROTATES through the warps: the warp on duty waits until every
     * warp is through the buffer's H pass, and its lane 0 requests the block nbuf ahead while
     * its other lanes idle -- ~860 cycles of a ~9 300-cycle block (a chain of dependent
     * instructions issued among eleven other warps).  With warp 0 on duty at every block the
     * CTA ran at warp 0's pace and the other three warps waited for bytes 16 % of their time
     * (clock64 around the waits, profiles/README.md).  What the requests of an item share
     * -- box unit and width, frame, first tile row, tile rows, rows of the first block -- is
     * worked out once per item (cur_rec).  Order: a hand-over follows the arrivals of all warps
     * at the buffer's hbar (release / acquire), the warp on duty at the next block is one of
     * them, and the bytes a request brings are awaited through the expect_tx arrival of its
     * lane 0 -- so the cursor, and the slots thread 0 publishes drawn items in, are seen in
     * order by everybody who reads them. */
    int d_idx = n_items;
    uint4 d_q = none;
    auto cursor_to = [&](const uint4 q) {
        const item_geo g = decode_item<C>(q, W);
        const int lead = (2 * g.r) & (kTB - 1);
        const int n_first = lead == 0 || lead > g.th ? (g.th < kTB ? g.th : kTB) : lead;
        cur_rec[0] = make_int4(box_unit<T, MIXED>(g), g.y0 - g.r, g.th, n_first);
        cur_rec[1] = make_int4(g.f, width_of(g), 0, 0);
    };
    /* by lane 0 of the warp on duty; item_no_ / par_: the item of the block that is handed over */
    auto request_next = [&](int item_no_, int par_, int idx_nxt_, const uint4 &q_nxt_) {
        int4 st = *cur_state; /* crb, citem, valid, buffer */
        if (!st.z) return;
        const int4 ra = cur_rec[0], rb2 = cur_rec[1]; /* unit, first tile row, tile rows, rows of block 0; frame, width */
        const int nrows = st.x == 0 ? ra.w : (ra.z - st.x < kTB ? ra.z - st.x : kTB);
        /* the box starts at the 16-byte unit that holds the stream's first byte (possibly left of
         * the image: TMA fills what is outside with zeros) and at the first source row clamped
         * into the image */
        mbar_expect_tx(bar + st.w, (uint32_t)((nq - (rb2.y << nq_shift)) * kQB * kTB));
        tma_load_4d(smem_raw + st.w * raw_bytes, &tmaps.m[rb2.y], bar + st.w, 0, ra.x,
                    fast_clamp(ra.y + st.x, 0, H - 1), rb2.x);
        st.w ^= nbuf - 1;
        st.x += nrows;
        if (st.x >= ra.z) { /* on to the following item: the next one, or the one after it */
            st.x = 0;
            st.y++;
            const bool nxt = st.y - item_no_ == 1;
            st.z = (nxt ? idx_nxt_ : slot_idx[par_]) < n_items;
            if (st.z) cursor_to(nxt ? q_nxt_ : slot_desc[par_]);
        }
        *cur_state = st;
    };
    if (tid == 0) {
        *cur_state = make_int4(0, 0, idx < n_items, 0);
        if (idx < n_items) {
            cursor_to(q_cur);
            for (int i = 0; i < nbuf; i++) request_next(0, 0, idx_nxt, q_nxt);
            /* item 2 of this CTA: published when item 0 has its first bytes */
            d_idx = 2 * stride + atomicAdd(cursor, 1);
            d_q = load_item(d_idx);
        }
    }

    int bc = 0; /* blocks this CTA has been through: buffer bc % nbuf, its phase (bc / nbuf) & 1 */
    int wslot = 0, par = 0, item_no = 0;
    for (; idx < n_items; idx = idx_nxt, q_cur = q_nxt, wslot ^= 1, par ^= 1, item_no++) {
        const float *w_cur = wts + (warp * 3 + wslot) * wts_floats; /* taps, V pass */
        /* H pass: its own copy -- scaled by 2^120 for uint8 frames (bytes_to_float4_s);
         * padded with zf zeros in front for float32 frames (h_float) */
        float *w_h = wts + (warp * 3 + 2) * wts_floats;
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        /* Item geometry: g (and r, th, tw: the longest filter of the item) rules what the CTA
         * shares -- the TMA box, the blocks of tile rows, the clamp-to-edge patch; the warp's
         * own filter (rw, Lw: the item's, or its column's in a mixed item) rules its taps, the
         * tile rows its H pass needs -- dw fewer at either end -- and its V pass. */
        const item_geo g = decode_item<C>(q_cur, W);
        const int x0 = g.x0, y0 = g.y0, fw = g.fw, fh = g.fh, r = g.r;
        const int th = g.th, tw = g.tw;
        const int rw = MIXED ? warp_radius(q_cur, warp) : r, Lw = 2 * rw + 1, dw = r - rw;
        const int nchunk = (Lw + 3) >> 2;
        const int zpad = 4 * nchunk - Lw;                  /* zeros in front of the taps: 3 or 1 */
        const int xw = x0 + 8 * warp - rw;                 /* first tile pixel of the warp's columns */
        const int zf = kBytes ? zpad : xw & 3;             /* zero taps in front, H pass */
        const int nchunk_h = (zf + Lw + 3) >> 2;
        {
            if (kBytes) {
                const int n = Lw + zpad + 4;
                for (int i = lane; i < n; i += 32) w_h[i] = w_cur[i] * kTapScaleH;
            } else {
                const int n = 4 * nchunk_h + 4;
                for (int i = lane; i < n; i += 32)
                    w_h[i] = i >= zf && i < zf + Lw ? w_cur[i - zf + zpad] : 0.0f;
            }
            __syncwarp();
        }
        T *dst = out + (size_t)g.f * H * W * C;
        const int box0 = box_unit<T, MIXED>(g) * (kBytes ? 16 : 4); /* image element of the box's first */
        const int pitch = (nq - (width_of(g) << nq_shift)) * kQB;   /* bytes between rows of the raw block */
        /* the warp's stream (element 0 meets the first tap, padding included) inside the box */
        const int sw = (xw - zf) * C - box0;
        const int skew = (x0 - r) * C - box0;                      /* tile float 0 = raw element skew */
        const int nl = r - x0 > 0 ? r - x0 : 0;                    /* tile pixels left of the image */
        const int nr = x0 + fw + r - W > 0 ? x0 + fw + r - W : 0; /* ... and right of it */
        const int ncol = fw * C - kSegF * warp < kSegF ? fw * C - kSegF * warp : kSegF;
        const bool active = ncol > 0;
        const int thw = fh + 2 * rw;                               /* tile rows of the warp */
        const int ngroups = (fh + kRV - 1) / kRV;
        const int lead = (2 * r) & (kTB - 1);
        const int n_first = lead == 0 || lead > th ? (th < kTB ? th : kTB) : lead;
        int vdone = 0;
        int rbm = dw ? icap - dw : 0; /* ring row of tile row rb: the warp's rows start at tile row dw */
        bool have_next = idx_nxt < n_items;
        for (int rb = 0, nrows = n_first; rb < th; rb += nrows, nrows = th - rb < kTB ? th - rb : kTB) {
            const int ys = y0 - r + rb;
            const int ys_c = fast_clamp(ys, 0, H - 1);
            const int buf = bc & (nbuf - 1);
            const uint32_t phase = (uint32_t)((nbuf == 2 ? bc >> 1 : bc) & 1);
            unsigned char *raw = smem_raw + buf * raw_bytes;
            const uint32_t raw_s = smem_u32(raw);
            const int duty = bc & (kWarps - 1); /* the warp that hands this block's buffer over */
            bc++;
            mbar_wait(bar + buf, phase); /* the block's bytes have landed */
            FK_DEBUG_CTA_SYNC();
            if (rb == 0) {
                if (item_no > 0) { /* the next item, published by thread 0 during the previous one */
                    idx_nxt = slot_idx[par ^ 1];
                    q_nxt = slot_desc[par ^ 1];
                    have_next = idx_nxt < n_items;
                }
                if (have_next) fill_taps(q_nxt, wslot ^ 1);
                if (tid == 0) {
                    /* The item after the next one -- drawn an item ago, its descriptor is here --
                     * goes into this item's slot, and the one after it is drawn.  The slot is
                     * free: these bytes were requested when every warp was through a block of
                     * the previous item, hence past its own reading of the slot (one item ago)
                     * and past every hand-over that read it (two items ago). */
                    slot_idx[par] = d_idx;
                    slot_desc[par] = d_q;
                    d_idx = 2 * stride + atomicAdd(cursor, 1);
                    d_q = load_item(d_idx);
                }
            }
            if (!kBytes) {
                if (box0 < 0 || skew + tw > W * C - box0) {
                    patch_x_edges_f32(raw, pitch, reinterpret_cast<const float *>(in) + (size_t)g.f * H * W * C,
                                      box0, skew + tw, W * C, ys_c, H, tid);
                    __syncthreads();
                }
            } else if (nl | nr) {
                /* clamp-to-edge in x (blockwise.py:147): the raw bytes left and right of the
                 * image become copies of the edge pixel.  Four lanes per box row, each one
                 * 16-byte chunk at a time: the run is periodic in 3 bytes, so a chunk is four of
                 * three pre-rotated words picked by the chunk's phase, merged under a byte mask
                 * with what is there (only the chunk at the image border keeps any of it --
                 * whatever lies beyond the tile's ends meets zero taps only). */
                const int prow = warp * kWR + (lane >> 2);
                unsigned char *rowp = raw + prow * pitch;
                auto at = [&](int m) -> uint32_t { return rowp[m]; };
                auto lowbytes = [](int n) { return n >= 4 ? 0xffffffffu : n <= 0 ? 0u : (1u << (8 * n)) - 1u; };
                auto fill = [&](int e, int A, int B) { /* bytes [A, B) <- pixel at byte e */
                    const uint32_t px = at(e) | (at(e + 1) << 8) | (at(e + 2) << 16);
                    const uint32_t rot[3] = {__byte_perm(px, 0u, 0x0210), __byte_perm(px, 0u, 0x1021),
                                             __byte_perm(px, 0u, 0x2102)};
#pragma unroll 1
                    for (int q = (A >> 4) + (lane & 3); q <= (B - 1) >> 4; q += 4) {
                        const int m0 = q * 16;
                        int ph = (m0 - e) % 3; /* channel of the chunk's first byte */
                        ph = ph < 0 ? ph + 3 : ph;
                        uint4 *cp = reinterpret_cast<uint4 *>(rowp + q * kQB);
                        uint4 v = *cp;
                        uint32_t *w = &v.x;
#pragma unroll
                        for (int k = 0; k < 4; k++) {
                            int f = ph + k;
                            f = f >= 3 ? f - 3 : f;
                            const uint32_t pat = f == 0 ? rot[0] : (f == 1 ? rot[1] : rot[2]);
                            const uint32_t mask = lowbytes(B - m0 - 4 * k) & ~lowbytes(A - m0 - 4 * k);
                            w[k] = (w[k] & ~mask) | (pat & mask);
                        }
                        *cp = v;
                    }
                };
                /* the edge pixels sit on a pixel boundary of the run they feed, so e fixes the
                 * phase; the far end of either run may be rounded out to its chunk */
                if (nl) fill(skew + nl * C, (skew & ~15), skew + nl * C);
                __syncwarp(); /* in a very narrow image both runs can meet in one chunk */
                if (nr) fill(skew + (W - 1 - x0 + r) * C, skew + tw - nr * C, ((skew + tw + 15) & ~15));
                __syncthreads();
            }
            /* horizontal pass (blockwise.py:151): lane = tile row (clamped in y through the
             * box row it reads), the warp's 24 columns; the rows of the block that lie outside
             * the warp's own halo (mixed items) are left out */
            if (active && lane < nrows && rb + lane >= dw && rb + lane < th - dw) {
                float hacc[kSegF];
                const int brow = fast_clamp(ys + lane, 0, H - 1) - ys_c; /* box row */
                if (kBytes)
                    h_bytes(raw_s + (uint32_t)(brow * pitch), sw, smem_u32(w_h), nchunk, zpad, hacc);
                else
                    h_float(raw_s + (uint32_t)(brow * pitch + (sw >> 2) * kQB), smem_u32(w_h),
                            nchunk_h, zf, 4 * nchunk_h - zf - Lw, hacc);
                int rr = rbm + lane + zpad; /* zpad rows down: see v_task_px */
                rr = rr >= icap ? rr - icap : rr;
                float *rp = ring + (size_t)(kSegF * warp) * ipitch + rr;
#pragma unroll
                for (int j = 0; j < kSegF; j++) rp[j * ipitch] = hacc[j];
            }
            __syncwarp();
            FK_DEBUG_CTA_SYNC();
            if (lane == 0) mbar_arrive(hbar + buf); /* this warp is through with the raw bytes */
            if (warp == duty) {
                /* every warp is through with this buffer: request the block nbuf ahead into it */
                mbar_wait(hbar + buf, phase);
                if (lane == 0) request_next(item_no, par, idx_nxt, q_nxt);
                __syncwarp();
            }
            rbm += nrows;
            while (rbm >= icap) rbm -= icap;

            /* vertical pass (blockwise.py:152) + rounding (convolve.py:15) over the groups of
             * 8 output rows whose 8 + 2 rw intermediate rows the warp has produced */
            int produced = rb + nrows - dw;
            produced = produced > thw ? thw : produced;
            int jend = ngroups;
            if (produced < thw) {
                const int avail = produced - 2 * rw - kRV;
                jend = avail >= 0 ? avail / kRV + 1 : 0;
                jend = jend < ngroups ? jend : ngroups;
            }
            if (active) {
                const int npx = ncol / C;
                const int ntask = (jend - vdone) * 8;
                for (int t = lane; t < ntask; t += 32) {
                    const int gi = vdone + (t >> 3), px = t & 7;
                    if (px < npx) {
                        /* 8 gi mod icap by the reciprocal (exact: 8 gi * icap < 2^32) */
                        const int r0 = gi * kRV - (int)__umulhi((uint32_t)(gi * kRV), icap_rcp) * icap;
                        float acc[kRV][C];
                        v_task_px(ring_s + 4u * (uint32_t)((kSegF * warp + C * px) * ipitch),
                                  4u * (uint32_t)ipitch, r0, icap, smem_u32(w_cur), nchunk, zpad, acc);
                        const uint64_t ob = reinterpret_cast<uint64_t>(
                            dst + ((size_t)(y0 + gi * kRV) * W + x0) * C + kSegF * warp + C * px);
#pragma unroll
                        for (int j = 0; j < kRV; j++) /* row j: one 32 x 32 -> 64-bit multiply-add */
                            store_px_if(gi * kRV + j < fh,
                                        reinterpret_cast<T *>(ob + (uint64_t)row_bytes * (uint64_t)j), acc[j]);
                    }
                }
            }
            vdone = jend;
        }
    }
}

struct cols_layout {
    int wts_floats, twp, icap, ipitch, npanel, cmw, pc;
    size_t smem;
};

/* Shared-memory layout for filters up to max_length walked in `npan` tap panels. */
cols_layout cols_layout_for(int max_length, bool tma, int npan)
{
    cols_layout l;
    const int nchunk = (max_length + 3) / 4;
    const int r = (max_length - 1) / 2;
    l.pc = (nchunk + npan - 1) / npan;
    l.wts_floats = 4 * nchunk + 4; /* one zero quad after the last chunk (tap prefetch) */
    const int twz = kC * (8 * kWarps + 4 + 4 * l.pc); /* one panel */
    int twp = (twz + 3) & ~3;
    if ((twp & 7) != 4) twp += 4; /* pitch = 4 (mod 8) floats */
    l.twp = twp;
    l.cmw = tma ? 0 : (kC * (8 * kWarps + 4 + 4 * nchunk) + 3) & ~3; /* column map: plain loads only */
    /* the intermediate: the short first block of an item aligns the blocks so that the V pass
     * has consumed everything older than 2r rows when the next 32 rows are written */
    l.icap = (2 * r + kTB + 3) & ~3;
    l.ipitch = (l.icap & 7) == 4 ? l.icap : l.icap + 4; /* 4 (mod 8) floats */
    l.npanel = tma ? (15 + (kSub + 2 * r) * kC + 4 + kPanelB - 1) / kPanelB : 0;
    l.smem = (size_t)l.npanel * kPanelBytes + 64 + (size_t)l.cmw * sizeof(int) +
             ((size_t)kWarps * 3 * l.wts_floats + (size_t)kTB * twp + (size_t)kRowF * l.ipitch) *
                 sizeof(float);
    return l;
}

template <typename T, bool TMA>
cudaError_t launch_cols(fk_handle *h, const CUtensorMap &map, const fk_plan_dev &pd, int klass,
                        const void *in, void *out, int class_length, cudaStream_t s, bool *taken)
{
    *taken = false;
    const size_t max_smem = h->prop.sharedMemPerBlockOptin;
    /* two CTAs per SM when up to four tap panels make the layout fit, else one */
    const size_t per_sm = h->prop.sharedMemPerMultiprocessor;
    const size_t reserved = h->prop.reservedSharedMemPerBlock;
    const size_t two_cta = per_sm / 2 > reserved ? per_sm / 2 - reserved : 0;
    cols_layout l = cols_layout_for(class_length, TMA, 1);
    if (l.smem > two_cta) {
        for (int np = 2; np <= 4; np++) {
            const cols_layout c = cols_layout_for(class_length, TMA, np);
            if (c.smem <= two_cta) {
                l = c;
                break;
            }
        }
    }
    if (l.smem > max_smem || (TMA && l.npanel > kMaxPanels)) return cudaSuccess;
    /* layouts that fit twice on an SM at most get the instantiation with the register budget
     * of two resident CTAs (244 registers for float32 frames instead of 168 with spills:
     * +3..5 % on the float32 configs; with two CTAs everywhere it is 3 % slower) */
    const bool two = 3 * (l.smem + reserved) > per_sm;
    auto kernel = two ? fk_blur_cols<T, TMA, 2> : fk_blur_cols<T, TMA, 3>;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)l.smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, l.smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaSuccess;
    const int grid = h->prop.multiProcessorCount * occ;
    /* float32 frames can be staged with 128-bit loads when rows start on 16-byte boundaries */
    const int f32vec = sizeof(T) == 4 && ((uintptr_t)in & 15) == 0 && (pd.width * kC) % 4 == 0 &&
                       ((size_t)pd.height * pd.width * kC) % 4 == 0;
    kernel<<<grid, kThreads, l.smem, s>>>(map, pd, (const T *)in, (T *)out, klass, l.wts_floats,
                                          l.twp, l.npanel, l.icap, l.ipitch, l.cmw, l.pc, f32vec);
    *taken = true;
    return cudaGetLastError();
}

/* The batch as a 4-D tensor (16 bytes, 16-byte units of a row, rows, frames) -- uint8: 16-byte
 * chunks, float32: quads of floats -- with boxes of 16 B x nq units x `rows` rows, which land as
 * [row][nq units] in shared memory. */
template <typename T>
bool make_tensor_map_rows(CUtensorMap *map, const void *in, int W, int H, int n_frames, int nq, int rows)
{
    encode_tiled_fn enc = get_encode_tiled();
    constexpr int per_unit = kQB / (int)sizeof(T); /* elements per unit */
    const size_t row_elems = (size_t)W * kC;
    if (!enc || ((uintptr_t)in & 15) != 0 || (row_elems % per_unit) != 0 || nq > 256) return false;
    const size_t pitch = row_elems * sizeof(T);
    cuuint64_t dims[4] = {(cuuint64_t)per_unit, (cuuint64_t)(row_elems / per_unit), (cuuint64_t)H,
                          (cuuint64_t)n_frames};
    cuuint64_t strides[3] = {(cuuint64_t)kQB, (cuuint64_t)pitch, (cuuint64_t)pitch * H};
    cuuint32_t box[4] = {(cuuint32_t)per_unit, (cuuint32_t)nq, (cuuint32_t)rows, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, sizeof(T) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     4, const_cast<void *>(in), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <typename T>
cudaError_t launch_tma(fk_handle *h, const fk_plan_dev &pd, int klass, const void *in, void *out,
                       int n_frames, int class_length, cudaStream_t s, bool *taken)
{
    *taken = false;
    constexpr bool bytes = sizeof(T) == 1;
    const int nchunk = (class_length + 3) / 4;
    const int r = (class_length - 1) / 2;
    /* float32: up to three more zeros in front of the H pass's taps (h_float) */
    const int nchunk_h = bytes ? nchunk : (class_length + 6) / 4;
    const int wts_floats = 4 * nchunk_h + 4;
    /* Box widths: the widest holds the class's longest filter, the narrowest its shortest; odd
     * numbers of units, so that the rows of a block -- 16 nq bytes apart -- spread over all
     * banks when every lane reads 128 bits of its own row. */
    const int nq = tma_units_for<T>(class_length) | 1;
    const int nq_lo = tma_units_for<T>(fk_class_lmin(klass) < class_length ? fk_class_lmin(klass) : class_length);
    int nq_shift = 1; /* widths 2, 4 or 8 units apart: the narrowest box about the class's shortest filter */
    while (nq_shift < 3 && nq - ((kMapWidths - 1) << nq_shift) > nq_lo) nq_shift++;
    /* the intermediate: 2r rows the V pass still needs + the 32 of the next block.  A warp of
     * a mixed item whose filter is shorter than the item's longest is not aligned to the groups
     * of 8 output rows (up to 7 more rows wait for their group), hence 8 rows of slack */
    const bool mixed_items = pd.mixed && pd.fragment < FK_RECT && (pd.fragment & 7) == 0; /* holds_mixed_items */
    const int icap = (2 * r + kTB + (mixed_items ? 8 : 0) + 3) & ~3;
    const int ipitch = (icap & 7) == 4 ? icap : icap + 4;
    const size_t raw_bytes = (size_t)nq * kQB * kTB;
    size_t smem = raw_bytes + 128 +
                  ((size_t)kWarps * 3 * wts_floats + (size_t)kRowF * ipitch) * sizeof(float);
    if (smem > h->prop.sharedMemPerBlockOptin) return cudaSuccess;
    fk_tmaps maps;
    static_assert(sizeof(fk_tmaps) == sizeof(fk_handle::tmap_slot::maps), "tensor-map cache slot");
    fk_handle::tmap_slot &slot = h->tmap_cache[(bytes ? 0 : FK_NCLASS) + klass];
    if (slot.in == in && slot.width == pd.width && slot.height == pd.height && slot.frames == n_frames &&
        slot.nq == nq && slot.shift == nq_shift) {
        memcpy(&maps, slot.maps, sizeof maps);
    } else {
        memset(&maps, 0, sizeof maps);
        for (int j = 0; j < kMapWidths; j++) {
            const int w = nq - (j << nq_shift) > 1 ? nq - (j << nq_shift) : 1; /* never picked below nq_lo */
            if (!make_tensor_map_rows<T>(&maps.m[j], in, pd.width, pd.height, n_frames, w, kTB)) return cudaSuccess;
        }
        memcpy(slot.maps, &maps, sizeof maps);
        slot.in = in;
        slot.width = pd.width;
        slot.height = pd.height;
        slot.frames = n_frames;
        slot.nq = nq;
        slot.shift = nq_shift;
    }
    /* Layouts that fit three times on an SM run with the register budget of three resident
     * CTAs, the others with that of two. */
    const size_t per_sm = h->prop.sharedMemPerMultiprocessor;
    const size_t reserved = h->prop.reservedSharedMemPerBlock;
    const bool two = 3 * (smem + reserved) > per_sm;
    auto kernel = mixed_items ? (two ? fk_blur_tma<T, 2, true> : fk_blur_tma<T, 3, true>)
                              : (two ? fk_blur_tma<T, 2, false> : fk_blur_tma<T, 3, false>);
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaSuccess;
    /* a second raw buffer where it does not cost a resident CTA (variant 6: never) */
    int nbuf = 1;
    const size_t smem2 = smem + raw_bytes;
    if (smem2 <= h->prop.sharedMemPerBlockOptin && h->variant != 6) {
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
        if (e != cudaSuccess) return e;
        int occ2 = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, kernel, kThreads, smem2);
        if (e != cudaSuccess) return e;
        static const int force2 = getenv("FK_NBUF_FORCE") ? atoi(getenv("FK_NBUF_FORCE")) : 0;
        if (occ2 >= occ || (force2 && occ2 >= 1 && occ2 + force2 >= occ)) {
            nbuf = 2;
            smem = smem2;
            occ = occ2 < occ ? occ2 : occ;
        }
    }
    const int grid = h->prop.multiProcessorCount * occ;
    kernel<<<grid, kThreads, smem, s>>>(maps, pd, (const T *)in, (T *)out, klass, wts_floats, nq,
                                        nq_shift, icap, ipitch, nbuf,
                                        (uint32_t)((0x100000000ull + (uint32_t)icap - 1) / (uint32_t)icap));
    *taken = true;
    return cudaGetLastError();
}

} // namespace

/* Only fk_blur_tma reads mixed items (fk_internal.h); a plan holds them when it was emitted
 * with pd.mixed for fragments of 8 or 16 pixels (fk_emit_items). */
static bool holds_mixed_items(const fk_plan_dev &pd)
{
    return pd.mixed && pd.fragment < FK_RECT && (pd.fragment & 7) == 0;
}

bool fk_blur_tma_usable(const void *in, int width, int height, int is_f32)
{
    (void)height;
    if (!get_encode_tiled() || ((uintptr_t)in & 15) != 0) return false;
    const size_t row = (size_t)width * kC;
    return is_f32 ? (row & 3) == 0 : (row & 15) == 0;
}

/* Renders the items of one class list of an RGB batch.  Returns cudaSuccess with
 * *taken = false when the kernel cannot take the class (filters too long for its
 * shared-memory layout).  h->variant 2 = plain-load staging (no TMA). */
cudaError_t fk_launch_blur_cols(fk_handle *h, const fk_plan_dev &pd, int klass, const void *in,
                                void *out, int n_frames, int is_f32, int class_length,
                                cudaStream_t s, bool *taken)
{
    CUtensorMap map;
    memset(&map, 0, sizeof map);
    if (is_f32) {
        /* float32 by TMA: fk_blur_tma<float>, the H pass reads the landed floats directly
         * (variants 2 and 4: plain-load staging through fk_blur_cols) */
        if (h->variant != 2 && h->variant != 4) {
            cudaError_t e = launch_tma<float>(h, pd, klass, in, out, n_frames, class_length, s, taken);
            if (e != cudaSuccess || *taken) return e;
        }
        if (holds_mixed_items(pd)) return cudaErrorNotSupported; /* fk_render_any re-emits first */
        return launch_cols<float, false>(h, map, pd, klass, in, out, class_length, s, taken);
    }
    /* uint8 by TMA: fk_blur_tma, the kernel whose H pass reads the TMA bytes directly -- no
     * working tile, no conversion pass, no CTA barrier, 3 CTAs per SM up to 105 taps.  (Until the taps were padded in front it only won for the long filters.)
     * Variant 4: fk_blur_cols for every class, variant 5: same as the default. */
    if (h->variant == 5 || h->variant == 0 || h->variant == 6) { /* 6: one raw buffer (A/B runs) */
        cudaError_t e = launch_tma<uint8_t>(h, pd, klass, in, out, n_frames, class_length, s, taken);
        if (e != cudaSuccess || *taken) return e;
    }
    if (holds_mixed_items(pd)) return cudaErrorNotSupported; /* fk_render_any re-emits first */
    const bool tma = h->variant != 2 && make_tensor_map(&map, in, pd.width, pd.height, kC, n_frames);
    if (tma) return launch_cols<uint8_t, true>(h, map, pd, klass, in, out, class_length, s, taken);
    return launch_cols<uint8_t, false>(h, map, pd, klass, in, out, class_length, s, taken);
}
