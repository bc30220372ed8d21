/*
 * fk_stage.cuh -- pieces shared by the two fast blur kernels (fk_blur_fast.cu, the
 * row-partitioned kernel still used for gray images, and fk_blur_cols.cu, the
 * column-partitioned kernel for RGB): tile geometry, TMA / mbarrier plumbing, the
 * byte -> fp32 converter and the register-blocked horizontal and vertical tasks.
 * Everything lives in an anonymous namespace: each translation unit gets its own copy.
 */
#ifndef FK_STAGE_CUH_
#define FK_STAGE_CUH_

#include <cuda.h>

#include "fk_internal.h"

namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kTB = 32;        /* tile rows staged per block */
constexpr int kWR = kTB / kWarps; /* tile rows owned by one warp: 8 */
constexpr int kRV = 8;         /* output rows per V task */
constexpr int kSub = FK_RECT;  /* rectangle edge */
constexpr int kPanelB = 128;   /* TMA box: bytes per row */
constexpr int kPanelBytes = kPanelB * kTB;
constexpr int kPanelWords = kPanelBytes / 4;
constexpr int kMaxPanels = 5;  /* (15 + twz + 4) / 128 for the longest fast-path filter */

template <typename T> struct fast_px;
template <> struct fast_px<uint8_t> {
    static __device__ __forceinline__ float load(const uint8_t *p) { return (float)__ldg(p); }
    static __device__ __forceinline__ uint8_t store(float v)
    {
        /* convolve.py:15: clip(floor(v + 0.5), 0, 255); cvt.rmi saturates to [0, 255] */
        uint32_t u;
        asm("cvt.rmi.sat.u8.f32 %0, %1;" : "=r"(u) : "f"(v + 0.5f));
        return (uint8_t)u;
    }
};
template <> struct fast_px<float> {
    static __device__ __forceinline__ float load(const float *p) { return __ldg(p); }
    static __device__ __forceinline__ float store(float v) { return v; }
};

__device__ __forceinline__ int fast_clamp(int v, int lo, int hi)
{
    return v < lo ? lo : (v > hi ? hi : v);
}

/* ---- TMA / mbarrier plumbing (PTX; SASS: UTMALDG, SYNCS) ------------------------- */
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_LOOP:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@p bra WAIT_DONE;\n\t"
        "bra WAIT_LOOP;\n\t"
        "WAIT_DONE:\n\t"
        "}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u) /* suspend-time hint: sleep in the barrier unit rather than
                                        spin (no measured difference on the bench) */
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c0, int c1, int c2)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

/* Four bytes of a word to four floats, exactly.  Two go through PRMT into the mantissa of
 * 2^23 + FADD (ALU + FMA pipes), two through I2F.U8 with a byte selector (conversion pipe),
 * so neither pipe is the limiter and the pass costs 6 issue slots per word. */
__device__ __forceinline__ float4 bytes_to_float4(uint32_t w)
{
    float4 f;
    f.x = __uint_as_float(__byte_perm(w, 0x4b000000u, 0x7440)) - 8388608.0f;
    f.y = (float)((w >> 8) & 0xffu);
    f.z = __uint_as_float(__byte_perm(w, 0x4b000000u, 0x7442)) - 8388608.0f;
    f.w = (float)(w >> 24);
    return f;
}

/*
 * Vector converter for one warp's kWR rows of a block whose rows need no clamping: tile
 * word wj = raw bytes [skew + 4 wj, +4) = two aligned words and a funnel shift.  NP (the
 * number of 32-word panels a row spans) is a template parameter so that the loads of four
 * rows x NP words are issued back to back before the first conversion: independent
 * chains, no branches; only the stores are predicated (lanes past the tile read other
 * shared memory of this CTA, harmlessly).
 */
template <int NP>
__device__ __forceinline__ void convert_rows_vec(const uint32_t *__restrict__ rp0,
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
                const float4 v = bytes_to_float4(__funnelshift_r(lo[i][p], hi[i][p], bsh));
                if (pred[p]) tp[(i0 + i) * tstride4 + 32 * p] = v;
            }
    }
}

/*
 * Horizontal task: out[j] = sum_k g[k] * in[j + C*k], j in [0, 8C), for one tile row.
 * `trow` points at the first input float of the segment (16-byte aligned), `wts` at the
 * zero-padded taps, nchunk = ceil(L / 4).
 */
template <int C>
__device__ __forceinline__ void h_task_acc(const float *__restrict__ trow,
                                           const float *__restrict__ wts, int nchunk,
                                           float (&acc)[8 * C])
{
    /* Ring of four slots of 4C input values.  A chunk of four taps reads slots p, p+1,
     * p+2 (values 0 .. 11C-1 past the chunk base) and, at its start, refills slot p+3 --
     * dead since the previous chunk -- with the values the NEXT chunk needs, so every
     * shared-memory load has a whole chunk of FFMAs to land. */
    constexpr int NW = 16 * C;
    constexpr int NA = 8 * C; /* accumulators */
    float win[NW];
#pragma unroll
    for (int j = 0; j < NA; j++) acc[j] = 0.0f;
    const float4 *src = reinterpret_cast<const float4 *>(trow);
#pragma unroll
    for (int v = 0; v < 3 * C; v++) {
        const float4 x = src[v];
        win[4 * v + 0] = x.x;
        win[4 * v + 1] = x.y;
        win[4 * v + 2] = x.z;
        win[4 * v + 3] = x.w;
    }
    const float4 *nxt = src + 3 * C;
    const float4 *wp = reinterpret_cast<const float4 *>(wts);
    float4 g4 = wp[0];
    for (int c = 0; c < nchunk; c += 4) {
#pragma unroll
        for (int p = 0; p < 4; p++) {
            if (p > 0 && c + p >= nchunk) break;
            const float g[4] = {g4.x, g4.y, g4.z, g4.w};
            g4 = wp[c + p + 1]; /* next chunk's taps (one padding quad follows the last) */
#pragma unroll
            for (int v = 0; v < C; v++) {
                const float4 x = nxt[v];
                const int q = (((p + 3) % 4) * C + v) * 4;
                win[q + 0] = x.x;
                win[q + 1] = x.y;
                win[q + 2] = x.z;
                win[q + 3] = x.w;
            }
            nxt += C;
#pragma unroll
            for (int t = 0; t < 4; t++) {
#pragma unroll
                for (int j = 0; j < NA; j++)
                    acc[j] = fmaf(g[t], win[(p * 4 * C + C * t + j) % NW], acc[j]);
            }
        }
    }
}

/* The same, stored as one row segment of a row-major intermediate. */
template <int C>
__device__ __forceinline__ void h_task(const float *__restrict__ trow,
                                       const float *__restrict__ wts, int nchunk,
                                       float *__restrict__ irow)
{
    constexpr int NA = 8 * C;
    float acc[NA];
    h_task_acc<C>(trow, wts, nchunk, acc);
    float4 *dst = reinterpret_cast<float4 *>(irow);
#pragma unroll
    for (int v = 0; v < NA / 4; v++)
        dst[v] = make_float4(acc[4 * v], acc[4 * v + 1], acc[4 * v + 2], acc[4 * v + 3]);
}

/*
 * Vertical task: acc[j][i] = sum_k g[k] * I[row0 + j + k][col0 + i], j < 8, i < 4.
 * `icol` points at I[row0][col0]; pitch in floats.  Same four-slot ring, over rows.
 */
template <int NV>
__device__ __forceinline__ void v_task(const float *__restrict__ ring, int pitch, int row0,
                                       int cap, const float *__restrict__ wts, int nchunk,
                                       float (&acc)[kRV][NV])
{
    /* `ring` points at column col0 of row 0 of the intermediate ring buffer of `cap` rows;
     * row0 and cap are multiples of 4, so a group of four rows never straddles the wrap.
     * NV = 4: one LDS.128 per row; NV = 3 (one RGB pixel): three conflict-free LDS.32. */
    float win[16][NV];
    auto load_row = [&](float (&dst)[NV], const float *src) {
        if (NV == 4) {
            const float4 x = *reinterpret_cast<const float4 *>(src);
            dst[0] = x.x;
            dst[1] = x.y;
            dst[2] = x.z;
            dst[NV - 1] = x.w;
        } else {
#pragma unroll
            for (int i = 0; i < NV; i++) dst[i] = src[i];
        }
    };
#pragma unroll
    for (int j = 0; j < kRV; j++)
#pragma unroll
        for (int i = 0; i < NV; i++) acc[j][i] = 0.0f;
    int rp = row0;
#pragma unroll
    for (int v = 0; v < 3; v++) {
        const float *base = ring + (size_t)rp * pitch;
#pragma unroll
        for (int t = 0; t < 4; t++) load_row(win[4 * v + t], base + (size_t)t * pitch);
        rp += 4;
        rp = rp >= cap ? rp - cap : rp;
    }
    const float4 *wp = reinterpret_cast<const float4 *>(wts);
    float4 g4 = wp[0];
    for (int c = 0; c < nchunk; c += 4) {
#pragma unroll
        for (int p = 0; p < 4; p++) {
            if (p > 0 && c + p >= nchunk) break;
            const float g[4] = {g4.x, g4.y, g4.z, g4.w};
            g4 = wp[c + p + 1]; /* next chunk's taps */
            const float *nxt = ring + (size_t)rp * pitch;
#pragma unroll
            for (int t = 0; t < 4; t++)
                load_row(win[(4 * (p + 3) + t) % 16], nxt + (size_t)t * pitch);
            rp += 4;
            rp = rp >= cap ? rp - cap : rp;
#pragma unroll
            for (int t = 0; t < 4; t++) {
#pragma unroll
                for (int j = 0; j < kRV; j++) {
#pragma unroll
                    for (int i = 0; i < NV; i++)
                        acc[j][i] = fmaf(g[t], win[(4 * p + t + j) % 16][i], acc[j][i]);
                }
            }
        }
    }
}

/* Geometry every thread derives from a 16-byte item descriptor (fk_internal.h). */
struct item_geo {
    int f, x0, y0, fw, fh, L;
    int r, nchunk, th, nseg, tw, twz;
    int xs_c, skew, npanel;
    bool xin;
    uint32_t taps_off;
};

template <int C> __device__ __forceinline__ item_geo decode_item(const uint4 q, int W)
{
    constexpr int SEG = 8 * C;
    item_geo g;
    g.f = (int)q.x;
    g.x0 = (int)(q.y & 0xffffu);
    g.y0 = (int)(q.y >> 16);
    g.fw = (int)(q.z & 0xffu);
    g.fh = (int)(q.z >> 21);
    g.L = (int)((q.z >> 8) & 0x1fffu);
    g.taps_off = q.w;
    g.r = (g.L - 1) >> 1;
    g.nchunk = (g.L + 3) >> 2;
    g.th = g.fh + 2 * g.r;
    g.nseg = (g.fw * C + SEG - 1) / SEG;
    g.tw = (g.fw + 2 * g.r) * C;                  /* valid tile floats per row */
    g.twz = C * (8 * g.nseg + 4 + 4 * g.nchunk);  /* floats the H tasks may touch */
    g.xin = (g.x0 - g.r >= 0) && (g.x0 + g.fw + g.r <= W);
    g.xs_c = fast_clamp(g.x0 - g.r, 0, W - 1);
    /* TMA needs the box to start on a 16-byte boundary of the row: fetch from the
     * aligned-down byte and skip `skew` bytes when converting */
    g.skew = g.xs_c * C - ((g.xs_c * C) & ~15);
    g.npanel = (g.skew + g.tw + 4 + kPanelB - 1) / kPanelB; /* valid bytes only */
    return g;
}

typedef CUresult (*encode_tiled_fn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                    const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                    const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

encode_tiled_fn get_encode_tiled()
{
    static encode_tiled_fn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (encode_tiled_fn)p;
    }
    return fn;
}

/* 3-D byte tensor (W*C, H, N) over the input batch; false if TMA cannot describe it. */
bool make_tensor_map(CUtensorMap *map, const void *in, int W, int H, int C, int n_frames)
{
    encode_tiled_fn enc = get_encode_tiled();
    const size_t pitch = (size_t)W * C;
    if (!enc || ((uintptr_t)in & 15) != 0 || (pitch & 15) != 0) return false;
    cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)H, (cuuint64_t)n_frames};
    cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)pitch * H};
    cuuint32_t box[3] = {(cuuint32_t)kPanelB, (cuuint32_t)kTB, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void *>(in), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

} // namespace

#endif /* FK_STAGE_CUH_ */
