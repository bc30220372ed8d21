/*
 * proto_pair.cuh -- EXPLORATION ONLY (not part of libfovea.so; measured and dropped): the two blur passes on packed FMAs (fma.rn.f32x2, SASS FFMA2: two fp32 FMAs
 * per lane and issue slot), the inner loops of fk_blur_pair (fk_blur_cols.cu).
 *
 * An FFMA2 wants both its multiplicand and its accumulator as aligned register pairs.  A 1-D
 * convolution slides along its own axis, so pairs along that axis would need every input
 * value twice (even- and odd-aligned); pairs ACROSS the axis need nothing extra:
 *
 *   H pass (blockwise.py:151)  a lane owns TWO tile rows x 24 float columns; a pair is the same
 *                              column of the two rows.  Input pairs are made by the byte ->
 *                              fp32 PRMTs, which write any register they like.
 *   V pass (blockwise.py:152)  a lane owns THREE COLUMN PAIRS (two RGB pixels) x 8 output rows;
 *                              a pair is two adjacent columns of one row, which is how the
 *                              intermediate is laid out: [column pair][row][2 floats], so one
 *                              LDS.128 brings two rows of a pair.
 *
 * Each FMA of a pair is the scalar fmaf of the same operands in the same order, so the
 * results are bit-identical to fk_blur_generic.  Taps are kept DUPLICATED in shared memory
 * (g0, g0, g1, g1, ...): one LDS.128 yields two tap pairs.
 */
#ifndef FK_PAIR_CUH_
#define FK_PAIR_CUH_

#include <stdint.h>

namespace {

typedef unsigned long long u64;

constexpr int kTB2 = 64;             /* tile rows per block of the packed kernel */
constexpr int kQS2 = 16 * kTB2;      /* bytes between 16-byte chunks of the raw block: 1024 */

__device__ __forceinline__ u64 pack2(float lo, float hi)
{
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ u64 pack2u(uint32_t lo, uint32_t hi)
{
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
    return r;
}
__device__ __forceinline__ void unpack2(u64 v, float &lo, float &hi)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c)
{
    u64 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ void sts32(uint32_t addr, float v)
{
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ uint4 lds128u(uint32_t addr)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}
/* two 64-bit pairs with one LDS.128 */
__device__ __forceinline__ void lds2x64(uint32_t addr, u64 &a, u64 &b)
{
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr));
}

/*
 * Horizontal task on raw bytes, two rows: acc[j] = (sum_k g[k] * A[j + 3k], sum_k g[k] * B[j + 3k]),
 * j in [0, 24), where A / B are the byte streams of the lane's two rows starting `bsh / 8`
 * bytes (0..2) into the 16-byte chunk at rowA / rowB (shared addresses; the same chunk of the
 * next 16 bytes lies kQS2 further).  `wts2` = duplicated taps, already padded in front with
 * the zeros that absorb the whole pixels between the chunk boundary and the first input,
 * followed by at least one zero quad; nchunk = quads of taps.  The byte -> fp32 encoding and
 * the tap scale are those of bytes_to_float4_s (fk_blur_cols.cu).
 *
 * The stream is consumed in aligned 16-byte quads (one LDS.128 per row and 5 1/3 taps), so
 * which register holds which word is known at compile time; a turn of four chunks takes
 * three quads per row.  Window: ring of four slots of 12 pairs, slot p + 3 converted during
 * chunk p from words loaded a chunk earlier.
 */
__device__ __forceinline__ void h2_bytes(uint32_t rowA, uint32_t rowB, uint32_t bsh, uint32_t wts2,
                                         int nchunk, u64 (&acc)[24])
{
    u64 win[48];
    auto cvt = [&](const int slot4, uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
        const uint32_t wa = __funnelshift_r(a0, a1, bsh), wb = __funnelshift_r(b0, b1, bsh);
        win[slot4 + 0] = pack2u(__byte_perm(wa, 0u, 0x4044), __byte_perm(wb, 0u, 0x4044));
        win[slot4 + 1] = pack2u(__byte_perm(wa, 0u, 0x4144), __byte_perm(wb, 0u, 0x4144));
        win[slot4 + 2] = pack2u(__byte_perm(wa, 0u, 0x4244), __byte_perm(wb, 0u, 0x4244));
        win[slot4 + 3] = pack2u(__byte_perm(wa, 0u, 0x4344), __byte_perm(wb, 0u, 0x4344));
    };
    /* words 0..11 (quads 0..2) of both rows: slots 0..2 = words 0..8 (+ word 9 for the shift) */
    uint4 qa0 = lds128u(rowA), qb0 = lds128u(rowB);
    uint4 qa1 = lds128u(rowA + kQS2), qb1 = lds128u(rowB + kQS2);
    uint4 qcA = lds128u(rowA + 2 * kQS2), qcB = lds128u(rowB + 2 * kQS2); /* words 8..11 */
    uint4 qaA = lds128u(rowA + 3 * kQS2), qaB = lds128u(rowB + 3 * kQS2); /* words 12..15 */
    uint4 qbA = qaA, qbB = qaB;                                           /* words 16..19, loaded in phase 1 */
    cvt(0, qa0.x, qa0.y, qb0.x, qb0.y);
    cvt(4, qa0.y, qa0.z, qb0.y, qb0.z);
    cvt(8, qa0.z, qa0.w, qb0.z, qb0.w);
    cvt(12, qa0.w, qa1.x, qb0.w, qb1.x);
    cvt(16, qa1.x, qa1.y, qb1.x, qb1.y);
    cvt(20, qa1.y, qa1.z, qb1.y, qb1.z);
    cvt(24, qa1.z, qa1.w, qb1.z, qb1.w);
    cvt(28, qa1.w, qcA.x, qb1.w, qcB.x);
    cvt(32, qcA.x, qcA.y, qcB.x, qcB.y);
#pragma unroll
    for (int j = 0; j < 24; j++) acc[j] = 0ull;
    uint32_t nA = rowA, nB = rowB; /* quad k of the turn's base: + k * kQS2 */
    u64 g0, g1, g2, g3;
    lds2x64(wts2, g0, g1);
    lds2x64(wts2 + 16, g2, g3);
    uint32_t wa = wts2 + 32;
    auto fmas = [&](const int p, const u64 (&g)[4]) {
#pragma unroll
        for (int t = 0; t < 4; t++)
#pragma unroll
            for (int j = 0; j < 24; j++) acc[j] = ffma2(g[t], win[(12 * p + 3 * t + j) % 48], acc[j]);
    };
    for (int c = 0; c < nchunk; c += 4) {
        { /* phase 0: slot 3 <- words 9, 10, 11 (12) */
            const u64 g[4] = {g0, g1, g2, g3};
            lds2x64(wa, g0, g1);
            lds2x64(wa + 16, g2, g3);
            cvt(36, qcA.y, qcA.z, qcB.y, qcB.z);
            cvt(40, qcA.z, qcA.w, qcB.z, qcB.w);
            cvt(44, qcA.w, qaA.x, qcB.w, qaB.x);
            fmas(0, g);
        }
        if (c + 1 >= nchunk) break;
        { /* phase 1: slot 0 <- words 12, 13, 14 (15); load words 16..19 */
            const u64 g[4] = {g0, g1, g2, g3};
            lds2x64(wa + 32, g0, g1);
            lds2x64(wa + 48, g2, g3);
            qbA = lds128u(nA + 4 * kQS2);
            qbB = lds128u(nB + 4 * kQS2);
            cvt(0, qaA.x, qaA.y, qaB.x, qaB.y);
            cvt(4, qaA.y, qaA.z, qaB.y, qaB.z);
            cvt(8, qaA.z, qaA.w, qaB.z, qaB.w);
            fmas(1, g);
        }
        if (c + 2 >= nchunk) break;
        { /* phase 2: slot 1 <- words 15, 16, 17 (18); load words 20..23 */
            const u64 g[4] = {g0, g1, g2, g3};
            lds2x64(wa + 64, g0, g1);
            lds2x64(wa + 80, g2, g3);
            qcA = lds128u(nA + 5 * kQS2);
            qcB = lds128u(nB + 5 * kQS2);
            cvt(12, qaA.w, qbA.x, qaB.w, qbB.x);
            cvt(16, qbA.x, qbA.y, qbB.x, qbB.y);
            cvt(20, qbA.y, qbA.z, qbB.y, qbB.z);
            fmas(2, g);
        }
        if (c + 3 >= nchunk) break;
        { /* phase 3: slot 2 <- words 18, 19, 20 (21); load the next turn's words 12..15 */
            const u64 g[4] = {g0, g1, g2, g3};
            lds2x64(wa + 96, g0, g1);
            lds2x64(wa + 112, g2, g3);
            wa += 128;
            qaA = lds128u(nA + 6 * kQS2);
            qaB = lds128u(nB + 6 * kQS2);
            nA += 3 * kQS2;
            nB += 3 * kQS2;
            cvt(24, qbA.z, qbA.w, qbB.z, qbB.w);
            cvt(28, qbA.w, qcA.x, qbB.w, qcB.x);
            cvt(32, qcA.x, qcA.y, qcB.x, qcB.y);
            fmas(3, g);
        }
    }
}

/*
 * Vertical task on the paired intermediate: acc[j][k] = sum_t g[t] * P_k[row0 + j + t], j < 8
 * output rows, k < 3 adjacent column pairs (two RGB pixels); P_k[row] is the pair of floats at
 * col + k * cpitch + 8 * row (shared addresses); a column pair is a ring of `cap` rows; row0 and
 * cap are multiples of 4 so that a quad of rows never straddles the wrap.  `wts2` = duplicated
 * taps padded in front to a multiple of four, one zero quad behind.  Four-slot register ring
 * of four rows per column pair (two LDS.128), loaded a chunk ahead of its use.
 */
__device__ __forceinline__ void v2_task(uint32_t col, uint32_t cpitch, int row0, int cap, uint32_t wts2,
                                        int nchunk, int zpad, u64 (&acc)[8][3])
{
    u64 win[3][16];
    const uint32_t end = col + 8u * (uint32_t)cap;
    auto step = [&](uint32_t x) {
        x += 32;
        return x == end ? col : x;
    };
    auto load4 = [&](const int slot, const uint32_t la) { /* ring slot <- the quad of rows at la */
#pragma unroll
        for (int k = 0; k < 3; k++) {
            lds2x64(la + k * cpitch, win[k][(4 * slot + 0) % 16], win[k][(4 * slot + 1) % 16]);
            lds2x64(la + k * cpitch + 16, win[k][(4 * slot + 2) % 16], win[k][(4 * slot + 3) % 16]);
        }
    };
    uint32_t a = col + 8u * (uint32_t)row0;
#pragma unroll
    for (int v = 0; v < 3; v++) {
        load4(v, a);
        a = step(a);
    }
#pragma unroll
    for (int j = 0; j < 8; j++)
#pragma unroll
        for (int k = 0; k < 3; k++) acc[j][k] = 0ull;
    u64 g0, g1, g2, g3;
    lds2x64(wts2, g0, g1);
    lds2x64(wts2 + 16, g2, g3);
    uint32_t wa = wts2 + 32;
    auto chunk = [&](const int p, const uint32_t la) {
        const u64 g[4] = {g0, g1, g2, g3};
        lds2x64(wa, g0, g1);
        lds2x64(wa + 16, g2, g3);
        wa += 32;
        load4(p + 3, la);
#pragma unroll
        for (int t = 0; t < 4; t++)
#pragma unroll
            for (int j = 0; j < 8; j++)
#pragma unroll
                for (int k = 0; k < 3; k++)
                    acc[j][k] = ffma2(g[t], win[k][(4 * p + t + j) % 16], acc[j][k]);
    };
    (void)zpad;
    for (int c = 0; c < nchunk; c += 4) {
        uint32_t a1 = a + 32, a2 = a + 64, a3 = a + 96, an = a + 128;
        if (an >= end) {
            a1 = step(a);
            a2 = step(a1);
            a3 = step(a2);
            an = step(a3);
        }
        chunk(0, a);
        if (c + 1 >= nchunk) break;
        chunk(1, a1);
        if (c + 2 >= nchunk) break;
        chunk(2, a2);
        if (c + 3 >= nchunk) break;
        chunk(3, a3);
        a = an;
    }
}

} // namespace

#endif /* FK_PAIR_CUH_ */
