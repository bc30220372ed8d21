/*
 * proto_wide.cuh -- EXPLORATION ONLY (not part of libfovea.so): the two blur passes with 48 accumulators per lane, inner loops of a would-be
 * fk_blur_wide (fk_blur_cols.cu).
 *
 * Measured on B200 (tools/ubench_vloop.cu, tools/proto_ffma2.cu): the FFMA pattern of these
 * loops sustains 87-90 % of the FP32 peak from registers alone, a broadcast LDS.128 (taps) is
 * free, and every other LDS.128 costs about 4.5 issue cycles -- a shared-memory load is paid
 * by the byte, conflicts included.  What a pass spends next to its FFMAs is therefore set by
 * the BYTES IT LOADS PER FMA, and the only lever is register blocking:
 *
 *   H pass (blockwise.py:151)  a lane owns TWO tile rows x 24 float columns (fk_blur_tma: one
 *                              row): the taps and the loop control are shared by both rows, and
 *                              the raw bytes arrive as conflict-free LDS.128 quads (row pitch
 *                              16 B) instead of 4-way conflicting LDS.32 words.
 *   V pass (blockwise.py:152)  a lane owns one RGB pixel x SIXTEEN output rows (fk_blur_tma:
 *                              eight): (16 + 2r) / 16 window rows per output row instead of
 *                              (8 + 2r) / 8.
 *
 * Packed FMAs (fma.rn.f32x2) were measured and dropped: 82 % from registers, and no gain in
 * these loops -- they are bound by load bytes, not by issue slots.
 */
#ifndef FK_WIDE_CUH_
#define FK_WIDE_CUH_

#include <stdint.h>

namespace {

constexpr int kTB2 = 64;        /* tile rows per block of the wide kernel */
constexpr int kQS2 = 16 * kTB2; /* bytes between 16-byte chunks of a row in the raw block: 1024 */
constexpr int kRV2 = 16;        /* output rows per V task */

__device__ __forceinline__ uint4 lds128u(uint32_t addr)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}
__device__ __forceinline__ float4 lds128f(uint32_t addr)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}

/*
 * Horizontal task on raw bytes, two rows: accA[j] = sum_k g[k] * A[j + 3k], accB likewise,
 * j in [0, 24), where A / B are the byte streams of the lane's two rows starting `bsh / 8`
 * bytes (0..2) into the 16-byte chunk at rowA / rowB (shared addresses; the next 16 bytes of a
 * row lie kQS2 further).  `wts` = taps already padded in front with the zeros that absorb the
 * whole pixels between the chunk boundary and the first input, and followed by at least one
 * zero quad; nchunk = quads of taps.  Byte -> fp32 encoding and tap scale: bytes_to_float4_s
 * (fk_blur_cols.cu).
 *
 * The stream is consumed in aligned 16-byte quads, so which register holds which word is known
 * at compile time; a turn of four chunks takes three quads per row.  Window: ring of four
 * slots of 12 floats per row, slot p + 3 converted during chunk p from words loaded a chunk
 * earlier.
 */
__device__ __forceinline__ void h_bytes2(uint32_t rowA, uint32_t rowB, uint32_t bsh, uint32_t wts,
                                         int nchunk, float (&accA)[24], float (&accB)[24])
{
    float wA[48], wB[48];
    auto cvt = [&](const int s, uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
        const uint32_t va = __funnelshift_r(a0, a1, bsh), vb = __funnelshift_r(b0, b1, bsh);
        wA[s + 0] = __uint_as_float(__byte_perm(va, 0u, 0x4044));
        wA[s + 1] = __uint_as_float(__byte_perm(va, 0u, 0x4144));
        wA[s + 2] = __uint_as_float(__byte_perm(va, 0u, 0x4244));
        wA[s + 3] = __uint_as_float(__byte_perm(va, 0u, 0x4344));
        wB[s + 0] = __uint_as_float(__byte_perm(vb, 0u, 0x4044));
        wB[s + 1] = __uint_as_float(__byte_perm(vb, 0u, 0x4144));
        wB[s + 2] = __uint_as_float(__byte_perm(vb, 0u, 0x4244));
        wB[s + 3] = __uint_as_float(__byte_perm(vb, 0u, 0x4344));
    };
    /* words 0..11 (quads 0..2) of both rows: slots 0..2 = words 0..8 (+ word 9 for the shift) */
    const uint4 a0 = lds128u(rowA), b0 = lds128u(rowB);
    const uint4 a1 = lds128u(rowA + kQS2), b1 = lds128u(rowB + kQS2);
    uint4 qcA = lds128u(rowA + 2 * kQS2), qcB = lds128u(rowB + 2 * kQS2); /* words 8..11 */
    uint4 qaA = lds128u(rowA + 3 * kQS2), qaB = lds128u(rowB + 3 * kQS2); /* words 12..15 */
    uint4 qbA = qaA, qbB = qaB;                                           /* words 16..19: phase 1 */
    cvt(0, a0.x, a0.y, b0.x, b0.y);
    cvt(4, a0.y, a0.z, b0.y, b0.z);
    cvt(8, a0.z, a0.w, b0.z, b0.w);
    cvt(12, a0.w, a1.x, b0.w, b1.x);
    cvt(16, a1.x, a1.y, b1.x, b1.y);
    cvt(20, a1.y, a1.z, b1.y, b1.z);
    cvt(24, a1.z, a1.w, b1.z, b1.w);
    cvt(28, a1.w, qcA.x, b1.w, qcB.x);
    cvt(32, qcA.x, qcA.y, qcB.x, qcB.y);
#pragma unroll
    for (int j = 0; j < 24; j++) accA[j] = accB[j] = 0.0f;
    uint32_t nA = rowA, nB = rowB; /* quad k of the turn's base: + k * kQS2 */
    float4 g4 = lds128f(wts);
    uint32_t wa = wts + 16;
    auto fmas = [&](const int p, const float (&g)[4]) {
#pragma unroll
        for (int t = 0; t < 4; t++)
#pragma unroll
            for (int j = 0; j < 24; j++) {
                accA[j] = fmaf(g[t], wA[(12 * p + 3 * t + j) % 48], accA[j]);
                accB[j] = fmaf(g[t], wB[(12 * p + 3 * t + j) % 48], accB[j]);
            }
    };
    for (int c = 0; c < nchunk; c += 4) {
        { /* phase 0: slot 3 <- words 9, 10, 11 (12) */
            const float g[4] = {g4.x, g4.y, g4.z, g4.w};
            g4 = lds128f(wa);
            cvt(36, qcA.y, qcA.z, qcB.y, qcB.z);
            cvt(40, qcA.z, qcA.w, qcB.z, qcB.w);
            cvt(44, qcA.w, qaA.x, qcB.w, qaB.x);
            fmas(0, g);
        }
        if (c + 1 >= nchunk) break;
        { /* phase 1: slot 0 <- words 12, 13, 14 (15); load words 16..19 */
            const float g[4] = {g4.x, g4.y, g4.z, g4.w};
            g4 = lds128f(wa + 16);
            qbA = lds128u(nA + 4 * kQS2);
            qbB = lds128u(nB + 4 * kQS2);
            cvt(0, qaA.x, qaA.y, qaB.x, qaB.y);
            cvt(4, qaA.y, qaA.z, qaB.y, qaB.z);
            cvt(8, qaA.z, qaA.w, qaB.z, qaB.w);
            fmas(1, g);
        }
        if (c + 2 >= nchunk) break;
        { /* phase 2: slot 1 <- words 15, 16, 17 (18); load words 20..23 */
            const float g[4] = {g4.x, g4.y, g4.z, g4.w};
            g4 = lds128f(wa + 32);
            qcA = lds128u(nA + 5 * kQS2);
            qcB = lds128u(nB + 5 * kQS2);
            cvt(12, qaA.w, qbA.x, qaB.w, qbB.x);
            cvt(16, qbA.x, qbA.y, qbB.x, qbB.y);
            cvt(20, qbA.y, qbA.z, qbB.y, qbB.z);
            fmas(2, g);
        }
        if (c + 3 >= nchunk) break;
        { /* phase 3: slot 2 <- words 18, 19, 20 (21); load the next turn's words 12..15 */
            const float g[4] = {g4.x, g4.y, g4.z, g4.w};
            g4 = lds128f(wa + 48);
            wa += 64;
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
 * Horizontal task on raw bytes, ONE row x 48 float columns (16 pixels): acc[j] = sum_k g[k] *
 * A[j + 3k], j in [0, 48).  Same stream conventions as h_bytes2.  Window: ring of eight slots
 * of 12 floats (a chunk of four taps reads 48 + 9 floats = five slots, the sixth is converted
 * for the next chunk; eight because the ring must turn with the quads: 2 turns = 8 chunks = 6
 * quads).  A converted byte is used by up to 16 FMAs instead of 8.
 */
__device__ __forceinline__ void h_bytes48(uint32_t rowA, uint32_t bsh, uint32_t wts, int nchunk,
                                          float (&acc)[48])
{
    float w[96];
    auto cvt = [&](const int s, uint32_t a0, uint32_t a1) {
        const uint32_t va = __funnelshift_r(a0, a1, bsh);
        w[s + 0] = __uint_as_float(__byte_perm(va, 0u, 0x4044));
        w[s + 1] = __uint_as_float(__byte_perm(va, 0u, 0x4144));
        w[s + 2] = __uint_as_float(__byte_perm(va, 0u, 0x4244));
        w[s + 3] = __uint_as_float(__byte_perm(va, 0u, 0x4344));
    };
    /* slots 0..4 = floats 0..59 = words 0..14 (+ word 15 for the shift): quads 0..3 */
    uint4 q0 = lds128u(rowA), q1 = lds128u(rowA + kQS2), q2 = lds128u(rowA + 2 * kQS2),
          q3 = lds128u(rowA + 3 * kQS2);
    cvt(0, q0.x, q0.y); cvt(4, q0.y, q0.z); cvt(8, q0.z, q0.w); cvt(12, q0.w, q1.x);
    cvt(16, q1.x, q1.y); cvt(20, q1.y, q1.z); cvt(24, q1.z, q1.w); cvt(28, q1.w, q2.x);
    cvt(32, q2.x, q2.y); cvt(36, q2.y, q2.z); cvt(40, q2.z, q2.w); cvt(44, q2.w, q3.x);
    cvt(48, q3.x, q3.y); cvt(52, q3.y, q3.z); cvt(56, q3.z, q3.w);
    /* the stream from word 15 on, in quads: qa = words 12..15 (q3), qb = 16..19, qc = 20..23 */
    uint4 qa = q3, qb = lds128u(rowA + 4 * kQS2), qc = qb;
#pragma unroll
    for (int j = 0; j < 48; j++) acc[j] = 0.0f;
    uint32_t nA = rowA;
    float4 g4 = lds128f(wts);
    uint32_t wa = wts + 16;
    auto fmas = [&](const int p, const float (&g)[4]) {
#pragma unroll
        for (int t = 0; t < 4; t++)
#pragma unroll
            for (int j = 0; j < 48; j++) acc[j] = fmaf(g[t], w[(12 * p + 3 * t + j) % 96], acc[j]);
    };
    /* chunk c (phase p = c mod 8) converts slot p + 5 = floats 12 (c + 5) .. = words 15 + 3c ..
     * 17 + 3c (+ 18 + 3c for the shift).  Word 15 + 3c lies in quad (15 + 3c) / 4: the word ->
     * register map repeats every 4 chunks (3 quads), the slot map every 8. */
    for (int c = 0; c < nchunk; c += 8) {
#pragma unroll
        for (int h = 0; h < 2; h++) { /* two turns of four chunks */
            const int p0 = 4 * h;
            { /* words 15, 16, 17 (18): qa.w, qb.x, qb.y, (qb.z); load words 20..23 */
                const float g[4] = {g4.x, g4.y, g4.z, g4.w};
                g4 = lds128f(wa);
                qc = lds128u(nA + 5 * kQS2);
                cvt((12 * (p0 + 5)) % 96 + 0, qa.w, qb.x);
                cvt((12 * (p0 + 5)) % 96 + 4, qb.x, qb.y);
                cvt((12 * (p0 + 5)) % 96 + 8, qb.y, qb.z);
                fmas(p0, g);
            }
            if (c + p0 + 1 >= nchunk) return;
            { /* words 18, 19, 20 (21): qb.z, qb.w, qc.x, (qc.y); load words 24..27 */
                const float g[4] = {g4.x, g4.y, g4.z, g4.w};
                g4 = lds128f(wa + 16);
                qa = lds128u(nA + 6 * kQS2);
                cvt((12 * (p0 + 6)) % 96 + 0, qb.z, qb.w);
                cvt((12 * (p0 + 6)) % 96 + 4, qb.w, qc.x);
                cvt((12 * (p0 + 6)) % 96 + 8, qc.x, qc.y);
                fmas(p0 + 1, g);
            }
            if (c + p0 + 2 >= nchunk) return;
            { /* words 21, 22, 23 (24): qc.y, qc.z, qc.w, (qa.x); load words 28..31 */
                const float g[4] = {g4.x, g4.y, g4.z, g4.w};
                g4 = lds128f(wa + 32);
                qb = lds128u(nA + 7 * kQS2);
                cvt((12 * (p0 + 7)) % 96 + 0, qc.y, qc.z);
                cvt((12 * (p0 + 7)) % 96 + 4, qc.z, qc.w);
                cvt((12 * (p0 + 7)) % 96 + 8, qc.w, qa.x);
                fmas(p0 + 2, g);
            }
            if (c + p0 + 3 >= nchunk) return;
            { /* words 24, 25, 26 (27): qa.x, qa.y, qa.z, (qa.w); no load */
                const float g[4] = {g4.x, g4.y, g4.z, g4.w};
                g4 = lds128f(wa + 48);
                wa += 64;
                cvt((12 * (p0 + 8)) % 96 + 0, qa.x, qa.y);
                cvt((12 * (p0 + 8)) % 96 + 4, qa.y, qa.z);
                cvt((12 * (p0 + 8)) % 96 + 8, qa.z, qa.w);
                nA += 3 * kQS2;
                fmas(p0 + 3, g);
            }
            if (c + p0 + 4 >= nchunk) return;
        }
    }
}

/*
 * Vertical task on the transposed intermediate: acc[j][k] = sum_t g[t] * col_k[row0 + j + t],
 * j < 16 output rows, k < 3 adjacent columns (one RGB pixel).  `col` = shared address of row 0
 * of the first column, `cpitch` bytes between columns; a column is a ring of `cap` rows; row0
 * and cap are multiples of 4, so a quad of rows never straddles the wrap.  Six-slot register
 * ring of four rows per column (16 + 3 rows a chunk reads, 4 loaded for the next), one
 * LDS.128 per column and chunk.  `wts` = taps padded in front to a multiple of four, one zero
 * quad behind.
 */
__device__ __forceinline__ void v_task16(uint32_t col, uint32_t cpitch, int row0, int cap, uint32_t wts,
                                         int nchunk, float (&acc)[kRV2][3])
{
    float win[3][24];
    const uint32_t end = col + 4u * (uint32_t)cap;
    auto step = [&](uint32_t x) {
        x += 16;
        return x == end ? col : x;
    };
    auto load4 = [&](const int slot, const uint32_t la) {
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const float4 x = lds128f(la + k * cpitch);
            win[k][(4 * slot + 0) % 24] = x.x;
            win[k][(4 * slot + 1) % 24] = x.y;
            win[k][(4 * slot + 2) % 24] = x.z;
            win[k][(4 * slot + 3) % 24] = x.w;
        }
    };
    uint32_t a = col + 4u * (uint32_t)row0;
#pragma unroll
    for (int v = 0; v < 5; v++) {
        load4(v, a);
        a = step(a);
    }
#pragma unroll
    for (int j = 0; j < kRV2; j++)
#pragma unroll
        for (int k = 0; k < 3; k++) acc[j][k] = 0.0f;
    float4 g4 = lds128f(wts);
    uint32_t wa = wts + 16;
    auto chunk = [&](const int p, const uint32_t la) {
        const float g[4] = {g4.x, g4.y, g4.z, g4.w};
        g4 = lds128f(wa);
        wa += 16;
        load4(p + 5, la);
#pragma unroll
        for (int t = 0; t < 4; t++)
#pragma unroll
            for (int j = 0; j < kRV2; j++)
#pragma unroll
                for (int k = 0; k < 3; k++)
                    acc[j][k] = fmaf(g[t], win[k][(4 * p + t + j) % 24], acc[j][k]);
    };
    for (int c = 0; c < nchunk; c += 6) {
        uint32_t a1 = a + 16, a2 = a + 32, a3 = a + 48, a4 = a + 64, a5 = a + 80, an = a + 96;
        if (an >= end) {
            a1 = step(a);
            a2 = step(a1);
            a3 = step(a2);
            a4 = step(a3);
            a5 = step(a4);
            an = step(a5);
        }
        chunk(0, a);
        if (c + 1 >= nchunk) break;
        chunk(1, a1);
        if (c + 2 >= nchunk) break;
        chunk(2, a2);
        if (c + 3 >= nchunk) break;
        chunk(3, a3);
        if (c + 4 >= nchunk) break;
        chunk(4, a4);
        if (c + 5 >= nchunk) break;
        chunk(5, a5);
        a = an;
    }
}

} // namespace

#endif /* FK_WIDE_CUH_ */
