// Prototype / microbenchmark of alternative formulations of the two blur passes against the
// loops of fk_blur_tma (h_bytes + v_task_px), on synthetic shared-memory contents (no TMA):
// measures the FMA rate the loops sustain (H only, V only, both) and checks every formulation
// against a plain sequential-fmaf reference, bit for bit.
//   "wide"  (tools/proto_wide.cuh) 48 accumulators per lane: H two rows x 24 columns from
//           conflict-free LDS.128 quads, V one pixel x 16 rows
//   "pair"  (tools/proto_pair.cuh, an earlier revision of this file) the same shapes on packed
//           fma.rn.f32x2 -- bit-identical, no faster
// Results (B200, round 2, profiles/README.md): every formulation ends at 58-63 % of the FP32
// peak in the H loop and 67-77 % in the V loop; none beats the shipped loops by enough to pay
// for its registers, so the product kernel keeps them.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o tools/proto_ffma2 tools/proto_ffma2.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2012_08655_b200/csrc/fk_blur_cols.cu"
#include "proto_wide.cuh"

namespace {

constexpr int kIters = 200;

// deterministic pseudo-random byte of (row, byte index)
__host__ __device__ inline uint32_t hash32(uint32_t x)
{
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
__host__ __device__ inline unsigned char src_byte(int row, int b) { return (unsigned char)(hash32(row * 4099u + b) >> 11); }

struct proto_args {
    int L;        // taps
    int skew;     // byte of the stream start inside its 16-byte chunk (old: skew_h; new: t0 mod 16)
    int iters;
    int hv;       // 1: H pass only, 2: V pass only, 3: both
    float *hout;  // [64][96] H results of the last iteration (row-major)
    float *vout;  // [64 - ... ] V results
    unsigned *sink;
};

// ---- mode 0: the loops of fk_blur_tma<uint8_t> as they are (32-row block) -------------------
__global__ void __launch_bounds__(128, 3) k_old(proto_args a, const float *taps)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    const int L = a.L, r = (L - 1) / 2, nchunk = (L + 3) / 4, zpad = 4 * nchunk - L;
    const int nq = (168 + 6 * r + 15) / 16;
    const int nblk0 = (32 + 2 * r + 31) / 32, rows_in = nblk0 * 32 + 4; // enough intermediate rows for 4 groups of 8 outputs
    const int icap = (rows_in + 3) & ~3, ipitch = (icap & 7) == 4 ? icap : icap + 4;
    unsigned char *raw = sm;
    float *wv = reinterpret_cast<float *>(sm + nq * 512);
    float *wh = wv + 4 * nchunk + 4;
    float *ring = wh + 4 * nchunk + 4;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < nq * 512; i += 128) {
        const int ch = i >> 9, row = (i >> 4) & 31, b = i & 15;
        raw[i] = src_byte(row, ch * 16 + b);
    }
    for (int i = tid; i < 4 * nchunk + 4; i += 128) {
        const float g = i >= zpad && i < zpad + L ? taps[i - zpad] : 0.0f;
        wv[i] = g;
        wh[i] = g * kTapScaleH;
    }
    for (int i = tid; i < kRowF * ipitch; i += 128) ring[i] = 0.0f;
    __syncthreads();
    const uint32_t raw_s = smem_u32(raw), ring_s = smem_u32(ring);
    unsigned sink = 0;
    for (int it = 0; it < a.iters; it++) {
        // H: lane = row; rows of the intermediate [it-th block] at ring rows zpad + lane (+32 k)
        for (int blk = 0; (a.hv & 1) && blk < nblk0; blk++) {
            float hacc[kSegF];
            h_bytes(raw_s + (uint32_t)(lane * kQB), a.skew + kSegF * warp, smem_u32(wh), nchunk, zpad, hacc);
            float *rp = ring + (size_t)(kSegF * warp) * ipitch + blk * 32 + lane + zpad;
#pragma unroll
            for (int j = 0; j < kSegF; j++) rp[j * ipitch] = hacc[j];
            if (a.hout && it == a.iters - 1 && blk == 0)
                for (int j = 0; j < kSegF; j++) a.hout[lane * 96 + kSegF * warp + j] = hacc[j];
        }
        __syncwarp();
        // V: 32 tasks = 4 groups x 8 pixels
        if (a.hv & 2) {
            const int gi = lane >> 3, px = lane & 7;
            float acc[kRV][kC];
            v_task_px(ring_s + 4u * (uint32_t)((kSegF * warp + kC * px) * ipitch), 4u * (uint32_t)ipitch,
                      gi * kRV, icap, smem_u32(wv), nchunk, zpad, acc);
#pragma unroll
            for (int j = 0; j < kRV; j++)
#pragma unroll
                for (int k = 0; k < kC; k++) {
                    sink ^= __float_as_uint(acc[j][k]);
                    if (a.vout && it == a.iters - 1) a.vout[(gi * kRV + j) * 96 + kSegF * warp + kC * px + k] = acc[j][k];
                }
        }
        __syncwarp();
    }
    if (sink == 0x12345u) a.sink[blockIdx.x] = sink;
}

// ---- mode 1: 48 accumulators per lane (64-row block): H two rows x 24 columns, V one pixel x 16 rows
__global__ void __launch_bounds__(128, 3) k_new(proto_args a, const float *taps)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    const int L = a.L, r = (L - 1) / 2, nchunk = (L + 3) / 4, zpad = 4 * nchunk - L;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // per-warp stream geometry: first needed byte a0 = skew + 24 warp (relative to the box's first
    // byte); window starts on the 16-byte chunk at or below, zf whole pixels + rem bytes early
    const int a0 = a.skew + kSegF * warp;
    const int d = a0 & 15, zf = d / 3, rem = d - 3 * zf;
    const int nchunk_h = (zf + L + 3) >> 2;
    const int nch_max = (5 + L + 3) >> 2;
    const int nq = (15 + 72 + 24 + 12 * nch_max + 16 + 16 + 15) / 16;
    const int nblk0 = (64 + 2 * r + 63) / 64, rows_in = nblk0 * 64 + 4;
    const int icap = (rows_in + 3) & ~3, ipitch = (icap & 7) == 4 ? icap : icap + 4;
    unsigned char *raw = sm;
    float *wv = reinterpret_cast<float *>(sm + nq * kQS2);
    float *wh = wv + 4 * nchunk + 4;           // per warp: 4 nch_max + 4
    float *ring = wh + kWarps * (4 * nch_max + 4);
    for (int i = tid; i < nq * kQS2; i += 128) {
        const int ch = i >> 10, row = (i >> 4) & 63, b = i & 15;
        raw[i] = src_byte(row & 31, ch * 16 + b); // rows 32..63 repeat rows 0..31 (same data as mode 0)
    }
    for (int i = tid; i < 4 * nchunk + 4; i += 128) wv[i] = i >= zpad && i < zpad + L ? taps[i - zpad] : 0.0f;
    {
        float *w = wh + warp * (4 * nch_max + 4);
        for (int i = lane; i < 4 * nchunk_h + 4; i += 32) w[i] = i >= zf && i < zf + L ? taps[i - zf] * kTapScaleH : 0.0f;
    }
    for (int i = tid; i < kRowF * ipitch; i += 128) ring[i] = 0.0f;
    __syncthreads();
    const uint32_t raw_s = smem_u32(raw), ring_s = smem_u32(ring);
    unsigned sink = 0;
    const uint32_t wh_s = smem_u32(wh + warp * (4 * nch_max + 4));
    for (int it = 0; it < a.iters; it++) {
        for (int blk = 0; (a.hv & 1) && blk < nblk0; blk++) {
            float hA[kSegF], hB[kSegF];
            const uint32_t rowA = raw_s + (uint32_t)((a0 >> 4) * kQS2 + lane * kQB);
            h_bytes2(rowA, rowA + 32 * kQB, (uint32_t)rem * 8u, wh_s, nchunk_h, hA, hB);
            float *rp = ring + (size_t)(kSegF * warp) * ipitch + blk * 64 + lane + zpad;
#pragma unroll
            for (int j = 0; j < kSegF; j++) {
                rp[j * ipitch] = hA[j];
                rp[j * ipitch + 32] = hB[j];
            }
            if (a.hout && it == a.iters - 1 && blk == 0)
                for (int j = 0; j < kSegF; j++) {
                    a.hout[lane * 96 + kSegF * warp + j] = hA[j];
                    a.hout[(lane + 32) * 96 + kSegF * warp + j] = hB[j];
                }
        }
        __syncwarp();
        if (a.hv & 2) {
            const int gi = lane >> 3, px = lane & 7;
            float acc[kRV2][3];
            v_task16(ring_s + 4u * (uint32_t)((kSegF * warp + kC * px) * ipitch), 4u * (uint32_t)ipitch,
                     gi * kRV2, icap, smem_u32(wv), nchunk, acc);
#pragma unroll
            for (int j = 0; j < kRV2; j++)
#pragma unroll
                for (int k = 0; k < 3; k++) {
                    sink ^= __float_as_uint(acc[j][k]);
                    if (a.vout && it == a.iters - 1) a.vout[(gi * kRV2 + j) * 96 + kSegF * warp + kC * px + k] = acc[j][k];
                }
        }
        __syncwarp();
    }
    if (sink == 0x12345u) a.sink[blockIdx.x] = sink;
}

// ---- mode 2: H pass only, one row x 48 columns per lane (64-pixel strips, 4 warps x 48 columns)
__global__ void __launch_bounds__(128, 2) k_h48(proto_args a, const float *taps)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    const int L = a.L;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int a0 = a.skew + 48 * warp;
    const int d = a0 & 15, zf = d / 3, rem = d - 3 * zf;
    const int nchunk_h = (zf + L + 3) >> 2;
    const int nch_max = (5 + L + 3) >> 2;
    const int nq = (15 + 144 + 48 + 12 * nch_max + 64 + 15) / 16;
    const int ipitch = 68;
    unsigned char *raw = sm;
    float *wh = reinterpret_cast<float *>(sm + nq * kQS2);
    float *ring = wh + kWarps * (4 * nch_max + 4);
    for (int i = tid; i < nq * kQS2; i += 128) {
        const int ch = i >> 10, row = (i >> 4) & 63, b = i & 15;
        raw[i] = src_byte(row & 31, ch * 16 + b);
    }
    {
        float *w = wh + warp * (4 * nch_max + 4);
        for (int i = lane; i < 4 * nchunk_h + 4; i += 32) w[i] = i >= zf && i < zf + L ? taps[i - zf] * kTapScaleH : 0.0f;
    }
    __syncthreads();
    const uint32_t raw_s = smem_u32(raw);
    const uint32_t wh_s = smem_u32(wh + warp * (4 * nch_max + 4));
    unsigned sink = 0;
    for (int it = 0; it < a.iters; it++) {
        for (int half = 0; half < 2; half++) {
            float h[48];
            const uint32_t rowA = raw_s + (uint32_t)((a0 >> 4) * kQS2 + (lane + 32 * half) * kQB);
            h_bytes48(rowA, (uint32_t)rem * 8u, wh_s, nchunk_h, h);
            float *rp = ring + (size_t)(48 * warp) * ipitch + lane + 32 * half;
#pragma unroll
            for (int j = 0; j < 48; j++) rp[j * ipitch] = h[j];
            if (a.hout && it == a.iters - 1)
                for (int j = 0; j < 48; j++) a.hout[(lane + 32 * half) * 192 + 48 * warp + j] = h[j];
        }
        __syncwarp();
    }
    if (sink == 0x12345u) a.sink[blockIdx.x] = sink;
}

} // namespace

static void reference(int L, int skew_bytes, const std::vector<float> &taps, int rows, int vrows,
                      std::vector<float> &h, std::vector<float> &v)
{
    // H: out[row][col] = sum_k (g[k] 2^120) * (byte 2^-133), ascending k, first tap a plain product
    h.assign((size_t)rows * 96, 0.f);
    for (int row = 0; row < rows; row++)
        for (int c = 0; c < 96; c++) {
            float acc = 0.f;
            for (int k = 0; k < L; k++) {
                const float x = ldexpf((float)src_byte(row & 31, skew_bytes + c + 3 * k), -133);
                const float g = taps[k] * kTapScaleH;
                acc = k == 0 ? g * x : fmaf(g, x, acc);
            }
            h[(size_t)row * 96 + c] = acc;
        }
    v.assign((size_t)vrows * 96, 0.f);
    for (int y = 0; y < vrows; y++)
        for (int c = 0; c < 96; c++) {
            float acc = 0.f;
            for (int k = 0; k < L; k++) {
                const float x = h[(size_t)((y + k) & 31) * 96 + c]; // every block repeats rows 0..31
                acc = k == 0 ? taps[k] * x : fmaf(taps[k], x, acc);
            }
            v[(size_t)y * 96 + c] = acc;
        }
}

int main(int argc, char **argv)
{
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double peak = 2.0 * p.multiProcessorCount * 128 * khz * 1e3 / 1e12;
    printf("%s, %d SMs, nominal FP32 %.2f TFLOP/s\n", p.name, p.multiProcessorCount, peak);
    // usage: proto_ffma2 [L hv mode]   (one configuration, for ncu) or no arguments (sweep)
    const int oneL = argc > 3 ? atoi(argv[1]) : 0, one_hv = argc > 3 ? atoi(argv[2]) : 0, one_mode = argc > 3 ? atoi(argv[3]) : -1;
    const int Ls[] = {13, 23, 35, 47, 53, 69, 89};
    float *hout, *vout, *dtaps;
    unsigned *sink;
    cudaMalloc(&hout, 64 * 96 * 4);
    cudaMalloc(&vout, 64 * 96 * 4);
    cudaMalloc(&dtaps, 256 * 4);
    cudaMalloc(&sink, 4096 * 4);
    for (int L : Ls)
        for (int skew = 0; skew < 16; skew += (argc == 2 ? 1 : 7)) {
            if (oneL && (L != oneL || skew != 7)) continue;
            const int r = (L - 1) / 2, nchunk = (L + 3) / 4, zpad = 4 * nchunk - L;
            std::vector<float> taps(L);
            double s = 0;
            for (int k = 0; k < L; k++) { taps[k] = expf(-(float)((k - r) * (k - r)) / (2.f * (L / 6.f) * (L / 6.f))); s += taps[k]; }
            for (int k = 0; k < L; k++) taps[k] = (float)(taps[k] / s);
            cudaMemcpy(dtaps, taps.data(), L * 4, cudaMemcpyHostToDevice);
            std::vector<float> href, vref;
            for (int hv = 1; hv <= 3; hv++)
            for (int mode = 0; mode < 2; mode++) {
                if (oneL && (hv != one_hv || mode != one_mode)) continue;
                // old: stream starts 3 zpad bytes before the tile (skew = byte of the STREAM start);
                // new: skew = byte of the TILE start.  Same tile: tile byte 0 = source byte skew + 3 zpad (old)
                const int tile0 = skew + 3 * zpad;
                size_t smem;
                int rows_h, vrows;
                if (mode == 0) {
                    const int nq = (168 + 6 * r + 15) / 16, rows_in = (32 + 2 * r + 31) / 32 * 32 + 4;
                    const int icap = (rows_in + 3) & ~3, ipitch = (icap & 7) == 4 ? icap : icap + 4;
                    smem = nq * 512 + (2 * (4 * nchunk + 4) + kRowF * ipitch) * 4;
                    rows_h = 32, vrows = 32;
                } else {
                    const int nch_max = (5 + L + 3) >> 2;
                    const int nq = (15 + 72 + 24 + 12 * nch_max + 16 + 16 + 15) / 16, rows_in = (64 + 2 * r + 63) / 64 * 64 + 4;
                    const int icap = (rows_in + 3) & ~3, ipitch = (icap & 7) == 4 ? icap : icap + 4;
                    smem = nq * kQS2 + ((4 * nchunk + 4) + kWarps * (4 * nch_max + 4) + kRowF * ipitch) * 4;
                    rows_h = 64, vrows = 64;
                }
                proto_args a{L, mode == 0 ? skew : tile0, kIters, hv, hv == 3 ? hout : nullptr, hv == 3 ? vout : nullptr, sink};
                int occ = 0;
                if (mode == 0) {
                    cudaFuncSetAttribute(k_old, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_old, 128, smem);
                } else {
                    cudaFuncSetAttribute(k_new, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_new, 128, smem);
                }
                const int grid = p.multiProcessorCount * occ;
                cudaMemset(hout, 0, 64 * 96 * 4);
                cudaMemset(vout, 0, 64 * 96 * 4);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                float best = 1e30f;
                for (int rep = 0; rep < 3; rep++) {
                    cudaEventRecord(e0);
                    if (mode == 0) k_old<<<grid, 128, smem>>>(a, dtaps);
                    else k_new<<<grid, 128, smem>>>(a, dtaps);
                    cudaEventRecord(e1);
                    cudaError_t e = cudaEventSynchronize(e1);
                    if (e != cudaSuccess) { printf("launch failed: %s\n", cudaGetErrorString(e)); return 1; }
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    best = ms < best ? ms : best;
                }
                // useful FMAs per iteration per CTA (real taps only)
                const int nblk = mode == 0 ? (32 + 2 * r + 31) / 32 : (64 + 2 * r + 63) / 64;
                const double fma_it = (hv & 1 ? (double)nblk * rows_h * 96 * L : 0.0) + (hv & 2 ? (double)vrows * 96 * L : 0.0);
                const double tf = 2.0 * fma_it * kIters * grid / (best * 1e-3) / 1e12;
                // check
                std::vector<float> hg(64 * 96), vg(64 * 96);
                cudaMemcpy(hg.data(), hout, hg.size() * 4, cudaMemcpyDeviceToHost);
                cudaMemcpy(vg.data(), vout, vg.size() * 4, cudaMemcpyDeviceToHost);
                reference(L, tile0, taps, rows_h, vrows, href, vref);
                long badh = 0, badv = 0;
                for (int i = 0; i < rows_h * 96; i++) badh += memcmp(&hg[i], &href[i], 4) != 0;
                // V outputs are comparable only when the ring holds whole periods of rows: compare H always,
                // V when the intermediate rows repeat with period 32 (they do: rows & 31)
                for (int i = 0; i < vrows * 96; i++) badv += memcmp(&vg[i], &vref[i], 4) != 0;
                printf("L %3d skew %2d hv %d %s occ %d  %8.3f ms  %6.2f TFLOP/s %5.1f%%  H bad %ld  V bad %ld\n", L, skew, hv,
                       mode ? "wide " : "ffma ", occ, best, tf, 100 * tf / peak, badh, badv);
                if (mode == 1 && hv == 1) { /* the 48-column H task, H only */
                    const int nch_max = (5 + L + 3) >> 2;
                    const int nq = (15 + 144 + 48 + 12 * nch_max + 64 + 15) / 16;
                    const size_t sm48 = nq * kQS2 + (kWarps * (4 * nch_max + 4) + 192 * 68) * 4;
                    float *h48;
                    cudaMalloc(&h48, 64 * 192 * 4);
                    proto_args a48{L, tile0, kIters, 1, h48, nullptr, sink};
                    cudaFuncSetAttribute(k_h48, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm48);
                    int occ48 = 0;
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ48, k_h48, 128, sm48);
                    const int grid48 = p.multiProcessorCount * occ48;
                    float best48 = 1e30f;
                    for (int rep = 0; rep < 3; rep++) {
                        cudaEventRecord(e0);
                        k_h48<<<grid48, 128, sm48>>>(a48, dtaps);
                        cudaEventRecord(e1);
                        if (cudaEventSynchronize(e1) != cudaSuccess) { printf("h48 launch failed\n"); return 1; }
                        float ms;
                        cudaEventElapsedTime(&ms, e0, e1);
                        best48 = ms < best48 ? ms : best48;
                    }
                    const double tf48 = 2.0 * 64.0 * 192 * L * kIters * grid48 / (best48 * 1e-3) / 1e12;
                    std::vector<float> hg48(64 * 192);
                    cudaMemcpy(hg48.data(), h48, hg48.size() * 4, cudaMemcpyDeviceToHost);
                    long bad48 = 0; /* reference: 192 columns of the same byte stream */
                    for (int row = 0; row < 64; row++)
                        for (int c2 = 0; c2 < 192; c2++) {
                            float acc = 0.f;
                            for (int k2 = 0; k2 < L; k2++) {
                                const float x = ldexpf((float)src_byte(row & 31, tile0 + c2 + 3 * k2), -133);
                                const float g = taps[k2] * kTapScaleH;
                                acc = k2 == 0 ? g * x : fmaf(g, x, acc);
                            }
                            bad48 += memcmp(&acc, &hg48[row * 192 + c2], 4) != 0;
                        }
                    printf("L %3d skew %2d hv 1 h48   occ %d  %8.3f ms  %6.2f TFLOP/s %5.1f%%  H bad %ld\n", L, skew, occ48,
                           best48, tf48, 100 * tf48 / peak, bad48);
                    cudaFree(h48);
                }

            }
        }
    return 0;
}
