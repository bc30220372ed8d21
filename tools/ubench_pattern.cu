// What FMA rate does the OPERAND PATTERN of the blur loops sustain on B200, with no loads at
// all?  acc[j] = fma(g[t], win[(3t + j) % 48], acc[j]) reads two fresh registers per FFMA (the
// tap comes from the operand reuse cache); the classic peak probe acc = fma(x, y, acc) reads one.
//   P0  acc[j] += x * y            (x, y loop-invariant: one fresh operand)
//   P1  acc[j] += g * win[j]       (two fresh operands, window index = accumulator index)
//   P2  acc[j] += g[t] * win[3t+j] (the H-pass pattern)
//   Q1/Q2  the same with packed fma.rn.f32x2 (24 accumulator pairs)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_pattern tools/ubench_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c)
{
    u64 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ u64 pack2(float lo, float hi)
{
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}

template <int MODE, int MINB> __global__ void __launch_bounds__(128, MINB) k(const float *in, float *out, int iters)
{
    float win[48], g[4];
#pragma unroll
    for (int i = 0; i < 48; i++) win[i] = in[(threadIdx.x + i) & 255];
#pragma unroll
    for (int i = 0; i < 4; i++) g[i] = in[256 + i];
    float s = 0.f;
    if (MODE <= 2) {
        float acc[24];
#pragma unroll
        for (int j = 0; j < 24; j++) acc[j] = 0.f;
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int p = 0; p < 4; p++)
#pragma unroll
                for (int t = 0; t < 4; t++)
#pragma unroll
                    for (int j = 0; j < 24; j++) {
                        if (MODE == 0) acc[j] = fmaf(g[0], g[1], acc[j]);
                        if (MODE == 1) acc[j] = fmaf(g[t], win[j], acc[j]);
                        if (MODE == 2) acc[j] = fmaf(g[t], win[(12 * p + 3 * t + j) % 48], acc[j]);
                    }
        }
#pragma unroll
        for (int j = 0; j < 24; j++) s += acc[j];
    } else {
        u64 acc[24], w2[48], g2[4];
#pragma unroll
        for (int j = 0; j < 24; j++) acc[j] = 0ull;
#pragma unroll
        for (int i = 0; i < 48; i++) w2[i] = pack2(win[i], win[47 - i]);
#pragma unroll
        for (int i = 0; i < 4; i++) g2[i] = pack2(g[i], g[i]);
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int p = 0; p < 4; p++)
#pragma unroll
                for (int t = 0; t < 4; t++)
#pragma unroll
                    for (int j = 0; j < 24; j++) {
                        if (MODE == 3) acc[j] = ffma2(g2[t], w2[j], acc[j]);
                        if (MODE == 4) acc[j] = ffma2(g2[t], w2[(12 * p + 3 * t + j) % 48], acc[j]);
                    }
        }
#pragma unroll
        for (int j = 0; j < 24; j++) {
            float lo, hi;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[j]));
            s += lo + hi;
        }
    }
    if (s == 12345.678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int MINB> void run(const char *name, int sms, double peak, const float *in, float *out)
{
    const int iters = 4000;
    auto kern = k<MODE, MINB>;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, 0);
    if (occ > MINB) occ = MINB;
    // limit residency to MINB CTAs per SM with dynamic shared memory
    size_t smem = (227 * 1024) / MINB - 2048;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem);
    const int grid = sms * occ;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
        cudaEventRecord(e0);
        kern<<<grid, 128, smem>>>(in, out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double fmas = (MODE <= 2 ? 1.0 : 2.0) * 4 * 4 * 24 * (double)iters * grid * 128;
    const double tf = 2.0 * fmas / (best * 1e-3) / 1e12;
    printf("%-34s warps/SM %2d  %7.2f TFLOP/s  %5.1f%% of peak\n", name, occ * 4, tf, 100.0 * tf / peak);
}

int main()
{
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double peak = 2.0 * p.multiProcessorCount * 128 * khz * 1e3 / 1e12;
    printf("%s, %d SMs, nominal FP32 %.2f TFLOP/s\n", p.name, p.multiProcessorCount, peak);
    float *in, *out;
    cudaMalloc(&in, 1024 * 4);
    cudaMalloc(&out, 4 << 20);
    float h[1024];
    for (int i = 0; i < 1024; i++) h[i] = 1.0f / (1 + i);
    cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
    const int sms = p.multiProcessorCount;
#define RUN(M, name) run<M, 2>(name, sms, peak, in, out); run<M, 3>(name, sms, peak, in, out); run<M, 4>(name, sms, peak, in, out);
    RUN(0, "P0 acc += x*y");
    RUN(1, "P1 acc[j] += g[t]*win[j]");
    RUN(2, "P2 acc[j] += g[t]*win[3t+j]");
    RUN(3, "Q1 ffma2 acc[j] += g[t]*win[j]");
    RUN(4, "Q2 ffma2 acc[j] += g[t]*win[3t+j]");
    return 0;
}
