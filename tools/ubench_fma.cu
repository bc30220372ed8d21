// Microbenchmarks that size the blur kernel's inner loop on B200 (sm_100a):
//   ffma      : 16 independent FFMA chains per thread
//   ffma2     : 8 independent packed fma.rn.f32x2 chains per thread (same FMA count)
//   ffma2+alu : ffma2 with one independent integer op per packed FMA (issue-slot test)
//   ffma+alu  : ffma with one independent integer op per 2 FMAs
//   ffma2+lds : ffma2 with one LDS.128 per 16 packed FMAs (the blur loop's ratio)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_fma tools/ubench_fma.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c)
{
    float2 d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(*reinterpret_cast<unsigned long long *>(&d))
        : "l"(*reinterpret_cast<unsigned long long *>(&a)),
          "l"(*reinterpret_cast<unsigned long long *>(&b)),
          "l"(*reinterpret_cast<unsigned long long *>(&c)));
    return d;
}

template <int MODE> __global__ void __launch_bounds__(256) k(float *out, int iters)
{
    __shared__ float4 sm[256];
    sm[threadIdx.x] = make_float4(1.f, 2.f, 3.f, 4.f);
    __syncthreads();
    const float x = 1.0f + 1e-7f * threadIdx.x, y = 1e-9f * blockIdx.x;
    float a[16];
    float2 p[8];
    unsigned u[8];
#pragma unroll
    for (int i = 0; i < 16; i++) a[i] = (float)i;
#pragma unroll
    for (int i = 0; i < 8; i++) { p[i] = make_float2(i, i + 0.5f); u[i] = threadIdx.x + i; }
    const float2 x2 = make_float2(x, x), y2 = make_float2(y, y);
    float4 acc4 = make_float4(0, 0, 0, 0);
    for (int it = 0; it < iters; it++) {
        if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 16; i++) a[i] = fmaf(a[i], x, y);
        } else if (MODE == 1) {
#pragma unroll
            for (int i = 0; i < 8; i++) p[i] = ffma2(p[i], x2, y2);
        } else if (MODE == 2) {
#pragma unroll
            for (int i = 0; i < 8; i++) { p[i] = ffma2(p[i], x2, y2); u[i] = (u[i] ^ (u[i] >> 3)) + 0x9e3779b9u; }
        } else if (MODE == 3) {
#pragma unroll
            for (int i = 0; i < 16; i++) { a[i] = fmaf(a[i], x, y); if (i & 1) u[i >> 1] = (u[i >> 1] ^ (u[i >> 1] >> 3)) + 0x9e3779b9u; }
        } else if (MODE == 4) {
#pragma unroll
            for (int r = 0; r < 2; r++) {
#pragma unroll
                for (int i = 0; i < 8; i++) p[i] = ffma2(p[i], x2, y2);
            }
            float4 v = sm[(threadIdx.x + it) & 255];
            acc4.x += v.x; 
        } else if (MODE == 5) {
#pragma unroll
            for (int r = 0; r < 2; r++) {
#pragma unroll
                for (int i = 0; i < 16; i++) a[i] = fmaf(a[i], x, y);
            }
            float4 v = sm[(threadIdx.x + it) & 255];
            acc4.x += v.x;
        }
    }
    float s = acc4.x;
#pragma unroll
    for (int i = 0; i < 16; i++) s += a[i];
#pragma unroll
    for (int i = 0; i < 8; i++) s += p[i].x + p[i].y + (float)u[i];
    if (s == 12345.678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE> void run(const char *name, double fma_per_iter, int sms)
{
    float *buf;
    cudaMalloc(&buf, sizeof(float) * sms * 8 * 256);
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 2; w++) k<MODE><<<sms * 8, 256>>>(buf, iters);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        k<MODE><<<sms * 8, 256>>>(buf, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    double flops = 2.0 * fma_per_iter * iters * (double)sms * 8 * 256;
    printf("%-10s %8.3f ms  %7.2f TFLOP/s\n", name, best, flops / (best * 1e-3) / 1e12);
    cudaFree(buf);
}

int main()
{
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    printf("%s, %d SMs\n", p.name, p.multiProcessorCount);
    int sms = p.multiProcessorCount;
    run<0>("ffma", 16, sms);
    run<1>("ffma2", 16, sms);
    run<2>("ffma2+alu", 16, sms);
    run<3>("ffma+alu", 16, sms);
    run<4>("ffma2+lds", 32, sms);
    run<5>("ffma+lds", 32, sms);
    return 0;
}
