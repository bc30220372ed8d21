// Does an FFMA whose two non-reused sources sit in the same register bank (same parity)
// issue at half rate on B200?  acc and A are float4 arrays kept in aligned register quads
// by 128-bit loads/stores; variant 0 pairs acc[q].c with A[q].c (same parity), variant 1
// with A[q].(c^1) (opposite parity).  The tap g is the .reuse operand in both.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_bank tools/ubench_bank.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int VAR> __global__ void __launch_bounds__(128) k(const float4 *in, float4 *out, int iters, float g0)
{
    __shared__ float4 sm[128 * 6];
    for (int q = 0; q < 6; q++) sm[q * 128 + threadIdx.x] = in[(q * 128 + threadIdx.x) % 64];
    __syncthreads();
    float4 A[6], acc[6];
#pragma unroll
    for (int q = 0; q < 6; q++) { A[q] = sm[q * 128 + threadIdx.x]; acc[q] = make_float4(0, 0, 0, 0); }
    float g = g0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int rep = 0; rep < 4; rep++) {
#pragma unroll
            for (int q = 0; q < 6; q++) {
                if (VAR == 0) {
                    acc[q].x = fmaf(g, A[q].x, acc[q].x); acc[q].y = fmaf(g, A[q].y, acc[q].y);
                    acc[q].z = fmaf(g, A[q].z, acc[q].z); acc[q].w = fmaf(g, A[q].w, acc[q].w);
                } else {
                    acc[q].x = fmaf(g, A[q].y, acc[q].x); acc[q].y = fmaf(g, A[q].x, acc[q].y);
                    acc[q].z = fmaf(g, A[q].w, acc[q].z); acc[q].w = fmaf(g, A[q].z, acc[q].w);
                }
            }
        }
        g += 1e-9f;
    }
#pragma unroll
    for (int q = 0; q < 6; q++) out[(blockIdx.x * 6 + q) * 128 + threadIdx.x] = acc[q];
}

template <int VAR> void run(const char *name, int sms)
{
    float4 *in, *out;
    cudaMalloc(&in, 64 * sizeof(float4)); cudaMemset(in, 0, 64 * sizeof(float4));
    cudaMalloc(&out, (size_t)sms * 8 * 6 * 128 * sizeof(float4));
    const int iters = 20000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<VAR><<<sms * 8, 128>>>(in, out, iters, 0.5f);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0); k<VAR><<<sms * 8, 128>>>(in, out, iters, 0.5f); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    double flops = 2.0 * 96.0 * iters * (double)sms * 8 * 128;
    printf("%-28s %8.3f ms %7.2f TFLOP/s\n", name, best, flops / (best * 1e-3) / 1e12);
}

int main()
{
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("%s\n", p.name);
    run<0>("same parity (acc.c, A.c)", p.multiProcessorCount);
    run<1>("opposite parity (acc.c, A.c^1)", p.multiProcessorCount);
    return 0;
}
