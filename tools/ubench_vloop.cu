// Ablation of the V-pass chunk loop on B200: what does each ingredient cost?
//   M0  FFMA pattern only (window and taps static in registers)
//   M1  + one tap LDS.128 per chunk (prefetched a chunk ahead)
//   M2  + three window LDS.128 per chunk into the ring (conflict-free addresses)
//   M3  M2 with the window loads as 6 LDS.64
//   M4  M2 with taps read by LDS.128 from ONE address by all lanes (broadcast) -- same as M1/M2 really
//   M5  M0 + 4 LDS.128 per chunk whose results are never used by an FFMA (xor-folded at the end)
// All modes: 96 FFMA per chunk, four chunk phases unrolled, 3 or 4 CTAs of 128 threads per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_vloop.bin tools/ubench_vloop.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 lds128(unsigned addr)
{
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ float2 lds64(unsigned addr)
{
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

template <int MODE, int MINB> __global__ void __launch_bounds__(128, MINB) k(const float *in, float *out, int turns)
{
    extern __shared__ __align__(16) float sm[];
    for (int i = threadIdx.x; i < 8192; i += 128) sm[i] = in[i & 1023];
    __syncthreads();
    const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
    // a lane's column: pitch 4 (mod 8) floats between lanes' columns, like the intermediate
    const unsigned col = base + (threadIdx.x & 31) * 3 * 4 * 52 + (threadIdx.x >> 5) * 16;
    const unsigned cp = 4 * 52;
    float win[3][16], acc[8][3];
#pragma unroll
    for (int k2 = 0; k2 < 3; k2++)
#pragma unroll
        for (int i = 0; i < 16; i++) win[k2][i] = in[(threadIdx.x + 16 * k2 + i) & 255];
#pragma unroll
    for (int j = 0; j < 8; j++)
#pragma unroll
        for (int k2 = 0; k2 < 3; k2++) acc[j][k2] = 0.f;
    float4 g4 = lds128(base + 16 * 500);
    unsigned wa = base + 16 * 500, a = col;
    unsigned junk = 0;
    for (int turn = 0; turn < turns; turn++) {
#pragma unroll
        for (int p = 0; p < 4; p++) {
            const float g[4] = {g4.x, g4.y, g4.z, g4.w};
            if (MODE >= 1 && MODE != 5) {
                g4 = lds128(wa + 16 * p);
            }
            if (MODE == 2 || MODE == 4) {
#pragma unroll
                for (int k2 = 0; k2 < 3; k2++) {
                    const float4 x = lds128(a + k2 * cp + 16 * p);
                    win[k2][(4 * (p + 3) + 0) % 16] = x.x;
                    win[k2][(4 * (p + 3) + 1) % 16] = x.y;
                    win[k2][(4 * (p + 3) + 2) % 16] = x.z;
                    win[k2][(4 * (p + 3) + 3) % 16] = x.w;
                }
            }
            if (MODE == 3) {
#pragma unroll
                for (int k2 = 0; k2 < 3; k2++) {
                    const float2 x = lds64(a + k2 * cp + 16 * p), y = lds64(a + k2 * cp + 16 * p + 8);
                    win[k2][(4 * (p + 3) + 0) % 16] = x.x;
                    win[k2][(4 * (p + 3) + 1) % 16] = x.y;
                    win[k2][(4 * (p + 3) + 2) % 16] = y.x;
                    win[k2][(4 * (p + 3) + 3) % 16] = y.y;
                }
            }
            if (MODE == 5) {
#pragma unroll
                for (int k2 = 0; k2 < 4; k2++) {
                    const float4 x = lds128(a + k2 * cp + 16 * p);
                    junk ^= __float_as_uint(x.x) ^ __float_as_uint(x.w);
                }
            }
#pragma unroll
            for (int t = 0; t < 4; t++)
#pragma unroll
                for (int j = 0; j < 8; j++)
#pragma unroll
                    for (int k2 = 0; k2 < 3; k2++)
                        acc[j][k2] = fmaf(g[t], win[k2][(4 * p + t + j) % 16], acc[j][k2]);
        }
        wa = base + 16 * (500 + (turn & 3) * 4);
        a = col + ((turn & 1) ? 64 : 0);
    }
    float s = __uint_as_float(junk) + g4.x;
#pragma unroll
    for (int j = 0; j < 8; j++)
#pragma unroll
        for (int k2 = 0; k2 < 3; k2++) s += acc[j][k2];
    if (s == 12345.678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int MINB> void run(const char *name, int sms, double peak, const float *in, float *out)
{
    const int turns = 3000;
    auto kern = k<MODE, MINB>;
    size_t smem = (227 * 1024) / MINB - 2048;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem);
    const int grid = sms * occ;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
        cudaEventRecord(e0);
        kern<<<grid, 128, smem>>>(in, out, turns);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double fmas = 4.0 * 96 * (double)turns * grid * 128;
    const double tf = 2.0 * fmas / (best * 1e-3) / 1e12;
    printf("%-44s warps/SM %2d  %7.2f TFLOP/s  %5.1f%% of peak\n", name, occ * 4, tf, 100.0 * tf / peak);
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
#define RUN(M, name) run<M, 3>(name, sms, peak, in, out); run<M, 4>(name, sms, peak, in, out);
    RUN(0, "M0 pattern only");
    RUN(1, "M1 + tap LDS.128 / chunk");
    RUN(2, "M2 + 3 window LDS.128 / chunk");
    RUN(3, "M3 window as 6 LDS.64 / chunk");
    RUN(5, "M5 pattern + 4 unused LDS.128 / chunk");
    return 0;
}
