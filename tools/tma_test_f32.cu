// Standalone check of the 4-D float32 "shifted quad grid" TMA box used by fk_blur_tma<float>:
// dims (D0, H, W*C/4 - 1, N) with strides (pitch, 16 B, frame), box (4, 32, nq, 1).
// usage: tma_test_f32 D0 c0 [q0] [y0]   (one configuration per process: a faulting TMA kills the context)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_test_f32 tools/tma_test_f32.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr int NQ = 12, ROWS = 32, BYTES = NQ * ROWS * 16;

__global__ void k(const __grid_constant__ CUtensorMap tmap, float *out, int c0, int c1, int c2, int c3)
{
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + BYTES);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(BYTES) : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                     ::"r"(smem_u32(smem)), "l"(&tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
    }
    __syncthreads();
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra D;\n\tbra W;\n\tD:\n\t}"
                 ::"r"(smem_u32(bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < BYTES / 4; i += blockDim.x) out[i] = reinterpret_cast<float *>(smem)[i];
}

int main(int argc, char **argv)
{
    const int D0 = argc > 1 ? atoi(argv[1]) : 7, c0 = argc > 2 ? atoi(argv[2]) : 1;
    const int q0 = argc > 3 ? atoi(argv[3]) : 2, y0 = argc > 4 ? atoi(argv[4]) : 3;
    const int WC = 96, H = 64, N = 2;
    std::vector<float> h((size_t)WC * H * N);
    for (size_t i = 0; i < h.size(); i++) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, BYTES);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void *fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    typedef CUresult (*enc_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                              const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    CUtensorMap map;
    const int NQG = D0 > 4 ? WC / 4 - 1 : WC / 4;
    cuuint64_t dims[4] = {(cuuint64_t)D0, H, (cuuint64_t)NQG, N};
    cuuint64_t strides[3] = {(cuuint64_t)WC * 4, 16, (cuuint64_t)WC * 4 * H};
    cuuint32_t box[4] = {4, ROWS, NQ, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = ((enc_t)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("D0=%d c0=%d q0=%d y0=%d encode rc=%d\n", D0, c0, q0, y0, (int)r);
    if (r != CUDA_SUCCESS) return 1;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaMemset(o, 0xEE, BYTES);
    k<<<1, 128, 64 * 1024>>>(map, o, c0, y0, q0, 1);
    cudaError_t e = cudaDeviceSynchronize();
    printf("run: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 2;
    std::vector<float> got(BYTES / 4);
    cudaMemcpy(got.data(), o, BYTES, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int qq = 0; qq < NQ; qq++) for (int y = 0; y < ROWS; y++) for (int i = 0; i < 4; i++) {
        const int gq = q0 + qq, gy = y0 + y, gi = c0 + i;
        const bool in = gq >= 0 && gq < NQG && gy >= 0 && gy < H && gi >= 0 && gi < D0;
        const float want = in ? h[((size_t)1 * H + gy) * WC + 4 * gq + gi] : 0.0f;
        const float g = got[(qq * ROWS + y) * 4 + i];
        if (g != want) { if (bad < 5) printf("  q %d y %d i %d: got %g want %g\n", qq, y, i, g, want); bad++; }
    }
    printf("mismatches %ld\n", bad);
    return bad != 0;
}
