// Standalone check of the TMA box load used by fk_blur_fast (u8 3-D tensor, 128x32x1 box).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_test tools/tma_test.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tmap, unsigned char *out, int c0, int c1, int c2, unsigned *info)
{
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 4096);
    if (threadIdx.x == 0) {
        info[0] = smem_u32(smem);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(4096) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                     ::"r"(smem_u32(smem)), "l"(&tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
    }
    __syncthreads();
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@p bra D;\n\tbra W;\n\tD:\n\t}"
                 ::"r"(smem_u32(bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = smem[i];
}

int main()
{
    const int W = 128, H = 96, N = 2;
    std::vector<unsigned char> h(W * H * N);
    for (size_t i = 0; i < h.size(); i++) h[i] = (unsigned char)(i * 7 + i / W);
    unsigned char *d, *o; unsigned *info;
    cudaMalloc(&d, h.size()); cudaMalloc(&o, 4096); cudaMalloc(&info, 16);
    cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
    void *fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    typedef CUresult (*enc_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                              const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    CUtensorMap map;
    cuuint64_t dims[3] = {W, H, N}, strides[2] = {W, (cuuint64_t)W * H};
    cuuint32_t box[3] = {128, 32, 1}, es[3] = {1, 1, 1};
    CUresult r = ((enc_t)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)r);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    int tests[][3] = {{0, 0, 0}, {16, 3, 1}, {5, 3, 0}, {-7, -4, 1}, {100, 80, 1}, {3, 70, 0}};
    for (auto &t : tests) {
        cudaMemset(o, 0xEE, 4096);
        k<<<1, 128, 100 * 1024>>>(map, o, t[0], t[1], t[2], info);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<unsigned char> got(4096); unsigned inf[4];
        cudaMemcpy(got.data(), o, 4096, cudaMemcpyDeviceToHost);
        cudaMemcpy(inf, info, 16, cudaMemcpyDeviceToHost);
        long bad = 0;
        for (int y = 0; y < 32; y++) for (int x = 0; x < 128; x++) {
            int gx = t[0] + x, gy = t[1] + y;
            unsigned char want = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? h[((size_t)t[2] * H + gy) * W + gx] : 0;
            bad += got[y * 128 + x] != want;
        }
        printf("coords (%d,%d,%d): %s, smem base 0x%x, mismatches %ld\n", t[0], t[1], t[2], cudaGetErrorString(e), inf[0], bad);
        if (e != cudaSuccess) break;
    }
    return 0;
}
