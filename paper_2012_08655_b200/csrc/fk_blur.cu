/*
 * fk_blur.cu -- per-fragment separable Gaussian blur (sm_100a).
 *
 * Replaces blockwise.py:136-186 (_render_cell / render) and convolve.py:9-15
 * (quantize_u8): clamp-to-edge gather of the fragment plus its halo, horizontal pass
 * over every tile row into a real-valued intermediate, vertical pass, one rounding.
 * Arithmetic is fp32 (weights and accumulators); the reference's is fp64, the parity
 * bar is +-1 LSB on uint8 and 1e-4 relative on float32 frames.
 *
 * Kernels
 *   fk_blur_generic  any tap count, any geometry: intermediate in shared memory,
 *                    input read straight from global/L2.  Correctness baseline and
 *                    fallback for fragments the fast kernel does not take.
 */
#include "fk_internal.h"

namespace {

template <typename T> struct fk_px;
template <> struct fk_px<uint8_t> {
    static __device__ __forceinline__ float load(const uint8_t *p) { return (float)*p; }
    static __device__ __forceinline__ uint8_t store(float v)
    {
        /* convolve.py:15: clip(floor(v + 0.5), 0, 255) */
        v = floorf(v + 0.5f);
        v = fminf(fmaxf(v, 0.0f), 255.0f);
        return (uint8_t)v;
    }
};
template <> struct fk_px<float> {
    static __device__ __forceinline__ float load(const float *p) { return *p; }
    static __device__ __forceinline__ float store(float v) { return v; }
};

__device__ __forceinline__ void fk_span_dev(int extent, int F, int off, int g, int &a, int &b)
{
    const int lead = off > 0 ? 1 : 0;
    if (lead && g == 0) {
        a = 0;
        b = off < extent ? off : extent;
    } else {
        a = off + (g - lead) * F;
        b = a + F < extent ? a + F : extent;
    }
}

__device__ __forceinline__ int fk_clamp(int v, int lo, int hi)
{
    return v < lo ? lo : (v > hi ? hi : v);
}

/*
 * One CTA per (frame, order slot).  Shared memory: taps[w_floats] then the H-pass
 * intermediate, interm_floats floats; fragments whose (fh + 2r) * fw * C intermediate
 * does not fit are processed in column strips.
 */
template <typename T>
__global__ void __launch_bounds__(256)
fk_blur_generic(fk_plan_dev pd, const T *__restrict__ in, T *__restrict__ out, int n_frames,
                int C, int w_floats, int interm_floats)
{
    extern __shared__ float smem[];
    float *wts = smem;
    float *interm = smem + w_floats;

    const int f = blockIdx.x / pd.cap;
    const int slot = blockIdx.x - f * pd.cap;
    if (f >= n_frames) return;
    const int32_t *meta = pd.meta + (size_t)f * FK_META_WORDS;
    if (meta[FK_META_STATUS] != 0) return;
    const int gw = meta[FK_META_GW], gh = meta[FK_META_GH];
    if (slot >= gw * gh) return;
    const int cell = (int)pd.order[(size_t)f * pd.cap + slot];
    const int gy = cell / gw, gx = cell - gy * gw;
    const int W = pd.width, H = pd.height;
    int x0, x1, y0, y1;
    fk_span_dev(W, pd.fragment, meta[FK_META_SX], gx, x0, x1);
    fk_span_dev(H, pd.fragment, meta[FK_META_SY], gy, y0, y1);
    const int L = pd.length[(size_t)f * pd.cap + cell];
    const int fw = x1 - x0, fh = y1 - y0;
    const size_t frame_off = (size_t)f * H * W * C;
    const T *src = in + frame_off;
    T *dst = out + frame_off;
    const int tid = threadIdx.x, nt = blockDim.x;

    if (L == 1) { /* blockwise.py:141-143: identity fragments are copied through */
        const int rowlen = fw * C;
        for (int i = tid; i < fh * rowlen; i += nt) {
            const int y = i / rowlen, c = i - y * rowlen;
            const size_t o = ((size_t)(y0 + y) * W + x0) * C + c;
            dst[o] = src[o];
        }
        return;
    }
    const int r = (L - 1) >> 1;
    const float *taps = pd.taps + pd.offset[(size_t)f * pd.cap + cell];
    for (int i = tid; i < L; i += nt) wts[i] = taps[i];

    const int th = fh + 2 * r;
    int ws = interm_floats / (th * C);
    ws = ws > fw ? fw : ws;
    if (ws < 1) return; /* host sizes the buffer so that this cannot happen */
    __syncthreads();

    for (int xs = x0; xs < x1; xs += ws) {
        const int sw = (x1 - xs) < ws ? (x1 - xs) : ws;
        const int cols = sw * C;
        /* horizontal pass over every tile row (blockwise.py:151) */
        for (int i = tid; i < th * cols; i += nt) {
            const int ty = i / cols, col = i - ty * cols;
            const int px = col / C, c = col - px * C;
            const int yy = fk_clamp(y0 - r + ty, 0, H - 1);
            const T *row = src + (size_t)yy * W * C + c;
            const int xb = xs + px - r;
            float acc = 0.0f;
            for (int k = 0; k < L; k++) {
                const int xx = fk_clamp(xb + k, 0, W - 1);
                acc = fmaf(wts[k], fk_px<T>::load(row + (size_t)xx * C), acc);
            }
            interm[i] = acc;
        }
        __syncthreads();
        /* vertical pass over the real-valued intermediate (blockwise.py:152-153) */
        for (int i = tid; i < fh * cols; i += nt) {
            const int y = i / cols, col = i - y * cols;
            const float *colp = interm + (size_t)y * cols + col;
            float acc = 0.0f;
            for (int k = 0; k < L; k++) acc = fmaf(wts[k], colp[(size_t)k * cols], acc);
            dst[((size_t)(y0 + y) * W + xs) * C + col] = fk_px<T>::store(acc);
        }
        __syncthreads();
    }
}

/* FP32 peak probe: 16 independent FFMA chains per thread, no memory traffic. */
__global__ void __launch_bounds__(256) fk_fp32_probe(float *out, int iters)
{
    float a[16];
    const float x = 1.0f + 1e-7f * (float)threadIdx.x, y = 1e-9f * (float)blockIdx.x;
#pragma unroll
    for (int i = 0; i < 16; i++) a[i] = (float)i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) a[i] = fmaf(a[i], x, y);
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; i++) s += a[i];
    if (s == 12345.678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

} // namespace

cudaError_t fk_launch_fp32_probe(float *buf, int sm_count, int iters, cudaStream_t s)
{
    fk_fp32_probe<<<sm_count * 8, 256, 0, s>>>(buf, iters);
    return cudaGetLastError();
}

cudaError_t fk_launch_blur(fk_handle *h, const fk_plan_dev &pd, const void *in, void *out,
                           int n_frames, int channels, int is_f32, int bound_length,
                           cudaStream_t s, int *launches)
{
    if (h->variant != 1) { /* fast path unless the generic kernel is forced */
        bool taken = false;
        cudaError_t fe = fk_launch_blur_fast(h, pd, in, out, n_frames, channels, is_f32,
                                             bound_length, s, &taken);
        if (fe != cudaSuccess) return fe;
        if (taken) {
            *launches += 1;
            return cudaSuccess;
        }
    }
    const int F = pd.fragment;
    const int r = (bound_length - 1) / 2;
    const int w_floats = (bound_length + 3) & ~3;
    const int max_smem = (int)h->prop.sharedMemPerBlockOptin;
    /* whole fragment if it fits in ~96 KB (2 CTAs/SM), else strips down to one column */
    long long want = (long long)(F + 2 * r) * F * channels;
    long long cap_floats = (96 * 1024) / 4 - w_floats;
    long long min_floats = (long long)(F + 2 * r) * channels;
    if (cap_floats < min_floats) cap_floats = min_floats;
    long long interm = want < cap_floats ? want : cap_floats;
    size_t smem = (size_t)(w_floats + interm) * sizeof(float);
    if (smem > (size_t)max_smem) return cudaErrorInvalidConfiguration;
    const long long blocks = (long long)n_frames * pd.cap;
    if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    cudaError_t e;
    if (is_f32) {
        e = cudaFuncSetAttribute(fk_blur_generic<float>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        fk_blur_generic<float><<<(unsigned)blocks, 256, smem, s>>>(
            pd, (const float *)in, (float *)out, n_frames, channels, w_floats, (int)interm);
    } else {
        e = cudaFuncSetAttribute(fk_blur_generic<uint8_t>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        fk_blur_generic<uint8_t><<<(unsigned)blocks, 256, smem, s>>>(
            pd, (const uint8_t *)in, (uint8_t *)out, n_frames, channels, w_floats, (int)interm);
    }
    *launches += 1;
    return cudaGetLastError();
}
