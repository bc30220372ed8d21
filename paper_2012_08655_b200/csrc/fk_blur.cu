/*
 * fk_blur.cu -- per-fragment separable Gaussian blur (sm_100a): dispatcher, the generic
 * kernel and the FP32 probe.
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
 *                    fallback for the work classes the fast kernel (fk_blur_fast.cu)
 *                    does not take.
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

__device__ __forceinline__ int fk_clamp(int v, int lo, int hi)
{
    return v < lo ? lo : (v > hi ? hi : v);
}

/*
 * Persistent CTAs walk one class list through its atomic cursor.  Shared memory:
 * taps[w_floats] then the H-pass intermediate, interm_floats floats; rectangles whose
 * (fh + 2r) * fw * C intermediate does not fit are processed in column strips.
 */
template <typename T>
__global__ void __launch_bounds__(256)
fk_blur_generic(fk_plan_dev pd, const T *__restrict__ in, T *__restrict__ out, int klass, int C,
                int w_floats, int interm_floats)
{
    extern __shared__ float smem[];
    __shared__ int s_idx;
    float *wts = smem;
    float *interm = smem + w_floats;
    const fk_class_list list = fk_list_of(pd, klass);
    const int n_items = list.n_items;
    int *cursor = pd.counters + FK_NCLASS + klass;
    const int W = pd.width, H = pd.height;
    const int tid = threadIdx.x, nt = blockDim.x;

    for (;;) {
        __syncthreads();
        if (tid == 0) s_idx = atomicAdd(cursor, 1);
        __syncthreads();
        const int idx = s_idx;
        if (idx >= n_items) break;
        const uint4 q = __ldg(reinterpret_cast<const uint4 *>(list.at(idx)));
        const int fw = (int)(q.z & 0xffu), fh_all = (int)(q.z >> 21);
        if (fw == 0 || fh_all == 0) continue;
        const int f = (int)q.x;
        const int x0 = (int)(q.y & 0xffffu), y0_all = (int)(q.y >> 16);
        const int x1 = x0 + fw;
        const int L = (int)((q.z >> 8) & 0x1fffu);
        const size_t frame_off = (size_t)f * H * W * C;
        const T *src = in + frame_off;
        T *dst = out + frame_off;

        if (L == 1) { /* blockwise.py:141-143: identity fragments are copied through */
            const int rowlen = fw * C;
            for (int i = tid; i < fh_all * rowlen; i += nt) {
                const int y = i / rowlen, c = i - y * rowlen;
                const size_t o = ((size_t)(y0_all + y) * W + x0) * C + c;
                dst[o] = src[o];
            }
            continue;
        }
        const int r = (L - 1) >> 1;
        const float *taps = pd.taps + q.w;
        for (int i = tid; i < L; i += nt) wts[i] = taps[i];

        __syncthreads();
        /* a strip is rendered FK_RECT rows at a time (the intermediate is sized for that) */
        for (int y0 = y0_all; y0 < y0_all + fh_all; y0 += FK_RECT) {
        const int fh = y0_all + fh_all - y0 < FK_RECT ? y0_all + fh_all - y0 : FK_RECT;
        const int th = fh + 2 * r;
        int ws = interm_floats / (th * C);
        ws = ws > fw ? fw : ws;
        if (ws < 1) break; /* host sizes the buffer so that this cannot happen */

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
    }
}

/* blockwise.py:141-143: identity fragments (the copy list) are copied through. */
template <typename T>
__global__ void __launch_bounds__(256)
fk_copy_items(fk_plan_dev pd, const T *__restrict__ in, T *__restrict__ out, int C)
{
    const fk_class_list list = fk_list_of(pd, FK_CLASS_COPY);
    const int n_items = list.n_items;
    const int W = pd.width, H = pd.height;
    for (int idx = blockIdx.x; idx < n_items; idx += gridDim.x) {
        const uint4 q = __ldg(reinterpret_cast<const uint4 *>(list.at(idx)));
        const int fw = (int)(q.z & 0xffu), fh = (int)(q.z >> 21);
        const int x0 = (int)(q.y & 0xffffu), y0 = (int)(q.y >> 16);
        const size_t frame_off = (size_t)q.x * H * W * C;
        const int rowlen = fw * C;
        for (int i = threadIdx.x; i < fh * rowlen; i += blockDim.x) {
            const int y = i / rowlen, c = i - y * rowlen;
            const size_t o = frame_off + ((size_t)(y0 + y) * W + x0) * C + c;
            out[o] = in[o];
        }
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

template <typename T>
cudaError_t launch_generic(fk_handle *h, const fk_plan_dev &pd, int klass, const void *in,
                           void *out, int channels, int class_length, cudaStream_t s)
{
    const int r = (class_length - 1) / 2;
    const int w_floats = (class_length + 3) & ~3;
    const size_t max_smem = h->prop.sharedMemPerBlockOptin;
    /* whole rectangle if it fits in ~96 KB (2 CTAs/SM), else strips down to one column */
    const long long want = (long long)(FK_RECT + 2 * r) * FK_RECT * channels;
    long long cap_floats = (96 * 1024) / 4 - w_floats;
    const long long min_floats = (long long)(FK_RECT + 2 * r) * channels;
    if (cap_floats < min_floats) cap_floats = min_floats;
    const long long interm = want < cap_floats ? want : cap_floats;
    const size_t smem = (size_t)(w_floats + interm) * sizeof(float);
    if (smem > max_smem) return cudaErrorInvalidConfiguration;
    auto kernel = fk_blur_generic<T>;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, 256, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    kernel<<<h->prop.multiProcessorCount * occ, 256, smem, s>>>(
        pd, (const T *)in, (T *)out, klass, channels, w_floats, (int)interm);
    return cudaGetLastError();
}

} // namespace

cudaError_t fk_launch_fp32_probe(float *buf, int sm_count, int iters, cudaStream_t s)
{
    fk_fp32_probe<<<sm_count * 8, 256, 0, s>>>(buf, iters);
    return cudaGetLastError();
}

/*
 * Render every class list of a plan.  Classes whose shortest possible filter exceeds the
 * plan's bound are empty by construction and are not launched; longest filters first.
 * h->variant: see fk_set_kernel_variant (include/fovea.h).
 */
cudaError_t fk_launch_blur(fk_handle *h, const fk_plan_dev &pd, const void *in, void *out,
                           int n_frames, int channels, int is_f32, int bound_length,
                           cudaStream_t s0, int *launches)
{
    /* rewind the render cursors (the counts stay) */
    cudaError_t e = cudaMemsetAsync(pd.counters + FK_NCLASS, 0, FK_NCLASS * sizeof(int32_t), s0);
    if (e != cudaSuccess) return e;
    /* The class lists cover disjoint pixels and share nothing but read-only data, so every
     * launch after the first goes to a side stream forked from s0 here and joined back below:
     * the persistent CTAs of a class start on whatever SMs the previous class's last items
     * leave idle instead of waiting for its tail. */
    const bool fork = !h->serial_classes;
    int nside = 0;
    bool first = true;
    /* the fork point precedes the first launch on s0, or the side streams would wait for it */
    if (fork) {
        e = cudaEventRecord(h->ev_fork, s0);
        if (e != cudaSuccess) return e;
    }
    for (int k = FK_CLASS_GENERIC; k >= 0; k--) {
        if (fk_class_lmin(k) > bound_length) continue;
        const int class_length = fk_class_lmax(k) < bound_length ? fk_class_lmax(k) : bound_length;
        cudaStream_t s = s0;
        if (fork && !first) {
            s = h->side[nside++];
            e = cudaStreamWaitEvent(s, h->ev_fork, 0);
            if (e != cudaSuccess) return e;
        }
        first = false;
        bool taken = false;
        if (h->variant != 1 && k < FK_CLASS_GENERIC) {
            /* RGB: column-partitioned kernel; gray (and variant 3): row-partitioned kernel */
            if (channels == 3 && h->variant != 3) {
                e = fk_launch_blur_cols(h, pd, k, in, out, n_frames, is_f32, class_length, s,
                                        &taken);
                if (e != cudaSuccess) return e;
            }
            if (!taken) {
                e = fk_launch_blur_fast(h, pd, k, in, out, n_frames, channels, is_f32,
                                        class_length, s, &taken);
                if (e != cudaSuccess) return e;
            }
        }
        if (!taken) {
            e = is_f32 ? launch_generic<float>(h, pd, k, in, out, channels, class_length, s)
                       : launch_generic<uint8_t>(h, pd, k, in, out, channels, class_length, s);
            if (e != cudaSuccess) return e;
        }
        *launches += 1;
    }
    /* identity fragments */
    const int grid = h->prop.multiProcessorCount * 4;
    if (is_f32)
        fk_copy_items<float><<<grid, 256, 0, s0>>>(pd, (const float *)in, (float *)out, channels);
    else
        fk_copy_items<uint8_t><<<grid, 256, 0, s0>>>(pd, (const uint8_t *)in, (uint8_t *)out, channels);
    *launches += 1;
    e = cudaGetLastError();
    for (int i = 0; i < nside && e == cudaSuccess; i++) { /* join */
        e = cudaEventRecord(h->ev_done[i], h->side[i]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s0, h->ev_done[i], 0);
    }
    return e;
}
