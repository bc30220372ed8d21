/*
 * fk_ssim.cu -- single-scale SSIM map on the device (sm_100a), the validation tool of the
 * render path.
 *
 * Restates quality.py:31-103 of the reference: BT.601 luma of both images (quality.py:31-35),
 * five separable windowed means over fully-valid windows -- mu_x, mu_y, E[xx], E[yy], E[xy]
 * (quality.py:45-48, 92-96) -- and the SSIM formula (quality.py:97-102), all in fp64 like the
 * reference.  The window (quality.py:38-42) is evaluated by the caller with the reference's
 * own expression and passed in, so its bits are the reference's.
 *
 *   fk_ssim_map_kernel    one CTA per 32 x 8 tile of the map: luma of the (32 + n - 1) x
 *                         (8 + n - 1) input patch of both images into shared memory, horizontal
 *                         pass of the five quantities, vertical pass, formula, store
 *                         (optionally accumulated onto the map: mean_ssim_map, quality.py:106-114).
 *   fk_ssim_stats_kernel  mean, minimum and the first flat index of the minimum (np.argmin),
 *                         one CTA, fixed reduction order (deterministic).
 *
 * HBM-bound in principle (2 x W x H x C bytes in, 8 x W x H bytes out) and tiny in practice
 * (1080p: 12 MB in, 16 MB out); fp64 throughout because it is a checker, not a hot path.
 */
#include "fk_internal.h"

namespace {

constexpr int kSX = 32, kSY = 8;   /* map tile */
constexpr int kSMaxWin = 15;       /* longest window the shared layout holds */
constexpr int kSThreads = 256;

struct ssim_args {
    const uint8_t *ref, *test;
    double *values;
    int W, H, C, n, mw, mh, accumulate;
    double c1, c2;
    double win[kSMaxWin];
};

__device__ __forceinline__ double ssim_luma(const uint8_t *p, int C)
{
    /* quality.py:31-35: data.astype(float64) @ [0.299, 0.587, 0.114]; gray: the value itself */
    if (C == 1) return (double)p[0];
    double v = __dmul_rn((double)p[0], 0.299);
    v = __dadd_rn(v, __dmul_rn((double)p[1], 0.587));
    return __dadd_rn(v, __dmul_rn((double)p[2], 0.114));
}

__global__ void __launch_bounds__(kSThreads) fk_ssim_map_kernel(const ssim_args a)
{
    constexpr int PW = kSX + kSMaxWin - 1, PH = kSY + kSMaxWin - 1;
    __shared__ double lx[PH][PW + 1], ly[PH][PW + 1];
    __shared__ double hz[5][PH][kSX + 1];
    const int n = a.n;
    const int x0 = blockIdx.x * kSX, y0 = blockIdx.y * kSY;
    const int pw = min(kSX, a.mw - x0) + n - 1, ph = min(kSY, a.mh - y0) + n - 1;
    const int tw = pw - (n - 1), th = ph - (n - 1);
    for (int i = threadIdx.x; i < pw * ph; i += kSThreads) {
        const int py = i / pw, px = i - py * pw;
        const size_t o = ((size_t)(y0 + py) * a.W + (x0 + px)) * a.C;
        lx[py][px] = ssim_luma(a.ref + o, a.C);
        ly[py][px] = ssim_luma(a.test + o, a.C);
    }
    __syncthreads();
    /* horizontal windowed sums of x, y, xx, yy, xy over every patch row (quality.py:47) */
    for (int i = threadIdx.x; i < tw * ph; i += kSThreads) {
        const int py = i / tw, px = i - py * tw;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
        for (int k = 0; k < n; k++) {
            const double g = a.win[k], x = lx[py][px + k], y = ly[py][px + k];
            s0 = __dadd_rn(s0, __dmul_rn(x, g));
            s1 = __dadd_rn(s1, __dmul_rn(y, g));
            s2 = __dadd_rn(s2, __dmul_rn(__dmul_rn(x, x), g));
            s3 = __dadd_rn(s3, __dmul_rn(__dmul_rn(y, y), g));
            s4 = __dadd_rn(s4, __dmul_rn(__dmul_rn(x, y), g));
        }
        hz[0][py][px] = s0;
        hz[1][py][px] = s1;
        hz[2][py][px] = s2;
        hz[3][py][px] = s3;
        hz[4][py][px] = s4;
    }
    __syncthreads();
    /* vertical pass (quality.py:48) and the formula (quality.py:92-102) */
    for (int i = threadIdx.x; i < tw * th; i += kSThreads) {
        const int ty = i / tw, tx = i - ty * tw;
        double m[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int k = 0; k < n; k++) {
            const double g = a.win[k];
#pragma unroll
            for (int q = 0; q < 5; q++) m[q] = __dadd_rn(m[q], __dmul_rn(hz[q][ty + k][tx], g));
        }
        const double mu_x = m[0], mu_y = m[1];
        const double var_x = __dsub_rn(m[2], __dmul_rn(mu_x, mu_x));
        const double var_y = __dsub_rn(m[3], __dmul_rn(mu_y, mu_y));
        const double cov = __dsub_rn(m[4], __dmul_rn(mu_x, mu_y));
        const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mu_x), mu_y), a.c1),
                                     __dadd_rn(__dmul_rn(2.0, cov), a.c2));
        const double den = __dmul_rn(
            __dadd_rn(__dadd_rn(__dmul_rn(mu_x, mu_x), __dmul_rn(mu_y, mu_y)), a.c1),
            __dadd_rn(__dadd_rn(var_x, var_y), a.c2));
        const double v = __ddiv_rn(num, den);
        double *dst = a.values + (size_t)(y0 + ty) * a.mw + (x0 + tx);
        *dst = a.accumulate ? __dadd_rn(*dst, v) : v;
    }
}

/* values /= divisor (when divisor != 1), then mean / min / first argmin.  stats: [mean, min,
 * argmin as a flat index]. */
__global__ void __launch_bounds__(1024)
fk_ssim_stats_kernel(double *__restrict__ values, long long count, double divisor,
                     double *__restrict__ stats)
{
    __shared__ double ssum[1024], smin[1024];
    __shared__ long long sidx[1024];
    const int t = threadIdx.x;
    double sum = 0.0, mn = 0.0;
    long long mi = -1;
    for (long long i = t; i < count; i += 1024) {
        double v = values[i];
        if (divisor != 1.0) {
            v = __ddiv_rn(v, divisor);
            values[i] = v;
        }
        sum += v;
        if (mi < 0 || v < mn) {
            mn = v;
            mi = i;
        }
    }
    ssum[t] = sum;
    smin[t] = mn;
    sidx[t] = mi;
    __syncthreads();
    for (int s = 512; s > 0; s >>= 1) {
        if (t < s) {
            ssum[t] += ssum[t + s];
            const long long oi = sidx[t + s];
            if (oi >= 0 && (sidx[t] < 0 || smin[t + s] < smin[t] ||
                            (smin[t + s] == smin[t] && oi < sidx[t]))) {
                smin[t] = smin[t + s];
                sidx[t] = oi;
            }
        }
        __syncthreads();
    }
    if (t == 0) {
        stats[0] = ssum[0] / (double)count;
        stats[1] = smin[0];
        stats[2] = (double)sidx[0];
    }
}

} // namespace

cudaError_t fk_launch_ssim_map(const uint8_t *ref, const uint8_t *test, int W, int H, int C,
                               const double *window, int n, double c1, double c2,
                               double *values, int accumulate, cudaStream_t s)
{
    if (n < 1 || n > kSMaxWin) return cudaErrorInvalidValue;
    ssim_args a;
    a.ref = ref;
    a.test = test;
    a.values = values;
    a.W = W;
    a.H = H;
    a.C = C;
    a.n = n;
    a.mw = W - n + 1;
    a.mh = H - n + 1;
    a.accumulate = accumulate;
    a.c1 = c1;
    a.c2 = c2;
    for (int i = 0; i < kSMaxWin; i++) a.win[i] = i < n ? window[i] : 0.0;
    dim3 grid((a.mw + kSX - 1) / kSX, (a.mh + kSY - 1) / kSY);
    fk_ssim_map_kernel<<<grid, kSThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t fk_launch_ssim_stats(double *values, long long count, double divisor, double *stats_dev,
                                 cudaStream_t s)
{
    fk_ssim_stats_kernel<<<1, 1024, 0, s>>>(values, count, divisor, stats_dev);
    return cudaGetLastError();
}
