/*
 * fk_api.cu -- the C ABI of libfovea.so (include/fovea.h): handles, plans, LUT
 * management, render dispatch and the host-buffer pipeline.  No torch types; the
 * Python shim passes raw pointers (tensor.data_ptr(), numpy ctypes pointers).
 */
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "fk_internal.h"

static thread_local std::string g_err;

int fk_fail(fk_handle *h, int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    if (h) h->err = buf;
    return code;
}

int fk_cuda_fail(fk_handle *h, cudaError_t e, const char *what)
{
    int code = (e == cudaErrorMemoryAllocation) ? FK_ENOMEM : FK_ECUDA;
    return fk_fail(h, code, "CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
}

static inline cudaStream_t as_stream(void *s) { return (cudaStream_t)s; }

int fk_strip_rows_for(int n_frames, int width, int height)
{
    static const int forced = [] {
        const char *e = getenv("FK_STRIP_ROWS_FORCE");
        return e ? atoi(e) : 0;
    }();
    if (forced > 0) return forced < FK_STRIP_ROWS ? forced : FK_STRIP_ROWS;
    /* By the 32 x 32 pixel units of the batch (what the persistent CTAs have to share; 2 040 per
     * 1080p frame), measured with the tall strips drawn first: one 1080p frame streams fastest
     * with 64-row strips, 8-16 frames with 256 (0.54 of the roofline against 0.51 with 1 024 at
     * 8 frames), 32 with 512, 64 and more with the tallest. */
    const long long cells = (long long)n_frames * ((width + FK_RECT - 1) / FK_RECT) *
                            ((height + FK_RECT - 1) / FK_RECT);
    return cells >= 131072 ? FK_STRIP_ROWS : cells >= 65536 ? 512 : cells >= 8192 ? 256
         : cells >= 4096 ? 128 : 64;
}

/* Host evaluation of the sigma chain (retinal.py:112-155) at distance d, used only to
 * bound the tap count before launching; the authoritative values come from the device. */
static double fk_sigma_at_distance(const fk_params *p, double d)
{
    double e = d / p->d_corner * p->e_corner;
    double fdeg = p->e2 / (p->alpha * (e + p->e2)) * p->log_inv_ct0;
    double fpix = 0.5 * fdeg / p->fmax;
    return p->strength / (p->two_pi * fpix);
}

static int fk_length_of_sigma(double sigma)
{
    if (!(sigma >= 0.0) || !std::isfinite(sigma)) return -1;
    double n6 = std::ceil(6.0 * sigma);
    if (n6 > 1.0e7) return -1;
    int n = n6 < 1.0 ? 1 : (int)n6;
    return (n & 1) ? n : n + 1;
}

extern "C" {

int fk_abi_version(void) { return FK_ABI_VERSION; }

int fk_device_count(int *count)
{
    if (!count) return fk_fail(nullptr, FK_EINVAL, "count is NULL");
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return fk_cuda_fail(nullptr, e, "cudaGetDeviceCount");
    }
    return FK_OK;
}

const char *fk_last_error(const fk_handle *h) { return h ? h->err.c_str() : g_err.c_str(); }

int fk_create(int device, fk_handle **out)
{
    if (!out) return fk_fail(nullptr, FK_EINVAL, "out is NULL");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fk_fail(nullptr, FK_ECUDA,
                       "no CUDA device available (%s); libfovea has no CPU fallback",
                       e != cudaSuccess ? cudaGetErrorString(e) : "device count is 0");
    if (device < 0 || device >= n)
        return fk_fail(nullptr, FK_EINVAL, "device %d outside [0, %d)", device, n);
    fk_handle *h = new (std::nothrow) fk_handle();
    if (!h) return fk_fail(nullptr, FK_ENOMEM, "out of host memory");
    h->device = device;
    FK_CUDA(h, cudaSetDevice(device));
    e = cudaGetDeviceProperties(&h->prop, device);
    if (e != cudaSuccess) {
        int rc = fk_cuda_fail(nullptr, e, "cudaGetDeviceProperties");
        delete h;
        return rc;
    }
    if (h->prop.major < 10) {
        int rc = fk_fail(nullptr, FK_ECUDA, "device %d is sm_%d%d; libfovea is built for sm_100a only",
                         device, h->prop.major, h->prop.minor);
        delete h;
        return rc;
    }
    for (int i = 0; i < fk_handle::kStreams; i++) {
        e = cudaStreamCreateWithFlags(&h->streams[i], cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            int rc = fk_cuda_fail(nullptr, e, "cudaStreamCreate");
            fk_destroy(h);
            return rc;
        }
    }
    for (int i = 0; i < fk_handle::kSide && e == cudaSuccess; i++) {
        e = cudaStreamCreateWithFlags(&h->side[i], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_done[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        int rc = fk_cuda_fail(nullptr, e, "side streams");
        fk_destroy(h);
        return rc;
    }
    int rc = fk_build_lut(h, FK_LUT_DEFAULT_MAX, nullptr);
    if (rc != FK_OK) {
        g_err = h->err;
        fk_destroy(h);
        return rc;
    }
    cudaStreamSynchronize(nullptr);
    *out = h;
    return FK_OK;
}

static void fk_release_stage(fk_handle *h)
{
    for (int i = 0; i < fk_handle::kStreams; i++) {
        if (h->stage_in[i]) cudaFree(h->stage_in[i]);
        if (h->stage_out[i]) cudaFree(h->stage_out[i]);
        if (h->stage_plan[i]) fk_plan_destroy(h->stage_plan[i]);
        h->stage_in[i] = h->stage_out[i] = nullptr;
        h->stage_plan[i] = nullptr;
    }
    h->stage_bytes = 0;
    h->stage_frames = 0;
}

int fk_destroy(fk_handle *h)
{
    if (!h) return FK_OK;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    fk_release_stage(h);
    for (int i = 0; i < fk_handle::kStreams; i++)
        if (h->streams[i]) cudaStreamDestroy(h->streams[i]);
    for (int i = 0; i < fk_handle::kSide; i++) {
        if (h->side[i]) cudaStreamDestroy(h->side[i]);
        if (h->ev_done[i]) cudaEventDestroy(h->ev_done[i]);
    }
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->lut64) cudaFree(h->lut64);
    if (h->lut32) cudaFree(h->lut32);
    if (h->probe) cudaFree(h->probe);
    if (h->ssim_stats) cudaFree(h->ssim_stats);
    delete h;
    return FK_OK;
}

int fk_get_device_info(fk_handle *h, fk_device_info *out)
{
    if (!h || !out) return fk_fail(h, FK_EINVAL, "NULL argument");
    memset(out, 0, sizeof *out);
    out->device = h->device;
    out->sm_count = h->prop.multiProcessorCount;
    out->cc_major = h->prop.major;
    out->cc_minor = h->prop.minor;
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, h->device);
    out->clock_khz = khz;
    out->l2_bytes = h->prop.l2CacheSize;
    out->global_mem_bytes = (int64_t)h->prop.totalGlobalMem;
    out->max_smem_optin = (int32_t)h->prop.sharedMemPerBlockOptin;
    snprintf(out->name, sizeof out->name, "%.63s", h->prop.name);
    return FK_OK;
}

/* ------------------------------------------------------------------------- LUT */
int fk_build_lut(fk_handle *h, int max_length, void *stream)
{
    if (!h) return fk_fail(nullptr, FK_EINVAL, "handle is NULL");
    if (max_length < 1 || max_length > 8191)
        return fk_fail(h, FK_EINVAL, "LUT max_length %d outside [1, 8191]", max_length);
    if ((max_length & 1) == 0) max_length += 1;
    if (max_length <= h->lut_max) return FK_OK;
    FK_CUDA(h, cudaSetDevice(h->device));
    /* Growing replaces the table: make sure nothing in flight still reads the old one. */
    if (h->lut32) FK_CUDA(h, cudaDeviceSynchronize());
    const size_t rr = (size_t)(max_length - 1) / 2 + 1;
    const size_t n = rr * rr;
    double *l64 = nullptr;
    float *l32 = nullptr;
    FK_CUDA(h, cudaMalloc(&l64, n * sizeof(double)));
    cudaError_t e = cudaMalloc(&l32, n * sizeof(float));
    if (e != cudaSuccess) {
        cudaFree(l64);
        return fk_cuda_fail(h, e, "cudaMalloc(lut32)");
    }
    e = fk_launch_build_lut(l64, l32, max_length, as_stream(stream));
    h->launches++;
    if (e == cudaSuccess) e = cudaStreamSynchronize(as_stream(stream));
    if (e != cudaSuccess) {
        cudaFree(l64);
        cudaFree(l32);
        return fk_cuda_fail(h, e, "fk_lut_kernel");
    }
    if (h->lut64) cudaFree(h->lut64);
    if (h->lut32) cudaFree(h->lut32);
    h->lut64 = l64;
    h->lut32 = l32;
    h->lut_max = max_length;
    return FK_OK;
}

int fk_lut_max_length(fk_handle *h, int *max_length)
{
    if (!h || !max_length) return fk_fail(h, FK_EINVAL, "NULL argument");
    *max_length = h->lut_max;
    return FK_OK;
}

int fk_lut_read(fk_handle *h, int length, double *taps_host)
{
    if (!h || !taps_host) return fk_fail(h, FK_EINVAL, "NULL argument");
    if (length < 1 || (length & 1) == 0)
        return fk_fail(h, FK_EINVAL, "tap count must be odd and >= 1, got %d", length);
    int rc = fk_build_lut(h, length, nullptr);
    if (rc != FK_OK) return rc;
    const size_t r = (size_t)(length - 1) / 2;
    FK_CUDA(h, cudaSetDevice(h->device));
    FK_CUDA(h, cudaMemcpy(taps_host, h->lut64 + r * r, (size_t)length * sizeof(double),
                          cudaMemcpyDeviceToHost));
    return FK_OK;
}

/* ------------------------------------------------------------------------ plans */
int fk_plan_create(fk_handle *h, int width, int height, int fragment_size, int max_frames,
                   fk_plan **out)
{
    if (!h || !out) return fk_fail(h, FK_EINVAL, "NULL argument");
    *out = nullptr;
    if (width < 1 || height < 1)
        return fk_fail(h, FK_EINVAL, "image dimensions must be positive, got %dx%d", width, height);
    if (fragment_size < 4)
        return fk_fail(h, FK_EINVAL, "fragment_size must be >= 4, got %d", fragment_size);
    if (max_frames < 1) return fk_fail(h, FK_EINVAL, "max_frames must be >= 1");
    if (width > 65535 || height > 65535)
        return fk_fail(h, FK_EINVAL, "images larger than 65535 pixels per side are not supported");
    FK_CUDA(h, cudaSetDevice(h->device));
    fk_plan *p = new (std::nothrow) fk_plan();
    if (!p) return fk_fail(h, FK_ENOMEM, "out of host memory");
    p->h = h;
    p->max_frames = max_frames;
    const int gwm = (width + fragment_size - 1) / fragment_size + 1;
    const int ghm = (height + fragment_size - 1) / fragment_size + 1;
    fk_plan_dev &d = p->d;
    d.width = width;
    d.height = height;
    d.fragment = fragment_size;
    d.cap = gwm * ghm;
    d.nsub_x = (fragment_size + FK_RECT - 1) / FK_RECT;
    d.nsub_y = (fragment_size + FK_STRIP_ROWS - 1) / FK_STRIP_ROWS;
    d.items_cap = (size_t)max_frames * d.cap * d.nsub_x * d.nsub_y;
    if ((double)d.items_cap > 2.0e9) {
        delete p;
        return fk_fail(h, FK_EINVAL, "batch too large: %d frames x %d fragments", max_frames, d.cap);
    }
    const size_t cells = (size_t)max_frames * d.cap;
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaMalloc(&d.sigma, cells * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&d.raw_length, cells * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&d.length, cells * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&d.offset, cells * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&d.strip, cells * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&d.items, FK_NCLASS * d.items_cap * sizeof(fk_item));
    if (e == cudaSuccess) e = cudaMalloc(&d.counters, FK_COUNTER_WORDS * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&d.meta, (size_t)max_frames * FK_META_WORDS * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&p->fix_dev, (size_t)max_frames * 2 * sizeof(double));
    if (e != cudaSuccess) {
        fk_plan_destroy(p);
        return fk_cuda_fail(h, e, "cudaMalloc(plan)");
    }
    d.taps = h->lut32;
    d.y_lo = 0;
    d.y_hi = 0x7fffffff;
    *out = p;
    return FK_OK;
}

int fk_plan_destroy(fk_plan *p)
{
    if (!p) return FK_OK;
    if (p->h) cudaSetDevice(p->h->device);
    cudaFree(p->d.sigma);
    cudaFree(p->d.raw_length);
    cudaFree(p->d.length);
    cudaFree(p->d.offset);
    cudaFree(p->d.strip);
    cudaFree(p->d.items);
    cudaFree(p->d.counters);
    cudaFree(p->d.meta);
    cudaFree(p->fix_dev);
    cudaFree(p->custom_taps);
    cudaFree(p->density_map);
    delete p;
    return FK_OK;
}

int fk_plan_cell_capacity(const fk_plan *p) { return p ? p->d.cap : 0; }

int fk_plan_model(fk_plan *p, const fk_params *prm, int n_frames, const double *fix_xy,
                  int fix_on_device, void *stream)
{
    if (!p || !prm || !fix_xy) return fk_fail(p ? p->h : nullptr, FK_EINVAL, "NULL argument");
    fk_handle *h = p->h;
    if (n_frames < 1 || n_frames > p->max_frames)
        return fk_fail(h, FK_EINVAL, "n_frames %d outside [1, %d]", n_frames, p->max_frames);
    if (prm->fragment_size != p->d.fragment)
        return fk_fail(h, FK_EINVAL, "params.fragment_size %d differs from the plan's %d",
                       prm->fragment_size, p->d.fragment);
    /* FoveationParams.__post_init__ (retinal.py:46-61) re-checked at the ABI */
    if (!(prm->alpha > 0) || !(prm->e2 > 0) || !(prm->ct0 > 0 && prm->ct0 < 1) ||
        !(prm->e_corner >= 0) || !(prm->strength >= 0) || !(prm->fmax > 0) ||
        !(prm->d_corner > 0) || !std::isfinite(prm->log_inv_ct0) || !(prm->two_pi > 0))
        return fk_fail(h, FK_EINVAL, "invalid foveation parameters");
    if (prm->use_shift == 2 && (prm->shift_x < 0 || prm->shift_x >= prm->fragment_size ||
                                prm->shift_y < 0 || prm->shift_y >= prm->fragment_size))
        return fk_fail(h, FK_EINVAL, "offset (%d, %d) outside [0, %d)", prm->shift_x,
                       prm->shift_y, prm->fragment_size);
    const int W = p->d.width, H = p->d.height;
    /* Upper bound of the tap count: sigma grows with distance, and no fragment midpoint
     * is farther from a fixation than the farthest image corner. */
    double dmax = 0.0;
    if (fix_on_device) {
        dmax = std::hypot((double)W, (double)H);
    } else {
        for (int i = 0; i < n_frames; i++) {
            double fx = fix_xy[2 * i], fy = fix_xy[2 * i + 1];
            if (!(fx >= 0 && fx < W && fy >= 0 && fy < H))
                return fk_fail(h, FK_EINVAL, "fixation (%g, %g) outside %dx%d image", fx, fy, W, H);
            double ddx = fx > W - fx ? fx : W - fx, ddy = fy > H - fy ? fy : H - fy;
            double d = std::hypot(ddx, ddy);
            dmax = d > dmax ? d : dmax;
        }
    }
    int bound = fk_length_of_sigma(fk_sigma_at_distance(prm, dmax));
    if (bound < 0 || bound + 2 > 8191)
        return fk_fail(h, FK_EINVAL, "sigma values must be finite and >= 0 and need <= 8191 taps");
    bound += 2; /* the device value is authoritative; leave one odd step of slack */
    FK_CUDA(h, cudaSetDevice(h->device));
    if (bound > h->lut_max) {
        int rc = fk_build_lut(h, bound, stream);
        if (rc != FK_OK) return rc;
    }
    cudaStream_t s = as_stream(stream);
    const double *fix_dev = fix_xy;
    if (!fix_on_device) {
        FK_CUDA(h, cudaMemcpyAsync(p->fix_dev, fix_xy, (size_t)n_frames * 2 * sizeof(double),
                                   cudaMemcpyHostToDevice, s));
        fix_dev = p->fix_dev;
    }
    p->d.taps = h->lut32;
    p->custom = 0;
    /* a request's plan (fk_request_create) zeroes its counters in the plan kernel and reports
     * to pinned host memory: no memset and no copy nodes in the captured graph */
    p->d.canonical = 1;
    p->d.self_zero = p->request_info != nullptr && n_frames == 1;
    p->d.info_out = n_frames == 1 ? p->request_info : nullptr;
    if (!p->d.self_zero)
        FK_CUDA(h, cudaMemsetAsync(p->d.counters, 0, FK_COUNTER_WORDS * sizeof(int32_t), s));
    const fk_density_dev no_density = {nullptr, 0, 0, 0.0};
    p->d.strip_rows = fk_strip_rows_for(n_frames, p->d.width, p->d.height);
    p->d.mixed = h->no_mixed ? 0 : 1;
    FK_CUDA(h, fk_launch_plan(p->d, *prm, n_frames, fix_dev, no_density, s));
    h->launches++;
    p->n_frames = n_frames;
    p->bound_length = bound;
    return FK_OK;
}

int fk_plan_density(fk_plan *p, const fk_params *prm, int n_frames, const double *fix_xy,
                    int fix_on_device, const uint8_t *map_host, int map_w, int map_h,
                    double sigma_max, void *stream)
{
    if (!p || !prm || !fix_xy || !map_host)
        return fk_fail(p ? p->h : nullptr, FK_EINVAL, "NULL argument");
    fk_handle *h = p->h;
    if (n_frames < 1 || n_frames > p->max_frames)
        return fk_fail(h, FK_EINVAL, "n_frames %d outside [1, %d]", n_frames, p->max_frames);
    if (prm->fragment_size != p->d.fragment)
        return fk_fail(h, FK_EINVAL, "params.fragment_size %d differs from the plan's %d",
                       prm->fragment_size, p->d.fragment);
    if (prm->use_shift == 2 && (prm->shift_x < 0 || prm->shift_x >= prm->fragment_size ||
                                prm->shift_y < 0 || prm->shift_y >= prm->fragment_size))
        return fk_fail(h, FK_EINVAL, "offset (%d, %d) outside [0, %d)", prm->shift_x,
                       prm->shift_y, prm->fragment_size);
    if (map_w < 1 || map_h < 1)
        return fk_fail(h, FK_EINVAL, "image dimensions must be positive, got %dx%d", map_w, map_h);
    if (!(sigma_max >= 0) || !std::isfinite(sigma_max)) /* retinal.py:221-222 */
        return fk_fail(h, FK_EINVAL, "sigma_max must be >= 0, got %g", sigma_max);
    const int W = p->d.width, H = p->d.height;
    if (!fix_on_device)
        for (int i = 0; i < n_frames; i++) {
            double fx = fix_xy[2 * i], fy = fix_xy[2 * i + 1];
            if (!(fx >= 0 && fx < W && fy >= 0 && fy < H))
                return fk_fail(h, FK_EINVAL, "fixation (%g, %g) outside %dx%d image", fx, fy, W, H);
        }
    int bound = fk_length_of_sigma(sigma_max); /* sigma = sigma_max * (1 - v/255) <= sigma_max */
    if (bound < 0 || bound + 2 > 8191)
        return fk_fail(h, FK_EINVAL, "sigma values must be finite and >= 0 and need <= 8191 taps");
    bound += 2;
    FK_CUDA(h, cudaSetDevice(h->device));
    if (bound > h->lut_max) {
        int rc = fk_build_lut(h, bound, stream);
        if (rc != FK_OK) return rc;
    }
    cudaStream_t s = as_stream(stream);
    const size_t map_bytes = (size_t)map_w * map_h;
    if (map_bytes > p->density_cap) {
        FK_CUDA(h, cudaStreamSynchronize(s));
        cudaFree(p->density_map);
        p->density_map = nullptr;
        p->density_cap = 0;
        FK_CUDA(h, cudaMalloc(&p->density_map, map_bytes));
        p->density_cap = map_bytes;
    }
    FK_CUDA(h, cudaMemcpyAsync(p->density_map, map_host, map_bytes, cudaMemcpyHostToDevice, s));
    const double *fix_dev = fix_xy;
    if (!fix_on_device) {
        FK_CUDA(h, cudaMemcpyAsync(p->fix_dev, fix_xy, (size_t)n_frames * 2 * sizeof(double),
                                   cudaMemcpyHostToDevice, s));
        fix_dev = p->fix_dev;
    }
    p->d.taps = h->lut32;
    p->custom = 0;
    FK_CUDA(h, cudaMemsetAsync(p->d.counters, 0, FK_COUNTER_WORDS * sizeof(int32_t), s));
    const fk_density_dev den = {p->density_map, map_w, map_h, sigma_max};
    p->d.strip_rows = fk_strip_rows_for(n_frames, p->d.width, p->d.height);
    p->d.mixed = h->no_mixed ? 0 : 1;
    p->d.canonical = 1;
    p->d.self_zero = 0;
    p->d.info_out = nullptr;
    FK_CUDA(h, fk_launch_plan(p->d, *prm, n_frames, fix_dev, den, s));
    h->launches++;
    p->n_frames = n_frames;
    p->bound_length = bound;
    return FK_OK;
}

int fk_plan_set_grid(fk_plan *p, int shift_x, int shift_y, int grid_w, int grid_h,
                     const int32_t *length, const int32_t *offset, const double *coeffs,
                     int n_coeffs, void *stream)
{
    if (!p || !length || !offset || !coeffs)
        return fk_fail(p ? p->h : nullptr, FK_EINVAL, "NULL argument");
    fk_handle *h = p->h;
    const fk_plan_dev &d = p->d;
    const int F = d.fragment;
    if (shift_x < 0 || shift_x >= F || shift_y < 0 || shift_y >= F)
        return fk_fail(h, FK_EINVAL, "shift (%d, %d) outside [0, %d)", shift_x, shift_y, F);
    const int gw = fk_span_count(d.width, F, shift_x), gh = fk_span_count(d.height, F, shift_y);
    if (gw != grid_w || gh != grid_h) /* blockwise.py:168-169 */
        return fk_fail(h, FK_EINVAL, "grid (%d, %d) does not match image %dx%d", grid_h, grid_w,
                       d.width, d.height);
    const int n = gw * gh;
    int lmax = 1;
    for (int i = 0; i < n; i++) {
        if (length[i] < 1 || (length[i] & 1) == 0)
            return fk_fail(h, FK_EINVAL, "filter lengths must be odd and >= 1, got %d", length[i]);
        if (offset[i] < 0 || offset[i] + length[i] > n_coeffs)
            return fk_fail(h, FK_EINVAL, "grid references taps outside the bank");
        lmax = length[i] > lmax ? length[i] : lmax;
    }
    if (lmax > 8191) return fk_fail(h, FK_EINVAL, "filters longer than 8191 taps are not supported");
    FK_CUDA(h, cudaSetDevice(h->device));
    cudaStream_t s = as_stream(stream);
    if (n_coeffs > p->custom_cap) {
        FK_CUDA(h, cudaStreamSynchronize(s));
        cudaFree(p->custom_taps);
        p->custom_taps = nullptr;
        FK_CUDA(h, cudaMalloc(&p->custom_taps, (size_t)n_coeffs * sizeof(float)));
        p->custom_cap = n_coeffs;
    }
    std::vector<float> taps32((size_t)n_coeffs);
    for (int i = 0; i < n_coeffs; i++) taps32[i] = (float)coeffs[i];
    int32_t meta[FK_META_WORDS] = {shift_x, shift_y, gw, gh, -1, -1, lmax, 0};
    FK_CUDA(h, cudaMemcpyAsync(p->custom_taps, taps32.data(), (size_t)n_coeffs * sizeof(float),
                               cudaMemcpyHostToDevice, s));
    FK_CUDA(h, cudaMemcpyAsync(d.length, length, (size_t)n * sizeof(int32_t),
                               cudaMemcpyHostToDevice, s));
    FK_CUDA(h, cudaMemcpyAsync(d.raw_length, length, (size_t)n * sizeof(int32_t),
                               cudaMemcpyHostToDevice, s));
    FK_CUDA(h, cudaMemcpyAsync(d.offset, offset, (size_t)n * sizeof(int32_t),
                               cudaMemcpyHostToDevice, s));
    FK_CUDA(h, cudaMemcpyAsync(d.meta, meta, sizeof meta, cudaMemcpyHostToDevice, s));
    /* the staging vectors above are pageable: the copies have been staged on return,
     * but synchronise anyway so `taps32` may die safely */
    FK_CUDA(h, cudaStreamSynchronize(s));
    p->d.taps = p->custom_taps;
    p->custom = 1;
    FK_CUDA(h, cudaMemsetAsync(p->d.counters, 0, FK_COUNTER_WORDS * sizeof(int32_t), s));
    p->d.strip_rows = fk_strip_rows_for(1, p->d.width, p->d.height);
    p->d.mixed = 0; /* a caller's bank: tap offsets are not the canonical r * r */
    p->d.canonical = 0;
    p->d.self_zero = 0;
    p->d.info_out = nullptr;
    FK_CUDA(h, fk_launch_order(p->d, 1, s));
    h->launches++;
    p->n_frames = 1;
    p->bound_length = lmax;
    return FK_OK;
}

int fk_plan_read_lengths(fk_plan *p, int first, int count, int32_t *lengths_host,
                         int32_t *meta_host, void *stream)
{
    if (!p) return fk_fail(nullptr, FK_EINVAL, "plan is NULL");
    fk_handle *h = p->h;
    if (first < 0 || count < 1 || first + count > p->n_frames)
        return fk_fail(h, FK_EINVAL, "frames [%d, %d) outside the %d planned", first,
                       first + count, p->n_frames);
    FK_CUDA(h, cudaSetDevice(h->device));
    FK_CUDA(h, cudaStreamSynchronize(as_stream(stream)));
    if (lengths_host)
        FK_CUDA(h, cudaMemcpy(lengths_host, p->d.length + (size_t)first * p->d.cap,
                              (size_t)count * p->d.cap * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (meta_host)
        FK_CUDA(h, cudaMemcpy(meta_host, p->d.meta + (size_t)first * FK_META_WORDS,
                              (size_t)count * FK_META_WORDS * sizeof(int32_t),
                              cudaMemcpyDeviceToHost));
    return FK_OK;
}

int fk_plan_read(fk_plan *p, int frame, fk_plan_view *out, void *stream)
{
    if (!p || !out) return fk_fail(p ? p->h : nullptr, FK_EINVAL, "NULL argument");
    fk_handle *h = p->h;
    if (frame < 0 || frame >= p->n_frames)
        return fk_fail(h, FK_EINVAL, "frame %d outside the %d planned", frame, p->n_frames);
    FK_CUDA(h, cudaSetDevice(h->device));
    FK_CUDA(h, cudaStreamSynchronize(as_stream(stream)));
    int32_t meta[FK_META_WORDS];
    FK_CUDA(h, cudaMemcpy(meta, p->d.meta + (size_t)frame * FK_META_WORDS, sizeof meta,
                          cudaMemcpyDeviceToHost));
    out->shift_x = meta[FK_META_SX];
    out->shift_y = meta[FK_META_SY];
    out->grid_w = meta[FK_META_GW];
    out->grid_h = meta[FK_META_GH];
    out->foveal_gy = meta[FK_META_FGY];
    out->foveal_gx = meta[FK_META_FGX];
    out->max_length = meta[FK_META_LMAX];
    out->status = meta[FK_META_STATUS];
    if (out->status != 0) return FK_OK;
    const size_t n = (size_t)out->grid_w * out->grid_h, base = (size_t)frame * p->d.cap;
    if (out->sigma && !p->custom)
        FK_CUDA(h, cudaMemcpy(out->sigma, p->d.sigma + base, n * sizeof(double),
                              cudaMemcpyDeviceToHost));
    if (out->raw_length)
        FK_CUDA(h, cudaMemcpy(out->raw_length, p->d.raw_length + base, n * sizeof(int32_t),
                              cudaMemcpyDeviceToHost));
    if (out->length)
        FK_CUDA(h, cudaMemcpy(out->length, p->d.length + base, n * sizeof(int32_t),
                              cudaMemcpyDeviceToHost));
    return FK_OK;
}

int fk_plan_item_classes(void) { return FK_NCLASS; }

int fk_plan_read_items(fk_plan *p, int klass, uint32_t *items_host, int capacity, int *count,
                       void *stream)
{
    if (!p || !count) return fk_fail(p ? p->h : nullptr, FK_EINVAL, "NULL argument");
    fk_handle *h = p->h;
    if (klass < 0 || klass >= FK_NCLASS)
        return fk_fail(h, FK_EINVAL, "class %d outside [0, %d)", klass, FK_NCLASS);
    FK_CUDA(h, cudaSetDevice(h->device));
    FK_CUDA(h, cudaStreamSynchronize(as_stream(stream)));
    /* a list has two ends (fk_class_list): tall strips at the front of its region, short ones
     * at the back; they are returned front first, in the order the render draws them */
    int32_t nf = 0, nb = 0;
    FK_CUDA(h, cudaMemcpy(&nf, p->d.counters + klass, sizeof nf, cudaMemcpyDeviceToHost));
    FK_CUDA(h, cudaMemcpy(&nb, p->d.counters + FK_COUNTER_BACK + klass, sizeof nb,
                          cudaMemcpyDeviceToHost));
    *count = nf + nb;
    if (!items_host || capacity <= 0) return FK_OK;
    const fk_item *base = p->d.items + (size_t)klass * p->d.items_cap;
    fk_item *dst = reinterpret_cast<fk_item *>(items_host);
    const int take_f = nf < capacity ? nf : capacity;
    if (take_f > 0)
        FK_CUDA(h, cudaMemcpy(dst, base, (size_t)take_f * sizeof(fk_item), cudaMemcpyDeviceToHost));
    const int take_b = nb < capacity - take_f ? nb : capacity - take_f;
    if (take_b > 0) {
        FK_CUDA(h, cudaMemcpy(dst + take_f, base + (p->d.items_cap - (size_t)take_b),
                              (size_t)take_b * sizeof(fk_item), cudaMemcpyDeviceToHost));
        for (int i = 0, j = take_b - 1; i < j; i++, j--) { /* drawn from the end downwards */
            const fk_item t = dst[take_f + i];
            dst[take_f + i] = dst[take_f + j];
            dst[take_f + j] = t;
        }
    }
    return FK_OK;
}

int fk_plan_status(fk_plan *p, int *bad_frames, void *stream)
{
    if (!p || !bad_frames) return fk_fail(p ? p->h : nullptr, FK_EINVAL, "NULL argument");
    fk_handle *h = p->h;
    *bad_frames = 0;
    if (p->n_frames < 1) return FK_OK;
    FK_CUDA(h, cudaSetDevice(h->device));
    int32_t bad = 0;
    FK_CUDA(h, cudaMemcpyAsync(&bad, p->d.counters + FK_COUNTER_BAD, sizeof bad,
                               cudaMemcpyDeviceToHost, as_stream(stream)));
    FK_CUDA(h, cudaStreamSynchronize(as_stream(stream)));
    *bad_frames = bad;
    return FK_OK;
}

/* ----------------------------------------------------------------------- render */
static int fk_render_any(fk_handle *h, const fk_plan *p, const void *in, void *out,
                         int n_frames, int channels, int is_f32, void *stream)
{
    if (!h || !p || !in || !out) return fk_fail(h, FK_EINVAL, "NULL argument");
    if (p->h != h) return fk_fail(h, FK_EINVAL, "plan belongs to another handle");
    if (channels != 1 && channels != 3) /* blockwise.py:160-161 */
        return fk_fail(h, FK_EINVAL, "render supports 1 or 3 channels, got %d", channels);
    /* the work lists cover every planned frame: rendering fewer would write past `out` */
    if (n_frames != p->n_frames)
        return fk_fail(h, FK_EINVAL, "%d frames to render but %d planned", n_frames, p->n_frames);
    if (in == out) return fk_fail(h, FK_EINVAL, "render cannot run in place");
    FK_CUDA(h, cudaSetDevice(h->device));
    int launches = 0;
    if (p->d.mixed && !(channels == 3 && (h->variant == 0 || h->variant == 5 || h->variant == 6) &&
                        fk_blur_tma_usable(in, p->d.width, p->d.height, is_f32))) {
        /* mixed items are read by fk_blur_tma only: this render falls back to another kernel,
         * so the plan's work lists are emitted once more without them (the cell arrays stay) */
        fk_plan *pm = const_cast<fk_plan *>(p);
        pm->d.mixed = 0;
        FK_CUDA(h, cudaMemsetAsync(pm->d.counters, 0, FK_COUNTER_BAD * sizeof(int32_t),
                                   as_stream(stream)));
        FK_CUDA(h, fk_launch_order(pm->d, n_frames, as_stream(stream)));
        launches++;
    }
    fk_plan_dev pd = p->d;
    if (!p->custom) pd.taps = h->lut32; /* the canonical table may have grown since planning */
    cudaError_t e = fk_launch_blur(h, pd, in, out, n_frames, channels, is_f32,
                                   p->bound_length, as_stream(stream), &launches);
    h->launches += launches;
    if (e == cudaErrorInvalidConfiguration)
        return fk_fail(h, FK_EINVAL, "filter of %d taps does not fit the device's shared memory",
                       p->bound_length);
    if (e != cudaSuccess) return fk_cuda_fail(h, e, "blur launch");
    return FK_OK;
}

int fk_render_u8(fk_handle *h, const fk_plan *p, const uint8_t *in_dev, uint8_t *out_dev,
                 int n_frames, int channels, void *stream)
{
    return fk_render_any(h, p, in_dev, out_dev, n_frames, channels, 0, stream);
}

int fk_render_f32(fk_handle *h, const fk_plan *p, const float *in_dev, float *out_dev,
                  int n_frames, int channels, void *stream)
{
    return fk_render_any(h, p, in_dev, out_dev, n_frames, channels, 1, stream);
}

int fk_set_kernel_variant(fk_handle *h, int variant)
{
    if (!h) return 0;
    int old = h->variant | (h->serial_classes ? 16 : 0) | (h->no_mixed ? 32 : 0);
    h->variant = variant & 15;
    h->serial_classes = (variant & 16) != 0;
    h->no_mixed = (variant & 32) != 0; /* plans made from now on hold no mixed items */
    return old;
}

int64_t fk_launch_count(const fk_handle *h) { return h ? h->launches : 0; }

/* ------------------------------------------------------------------- request graph */
/*
 * One gaze-contingent frame as one CUDA-graph launch: fixation (pinned host memory, read by the
 * plan kernel) -> plan -> render -> frame to pinned host memory.  The device-to-host copy of a
 * 1080p frame (6.2 MB at the ~58 GB/s of the link: 0.107 ms) is half of a request, so the frame
 * is rendered in TWO BANDS and the copy of the upper band runs under the render of the lower
 * one: two plans of the same fixation, planned side by side, whose kernels emit only the
 * rectangles that start in their band (fk_plan_dev::y_lo / y_hi) -- every pixel above the split
 * row belongs to a rectangle that starts above it, so those rows are final once the upper
 * band's launches are done.  FK_REQUEST_SPLIT (percent of the rows in the upper band; 0: one
 * band) is read at creation; small frames are not split.
 */
struct fk_request {
    fk_handle *h = nullptr;
    fk_plan *p = nullptr;
    fk_plan *p_low = nullptr;        /* plan of the lower band (owned) */
    int32_t *info_low = nullptr;     /* device scratch its plan kernel reports to */
    cudaStream_t s_plan = nullptr;   /* capture only: the lower band's plan */
    cudaStream_t s_copy = nullptr;   /* capture only: the upper band's copy */
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    double *fix_host = nullptr;   /* pinned, 2 doubles */
    int32_t *info_host = nullptr; /* pinned, 16 + cell capacity words */
};

int fk_request_destroy(fk_request *r)
{
    if (!r) return FK_OK;
    if (r->h) cudaSetDevice(r->h->device);
    if (r->exec) cudaGraphExecDestroy(r->exec);
    if (r->graph) cudaGraphDestroy(r->graph);
    if (r->s_plan) cudaStreamDestroy(r->s_plan);
    if (r->s_copy) cudaStreamDestroy(r->s_copy);
    fk_plan_destroy(r->p_low);
    cudaFree(r->info_low);
    cudaFreeHost(r->fix_host);
    cudaFreeHost(r->info_host);
    delete r;
    return FK_OK;
}

int fk_request_create(fk_handle *h, fk_plan *p, const fk_params *prm, const void *in_dev,
                      void *out_dev, void *out_host, int channels, int is_f32, void *stream,
                      fk_request **out)
{
    if (!h || !p || !prm || !in_dev || !out_dev || !out)
        return fk_fail(h, FK_EINVAL, "NULL argument");
    if (p->h != h) return fk_fail(h, FK_EINVAL, "plan belongs to another handle");
    cudaStream_t s = as_stream(stream);
    if (s == nullptr || s == cudaStreamLegacy)
        return fk_fail(h, FK_EINVAL, "a request is captured on a stream of its own, not the default stream");
    FK_CUDA(h, cudaSetDevice(h->device));
    const int W = p->d.width, H = p->d.height;
    const size_t row_bytes = (size_t)W * channels * (is_f32 ? 4 : 1);
    const size_t frame_bytes = row_bytes * H;
    fk_request *r = new fk_request();
    r->h = h;
    r->p = p;
    /* FK_REQUEST_PARTS (tuning runs): bit 0 plan, 1 render, 2 frame copy, 3 plan summary */
    const char *pe = getenv("FK_REQUEST_PARTS");
    const int parts = pe ? atoi(pe) : 15;
    /* rows of the upper band: 55 % (1080p: 0.227 ms per request with one band, 0.211 / 0.207 /
     * 0.207 / 0.213 ms with 40 / 50 / 60 / 70 %) -- the upper band's render is what no copy hides,
     * the lower band's has to fit under the upper band's copy */
    const char *se = getenv("FK_REQUEST_SPLIT");
    const int split_pct = se ? atoi(se) : 55;
    int y_split = 0;
    if (out_host && parts == 15 && split_pct > 0 && split_pct < 100 && frame_bytes >= (1u << 20))
        y_split = (int)((long long)H * split_pct / 100);
    cudaError_t e = cudaHostAlloc(&r->fix_host, 2 * sizeof(double), cudaHostAllocDefault);
    if (e == cudaSuccess)
        e = cudaHostAlloc(&r->info_host, (16 + (size_t)p->d.cap) * sizeof(int32_t), cudaHostAllocDefault);
    if (e == cudaSuccess && y_split > 0) e = cudaMalloc(&r->info_low, (16 + (size_t)p->d.cap) * sizeof(int32_t));
    if (e == cudaSuccess && y_split > 0) e = cudaStreamCreateWithFlags(&r->s_plan, cudaStreamNonBlocking);
    if (e == cudaSuccess && y_split > 0) e = cudaStreamCreateWithFlags(&r->s_copy, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        fk_request_destroy(r);
        return fk_cuda_fail(h, e, "request resources");
    }
    r->fix_host[0] = W / 2.0;
    r->fix_host[1] = H / 2.0;
    memset(r->info_host, 0, (16 + (size_t)p->d.cap) * sizeof(int32_t));
    int rc = FK_OK;
    if (y_split > 0) rc = fk_plan_create(h, W, H, p->d.fragment, 1, &r->p_low);
    fk_plan *pl = r->p_low;
    /* one plain run first: it validates the arguments, grows the tap table to the longest filter
     * a fixation on the device can need and sets every kernel attribute -- nothing of which may
     * happen inside a capture */
    if (rc == FK_OK) rc = fk_plan_model(p, prm, 1, r->fix_host, 0, stream);
    if (rc == FK_OK) rc = fk_plan_model(p, prm, 1, p->fix_dev, 1, stream);
    if (rc == FK_OK && pl) rc = fk_plan_model(pl, prm, 1, p->fix_dev, 1, stream);
    if (rc == FK_OK) rc = fk_render_any(h, p, in_dev, out_dev, 1, channels, is_f32, stream);
    if (rc == FK_OK && cudaStreamSynchronize(s) != cudaSuccess) rc = fk_fail(h, FK_ECUDA, "request warm-up failed");
    if (rc != FK_OK) {
        fk_request_destroy(r);
        return rc;
    }
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr}; /* fork, lower plan done, upper band rendered / copied */
    for (int i = 0; i < 3 && pl && e == cudaSuccess; i++) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) {
        for (cudaEvent_t v : ev)
            if (v) cudaEventDestroy(v);
        fk_request_destroy(r);
        return fk_cuda_fail(h, e, "cudaStreamBeginCapture");
    }
    if (pl) { /* the lower band's plan, side by side with the upper band's */
        e = cudaEventRecord(ev[0], s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(r->s_plan, ev[0], 0);
        if (e == cudaSuccess) {
            pl->d.y_lo = y_split;
            pl->request_info = r->info_low;
            rc = fk_plan_model(pl, prm, 1, r->fix_host, 1, r->s_plan);
            pl->request_info = nullptr;
            pl->d.y_lo = 0;
        }
        if (e == cudaSuccess && rc == FK_OK) e = cudaEventRecord(ev[1], r->s_plan);
    }
    if (e == cudaSuccess && rc == FK_OK && (parts & 1)) {
        /* pinned host memory is mapped into the device's address space (unified addressing):
         * the plan kernel reads the fixation from it and writes the plan summary to it */
        p->request_info = (parts & 8) ? r->info_host : nullptr;
        if (pl) p->d.y_hi = y_split;
        rc = fk_plan_model(p, prm, 1, r->fix_host, 1, stream);
        p->d.y_hi = 0x7fffffff;
        p->request_info = nullptr;
    }
    if (e == cudaSuccess && rc == FK_OK && (parts & 2))
        rc = fk_render_any(h, p, in_dev, out_dev, 1, channels, is_f32, stream);
    if (pl && e == cudaSuccess && rc == FK_OK) {
        /* rows [0, y_split) are final: their copy runs beside the lower band's render */
        e = cudaEventRecord(ev[2], s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(r->s_copy, ev[2], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(out_host, out_dev, row_bytes * y_split, cudaMemcpyDeviceToHost, r->s_copy);
        if (e == cudaSuccess) e = cudaEventRecord(ev[2], r->s_copy);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[1], 0);
        if (e == cudaSuccess) rc = fk_render_any(h, pl, in_dev, out_dev, 1, channels, is_f32, stream);
        if (e == cudaSuccess && rc == FK_OK)
            e = cudaMemcpyAsync((char *)out_host + row_bytes * y_split, (const char *)out_dev + row_bytes * y_split,
                                row_bytes * (H - y_split), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[2], 0);
    } else if (e == cudaSuccess && rc == FK_OK && out_host && (parts & 4)) {
        e = cudaMemcpyAsync(out_host, out_dev, frame_bytes, cudaMemcpyDeviceToHost, s);
    }
    cudaError_t e2 = cudaStreamEndCapture(s, &r->graph); /* always: leaves the stream usable */
    for (cudaEvent_t v : ev)
        if (v) cudaEventDestroy(v);
    if (rc == FK_OK && e != cudaSuccess) rc = fk_cuda_fail(h, e, "request capture");
    if (rc == FK_OK && e2 != cudaSuccess) rc = fk_cuda_fail(h, e2, "cudaStreamEndCapture");
    if (rc == FK_OK) {
        e = cudaGraphInstantiate(&r->exec, r->graph, 0);
        if (e != cudaSuccess) rc = fk_cuda_fail(h, e, "cudaGraphInstantiate");
    }
    if (rc != FK_OK) {
        fk_request_destroy(r);
        return rc;
    }
    *out = r;
    return FK_OK;
}

int fk_request_launch(fk_request *r, double fx, double fy, void *stream)
{
    if (!r) return FK_EINVAL;
    fk_handle *h = r->h;
    if (!(fx >= 0 && fx < r->p->d.width && fy >= 0 && fy < r->p->d.height))
        return fk_fail(h, FK_EINVAL, "fixation (%g, %g) outside %dx%d image", fx, fy,
                       r->p->d.width, r->p->d.height);
    FK_CUDA(h, cudaSetDevice(h->device));
    /* the previous request on this stream has been consumed by its upload node once the
     * caller synchronised; requests in flight on one stream must not overlap (the graph has
     * one set of buffers) */
    r->fix_host[0] = fx;
    r->fix_host[1] = fy;
    FK_CUDA(h, cudaGraphLaunch(r->exec, as_stream(stream)));
    h->launches += 1;
    return FK_OK;
}

const int32_t *fk_request_info(const fk_request *r) { return r ? r->info_host : nullptr; }

/* ------------------------------------------------------------ host-buffer pipeline */
static int fk_foveate_host_any(fk_handle *h, const fk_params *prm, int W, int H, int C, int N,
                               const double *fix, const void *in, void *out, int chunk,
                               int is_f32)
{
    if (!h || !prm || !fix || !in || !out) return fk_fail(h, FK_EINVAL, "NULL argument");
    if (C != 1 && C != 3) return fk_fail(h, FK_EINVAL, "render supports 1 or 3 channels, got %d", C);
    if (N < 1) return fk_fail(h, FK_EINVAL, "n_frames must be >= 1");
    if (W < 1 || H < 1) return fk_fail(h, FK_EINVAL, "image dimensions must be positive");
    const size_t esz = is_f32 ? 4 : 1;
    const size_t frame_bytes = (size_t)W * H * C * esz;
    if (chunk <= 0) {
        size_t c = ((size_t)48 << 20) / frame_bytes;
        chunk = (int)(c < 1 ? 1 : (c > 4096 ? 4096 : c));
    }
    if (chunk > N) chunk = N;
    /* keep all streams busy on small batches */
    if (N >= fk_handle::kStreams && chunk * fk_handle::kStreams > N)
        chunk = (N + fk_handle::kStreams - 1) / fk_handle::kStreams;
    FK_CUDA(h, cudaSetDevice(h->device));
    const size_t need = frame_bytes * chunk;
    const bool replan = h->stage_w != W || h->stage_h != H ||
                        h->stage_f != prm->fragment_size || h->stage_frames < chunk;
    if (need > h->stage_bytes || replan) {
        FK_CUDA(h, cudaDeviceSynchronize());
        fk_release_stage(h);
        for (int i = 0; i < fk_handle::kStreams; i++) {
            cudaError_t ce = cudaMalloc(&h->stage_in[i], need);
            if (ce == cudaSuccess) ce = cudaMalloc(&h->stage_out[i], need);
            int rc = ce == cudaSuccess ? fk_plan_create(h, W, H, prm->fragment_size, chunk,
                                                        &h->stage_plan[i])
                                       : fk_cuda_fail(h, ce, "cudaMalloc(staging)");
            if (rc != FK_OK) { /* no half-built pipeline is left behind */
                std::string msg = h->err;
                fk_release_stage(h);
                h->stage_w = h->stage_h = h->stage_f = 0;
                h->err = msg;
                return rc;
            }
        }
        h->stage_bytes = need;
        h->stage_w = W;
        h->stage_h = H;
        h->stage_f = prm->fragment_size;
        h->stage_frames = chunk;
    }
    /* every fixation is checked before anything is queued (retinal.py:73-74), so an invalid
     * one cannot leave earlier chunks' copies in flight */
    for (int i = 0; i < N; i++) {
        const double fx = fix[2 * i], fy = fix[2 * i + 1];
        if (!(fx >= 0 && fx < W && fy >= 0 && fy < H))
            return fk_fail(h, FK_EINVAL, "fixation (%g, %g) outside %dx%d image", fx, fy, W, H);
    }
    auto drain = [&](int rc) { /* an error mid-pipeline: wait for what is already queued */
        for (int i = 0; i < fk_handle::kStreams; i++) cudaStreamSynchronize(h->streams[i]);
        return rc;
    };
    int idx = 0;
    for (int first = 0; first < N; first += chunk, idx++) {
        const int n = (N - first) < chunk ? (N - first) : chunk;
        const int slot = idx % fk_handle::kStreams;
        cudaStream_t s = h->streams[slot];
        const size_t off = frame_bytes * first, bytes = frame_bytes * n;
        cudaError_t ce = cudaMemcpyAsync(h->stage_in[slot], (const char *)in + off, bytes,
                                         cudaMemcpyHostToDevice, s);
        if (ce != cudaSuccess) return drain(fk_cuda_fail(h, ce, "cudaMemcpyAsync(H2D)"));
        int rc = fk_plan_model(h->stage_plan[slot], prm, n, fix + 2 * (size_t)first, 0, s);
        if (rc != FK_OK) return drain(rc);
        rc = fk_render_any(h, h->stage_plan[slot], h->stage_in[slot], h->stage_out[slot], n, C,
                           is_f32, s);
        if (rc != FK_OK) return drain(rc);
        ce = cudaMemcpyAsync((char *)out + off, h->stage_out[slot], bytes, cudaMemcpyDeviceToHost, s);
        if (ce != cudaSuccess) return drain(fk_cuda_fail(h, ce, "cudaMemcpyAsync(D2H)"));
    }
    for (int i = 0; i < fk_handle::kStreams; i++) FK_CUDA(h, cudaStreamSynchronize(h->streams[i]));
    return FK_OK;
}

int fk_foveate_host_u8(fk_handle *h, const fk_params *params, int width, int height,
                       int channels, int n_frames, const double *fix_xy_host,
                       const uint8_t *in_host, uint8_t *out_host, int chunk_frames)
{
    return fk_foveate_host_any(h, params, width, height, channels, n_frames, fix_xy_host,
                               in_host, out_host, chunk_frames, 0);
}

int fk_foveate_host_f32(fk_handle *h, const fk_params *params, int width, int height,
                        int channels, int n_frames, const double *fix_xy_host,
                        const float *in_host, float *out_host, int chunk_frames)
{
    return fk_foveate_host_any(h, params, width, height, channels, n_frames, fix_xy_host,
                               in_host, out_host, chunk_frames, 1);
}

int fk_host_alloc(size_t bytes, void **out)
{
    if (!out) return fk_fail(nullptr, FK_EINVAL, "out is NULL");
    cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) return fk_cuda_fail(nullptr, e, "cudaHostAlloc");
    return FK_OK;
}

int fk_host_free(void *ptr)
{
    if (!ptr) return FK_OK;
    cudaError_t e = cudaFreeHost(ptr);
    if (e != cudaSuccess) return fk_cuda_fail(nullptr, e, "cudaFreeHost");
    return FK_OK;
}

/* --------------------------------------------------------------------- measurement */
int fk_measure_fp32_peak(fk_handle *h, double *tflops, double *ms_out)
{
    if (!h || !tflops) return fk_fail(h, FK_EINVAL, "NULL argument");
    FK_CUDA(h, cudaSetDevice(h->device));
    const int sm = h->prop.multiProcessorCount;
    if (!h->probe) FK_CUDA(h, cudaMalloc(&h->probe, (size_t)sm * 8 * 256 * sizeof(float)));
    const int iters = 40000;
    cudaEvent_t a, b;
    FK_CUDA(h, cudaEventCreate(&a));
    FK_CUDA(h, cudaEventCreate(&b));
    cudaStream_t s = h->streams[0];
    for (int i = 0; i < 3; i++) FK_CUDA(h, fk_launch_fp32_probe(h->probe, sm, iters, s));
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        FK_CUDA(h, cudaEventRecord(a, s));
        FK_CUDA(h, fk_launch_fp32_probe(h->probe, sm, iters, s));
        FK_CUDA(h, cudaEventRecord(b, s));
        FK_CUDA(h, cudaEventSynchronize(b));
        float ms = 0;
        FK_CUDA(h, cudaEventElapsedTime(&ms, a, b));
        best = ms < best ? ms : best;
    }
    h->launches += 8;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 16.0 * (double)iters * (double)sm * 8.0 * 256.0;
    *tflops = flops / (best * 1e-3) / 1e12;
    if (ms_out) *ms_out = best;
    return FK_OK;
}

/* ------------------------------------------------------------ SSIM (validation tool) */
int fk_ssim_u8(fk_handle *h, const uint8_t *ref_dev, const uint8_t *test_dev, int width,
               int height, int channels, const double *window_host, int window_size, double c1,
               double c2, double *values_dev, int accumulate, void *stream)
{
    if (!h || !ref_dev || !test_dev || !window_host || !values_dev)
        return fk_fail(h, FK_EINVAL, "NULL argument");
    if (channels != 1 && channels != 3)
        return fk_fail(h, FK_EINVAL, "channels must be 1 or 3, got %d", channels);
    if (window_size < 1 || window_size > 15)
        return fk_fail(h, FK_EINVAL, "window_size must be in [1, 15], got %d", window_size);
    if (width < window_size || height < window_size) /* quality.py:88-89 */
        return fk_fail(h, FK_EINVAL, "images must be at least %dpx per side", window_size);
    FK_CUDA(h, cudaSetDevice(h->device));
    FK_CUDA(h, fk_launch_ssim_map(ref_dev, test_dev, width, height, channels, window_host,
                                  window_size, c1, c2, values_dev, accumulate, as_stream(stream)));
    h->launches += 1;
    return FK_OK;
}

int fk_ssim_stats(fk_handle *h, double *values_dev, int64_t count, double divisor,
                  double *stats_host, void *stream)
{
    if (!h || !values_dev || !stats_host) return fk_fail(h, FK_EINVAL, "NULL argument");
    if (count < 1) return fk_fail(h, FK_EINVAL, "empty map");
    if (!(divisor > 0.0)) return fk_fail(h, FK_EINVAL, "divisor must be positive");
    FK_CUDA(h, cudaSetDevice(h->device));
    if (!h->ssim_stats) FK_CUDA(h, cudaMalloc(&h->ssim_stats, 3 * sizeof(double)));
    cudaStream_t s = as_stream(stream);
    FK_CUDA(h, fk_launch_ssim_stats(values_dev, (long long)count, divisor, h->ssim_stats, s));
    h->launches += 1;
    FK_CUDA(h, cudaMemcpyAsync(stats_host, h->ssim_stats, 3 * sizeof(double),
                               cudaMemcpyDeviceToHost, s));
    FK_CUDA(h, cudaStreamSynchronize(s));
    return FK_OK;
}

} /* extern "C" */
