/* fk_internal.h -- structures shared by the translation units of libfovea.so. */
#ifndef FK_INTERNAL_H_
#define FK_INTERNAL_H_

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/fovea.h"

/* Per-frame plan header, 8 x int32 (also what fk_plan_read_lengths returns). */
enum {
    FK_META_SX = 0,
    FK_META_SY = 1,
    FK_META_GW = 2,
    FK_META_GH = 3,
    FK_META_FGY = 4,
    FK_META_FGX = 5,
    FK_META_LMAX = 6,
    FK_META_STATUS = 7,
    FK_META_WORDS = 8
};

#define FK_LUT_DEFAULT_MAX 255
#define FK_PLAN_THREADS 256
#define FK_PLAN_THREADS_MAX 1024

/*
 * Work items.  The plan kernel turns the fragments of a frame into strips: rectangles at
 * most FK_RECT pixels wide and FK_STRIP_ROWS pixels tall that share one filter -- vertically
 * adjacent fragments with the same taps are merged, which is exact (every output pixel
 * depends only on the image and its filter) and lets them share the horizontal pass over
 * the 2r halo rows between them.  Strips are appended to one of FK_NCLASS lists by tap
 * count, so that each list can be rendered by a kernel launch whose shared-memory layout
 * fits its longest filter.  Inside a list, a frame's items are contiguous.
 */
#define FK_RECT 32
#define FK_STRIP_ROWS 1024
#define FK_NCLASS 7
/* Classes 0..4 are rendered by the fast kernels, each launch with the shared-memory layout
 * of the class's longest filter.  Frames staged by TMA (uint8 and float32): fk_blur_tma, 3
 * resident CTAs per SM -- its register budget -- while the layout fits three times (uint8: up
 * to 105 taps; float32, whose raw blocks are four times the size: up to ~55), else 2.  Buffers
 * TMA cannot describe: fk_blur_cols, 3 CTAs per SM in classes 0 and 1, 2 beyond, with the taps
 * walked in panels in class 4.  Class 5 (longer filters) goes to the generic kernel, class 6
 * holds the identity fragments (L = 1), plain copies.  (Merging classes 0-2 was measured:
 * nothing on uint8, 3-22 % slower on float32.) */
#ifndef FK_CLASS_L0 /* -DFK_CLASS_L0=.. -DFK_CLASS_L1=..: class-boundary experiments */
#define FK_CLASS_L0 23
#define FK_CLASS_L1 47
#endif
#define FK_CLASS_L2 69
#define FK_CLASS_L3 89
#define FK_CLASS_L4 127
#define FK_CLASS_GENERIC 5
#define FK_CLASS_COPY 6
/* counters: [0, N) items at the FRONT of each class list, [N, 2N) render cursors, [2N, 3N) items
 * at the BACK of each list, [3N] frames whose fixation lies outside the image */
#define FK_COUNTER_BACK (2 * FK_NCLASS)
#define FK_COUNTER_BAD (3 * FK_NCLASS)
#define FK_COUNTER_WORDS (3 * FK_NCLASS + 1)
/* strips taller than this many rows go to the front of their list (fk_class_list) */
#define FK_TALL_ROWS(L) ((L) <= FK_CLASS_L2 ? 64 : 128)

static __host__ __device__ __forceinline__ int fk_class_of(int L)
{
    return L <= 1 ? FK_CLASS_COPY
         : L <= FK_CLASS_L0 ? 0
         : L <= FK_CLASS_L1 ? 1
         : L <= FK_CLASS_L2 ? 2
         : L <= FK_CLASS_L3 ? 3
         : L <= FK_CLASS_L4 ? 4 : FK_CLASS_GENERIC;
}
/* longest / shortest filter a class can hold */
static inline int fk_class_lmax(int k)
{
    static const int lmax[FK_NCLASS] = {FK_CLASS_L0, FK_CLASS_L1, FK_CLASS_L2, FK_CLASS_L3,
                                        FK_CLASS_L4, 8191, 1};
    return lmax[k];
}
static inline int fk_class_lmin(int k)
{
    static const int lmin[FK_NCLASS] = {3, FK_CLASS_L0 + 2, FK_CLASS_L1 + 2, FK_CLASS_L2 + 2,
                                        FK_CLASS_L3 + 2, FK_CLASS_L4 + 2, 1};
    return lmin[k];
}

/* 16 bytes, loaded as one uint4 by the render kernels. */
struct fk_item {
    uint32_t frame;
    uint32_t xy;       /* x0 | y0 << 16 */
    uint32_t geom;     /* fw | L << 8 | fh << 21   (fw <= 255, L <= 8191, fh <= 2047) */
    uint32_t taps_off; /* offset of the L taps inside fk_plan_dev::taps, or FK_ITEM_MIXED | radii */
};
/*
 * Mixed items (fragments narrower than FK_RECT, canonical taps only).  The column-partitioned
 * kernels give each of their four warps 8 pixels of a strip in BOTH passes, with the warp's own
 * copy of the taps, so nothing forces the four columns of a strip to share a filter: an
 * aligned group of FK_RECT / F cells of a grid row whose tap counts differ becomes ONE item
 * whose taps_off holds FK_ITEM_MIXED and the radius r_w = (L_w - 1) / 2 of the filter of
 * pixel column 8 w at bits [6 w, 6 w + 6); `L` is the longest of them (it picks the class, the
 * tile rows and the TMA box), and the taps of radius r start at r * r (the canonical table).
 * Without them such cells are items 8 or 16 pixels wide that leave three or two warps idle.
 * Only fk_blur_tma reads mixed items; fk_launch_blur re-emits a plan's items without them
 * before it has to fall back to another kernel.
 */
#define FK_ITEM_MIXED 0x80000000u

/* Device-side view of a plan, passed by value to kernels. */
struct fk_plan_dev {
    int width, height, fragment;
    int cap;             /* per-frame stride of the cell arrays */
    int nsub_x;          /* strips per fragment across: ceil(fragment / FK_RECT) */
    int nsub_y;          /* strips per fragment down: ceil(fragment / FK_STRIP_ROWS) */
    int strip_rows;      /* tallest strip the plan kernel merges fragments into (fk_strip_rows_for) */
    int mixed;           /* emit mixed items (FK_ITEM_MIXED) for groups of cells that differ */
    int canonical;       /* taps are the canonical table: the filter of radius r starts at r * r */
    int self_zero;       /* one-frame plans: the plan kernel zeroes `counters` itself (no memset node) */
    int y_lo, y_hi;      /* only rectangles whose first row lies in [y_lo, y_hi) become items (a request
                            renders a frame in two bands from two plans, fk_request_create) */
    int32_t *info_out;   /* optional host-mapped words the plan kernel fills for frame 0:
                            [0, 8) meta, [8] rejected fixations, [16, 16 + cells) tap counts */
    size_t items_cap;    /* entries per class list: max_frames * cap * nsub_x * nsub_y */
    fk_item *items;      /* [FK_NCLASS][items_cap] */
    int32_t *counters;   /* FK_COUNTER_WORDS words, see FK_COUNTER_BACK */
    double *sigma;       /* [frames][cap] */
    int32_t *raw_length; /* [frames][cap] */
    int32_t *length;     /* [frames][cap], foveal cell forced to 1 */
    int32_t *offset;     /* [frames][cap], tap offset inside `taps` */
    int32_t *strip;      /* [frames][cap], scratch of the plan kernel: grid rows of the strip a
                            cell heads (0: the cell belongs to a strip headed further up) */
    int32_t *meta;       /* [frames][FK_META_WORDS] */
    const float *taps;   /* fp32 tap table the offsets index (canonical LUT or custom) */
};

/*
 * A class list has two ends.  The persistent CTAs of a render draw items in list order, so the
 * items drawn last decide how long the launch's tail is: the plan kernel puts the TALL strips
 * of every frame at the front of the list's region and the short ones at its back (filled
 * downwards from items_cap - 1), and item i of the list is front[i] for i < n_front, else
 * back[i - n_front] counted from the end.  Tall first is within 1-4 % of longest-processing-time
 * order on the bench workloads (tools/strip_model.py), against 3-19 % for frame order.
 */
struct fk_class_list {
    const fk_item *base;
    size_t last; /* items_cap - 1 */
    int n_front, n_items;
#ifdef __CUDACC__
    __device__ __forceinline__ const fk_item *at(int i) const
    {
        return i < n_front ? base + i : base + (last - (size_t)(i - n_front));
    }
#endif
};
#ifdef __CUDACC__
static __device__ __forceinline__ fk_class_list fk_list_of(const fk_plan_dev &pd, int klass)
{
    fk_class_list l;
    l.base = pd.items + (size_t)klass * pd.items_cap;
    l.last = pd.items_cap - 1;
    l.n_front = pd.counters[klass];
    l.n_items = l.n_front + pd.counters[FK_COUNTER_BACK + klass];
    return l;
}
#endif

/* Density-map source of the sigma field (map == nullptr: retinal model). */
struct fk_density_dev {
    const uint8_t *map; /* device, map_h x map_w */
    int map_w, map_h;
    double sigma_max;
};

struct fk_handle {
    int device = -1;
    cudaDeviceProp prop{};
    std::string err;
    /* canonical LUT: all odd L <= lut_max, filter L at [r*r, r*r+L) */
    int lut_max = 0;
    double *lut64 = nullptr;
    float *lut32 = nullptr;
    int variant = 0;
    int64_t launches = 0;
    /* the class launches of one render run side by side: the class lists cover disjoint
     * pixels, so the CTAs of the next class fill the SMs the previous one's tail leaves idle
     * (fk_launch_blur forks from the caller's stream and joins back into it) */
    static const int kSide = FK_NCLASS - 1;
    cudaStream_t side[kSide] = {};
    cudaEvent_t ev_fork = nullptr;
    cudaEvent_t ev_done[kSide] = {};
    int serial_classes = 0; /* fk_set_kernel_variant(v | 16): all classes on the caller's stream */
    int no_mixed = 0;       /* fk_set_kernel_variant(v | 32): plans without mixed items (A/B runs) */
    /* pipeline resources of fk_foveate_host_* */
    static const int kStreams = 3;
    cudaStream_t streams[kStreams] = {nullptr, nullptr, nullptr};
    void *stage_in[kStreams] = {nullptr, nullptr, nullptr};
    void *stage_out[kStreams] = {nullptr, nullptr, nullptr};
    size_t stage_bytes = 0;
    double *stage_fix[kStreams] = {nullptr, nullptr, nullptr};
    fk_plan *stage_plan[kStreams] = {nullptr, nullptr, nullptr};
    int stage_w = 0, stage_h = 0, stage_f = 0, stage_frames = 0;
    /* scratch for the FP32 peak probe */
    float *probe = nullptr;
    double *ssim_stats = nullptr; /* [3] device scratch of fk_ssim_stats */
    /* the tensor maps of the last fk_blur_tma launch per (element type, class): a render of the
     * same buffer with the same geometry (a stream of frames through one buffer, a bench loop)
     * does not encode them again */
    struct tmap_slot {
        const void *in = nullptr;
        int width = 0, height = 0, frames = 0, nq = 0, shift = 0;
        alignas(64) unsigned char maps[6 * 128];
    } tmap_cache[2 * FK_NCLASS];
};

struct fk_plan {
    fk_handle *h = nullptr;
    int max_frames = 0;
    int n_frames = 0;     /* frames planned by the last fk_plan_model / set_grid */
    int bound_length = 1; /* host upper bound of the tap count over those frames */
    int custom = 0;       /* taps point at custom_taps instead of the canonical LUT */
    float *custom_taps = nullptr;
    int custom_cap = 0;
    double *fix_dev = nullptr; /* [max_frames][2] staging for host fixations */
    uint8_t *density_map = nullptr; /* device copy of the last density map */
    size_t density_cap = 0;
    int32_t *request_info = nullptr; /* set around the capture of a request: fk_plan_dev::info_out */
    fk_plan_dev d{};
};

/* Tallest merged strip for a batch of n_frames frames of width x height pixels: taller strips
 * share more of the horizontal pass (the 2r halo rows between merged fragments) and cost fewer
 * item set-ups, shorter ones give the persistent CTAs of a small batch enough items to share.
 * FK_STRIP_ROWS_FORCE in the environment overrides it (tuning runs). */
int fk_strip_rows_for(int n_frames, int width, int height);

/* error plumbing (fk_api.cu) */
int fk_fail(fk_handle *h, int code, const char *fmt, ...);
int fk_cuda_fail(fk_handle *h, cudaError_t e, const char *what);
#define FK_CUDA(h, call)                                            \
    do {                                                            \
        cudaError_t e__ = (call);                                   \
        if (e__ != cudaSuccess) return fk_cuda_fail((h), e__, #call); \
    } while (0)

/* kernels (fk_plan.cu, fk_blur.cu) */
cudaError_t fk_launch_build_lut(double *lut64, float *lut32, int max_length, cudaStream_t s);
cudaError_t fk_launch_plan(const fk_plan_dev &pd, const fk_params &prm, int n_frames,
                           const double *fix_dev, const fk_density_dev &den, cudaStream_t s);
cudaError_t fk_launch_order(const fk_plan_dev &pd, int n_frames, cudaStream_t s);
cudaError_t fk_launch_blur(fk_handle *h, const fk_plan_dev &pd, const void *in, void *out,
                           int n_frames, int channels, int is_f32, int bound_length,
                           cudaStream_t s, int *launches);
cudaError_t fk_launch_blur_fast(fk_handle *h, const fk_plan_dev &pd, int klass, const void *in,
                                void *out, int n_frames, int channels, int is_f32,
                                int class_length, cudaStream_t s, bool *taken);
cudaError_t fk_launch_blur_cols(fk_handle *h, const fk_plan_dev &pd, int klass, const void *in,
                                void *out, int n_frames, int is_f32, int class_length,
                                cudaStream_t s, bool *taken);
/* true when fk_blur_tma can stage this RGB batch by TMA (16-byte aligned base and rows) */
bool fk_blur_tma_usable(const void *in, int width, int height, int is_f32);
cudaError_t fk_launch_fp32_probe(float *buf, int sm_count, int iters, cudaStream_t s);
/* fk_ssim.cu */
cudaError_t fk_launch_ssim_map(const uint8_t *ref, const uint8_t *test, int W, int H, int C,
                               const double *window, int n, double c1, double c2,
                               double *values, int accumulate, cudaStream_t s);
cudaError_t fk_launch_ssim_stats(double *values, long long count, double divisor,
                                 double *stats_dev, cudaStream_t s);

/* Host replica of the grid geometry (tiling.py:15-28). */
static inline int fk_span_count(int extent, int F, int offset)
{
    int n = extent > offset ? (extent - offset + F - 1) / F : 0;
    return n + (offset > 0 ? 1 : 0);
}

#endif /* FK_INTERNAL_H_ */
