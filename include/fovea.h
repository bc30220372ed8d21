/*
 * fovea.h -- C ABI of libfovea.so: blockwise foveated rendering on one B200 (sm_100a).
 *
 * The reference (foveakit 0.1.0, pure Python) has no FFI seam; its boundary for this
 * path is the Python API re-exported at pkg/src/foveakit/__init__.py:13-62.  Each entry
 * point below names the reference function(s) it replaces (file:line under
 * /root/reference/pkg/src/foveakit/).  paper_2012_08655_b200/_native.py is the ctypes
 * binding; INTEGRATION.md shows the stub a foveakit maintainer would add.
 *
 * Conventions
 *   - plain pointers and sizes only; every function returns an int status
 *     (FK_OK / FK_EINVAL -> ValueError / FK_ECUDA, FK_ENOMEM -> RuntimeError) and
 *     leaves a message retrievable with fk_last_error().
 *   - "dev" pointers are device memory on the handle's GPU, "host" pointers are host
 *     memory.  `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *   - frames are row-major interleaved [N][H][W][C], C in {1,3}, uint8 or float32
 *     (imaging.py:19-39); fixations are double (x, y) pairs in pixels.
 *   - all functions are re-entrant across handles; one handle serves one device and may
 *     be used from one thread at a time (blockwise.py:13-15, SPEC.md "Concurrency Model").
 *   - there is no CPU fallback: without a CUDA device fk_create fails with FK_ECUDA.
 */
#ifndef FOVEA_H_
#define FOVEA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FK_OK 0
#define FK_EINVAL 1 /* bad argument: the Python shim raises ValueError(fk_last_error) */
#define FK_ECUDA 2  /* CUDA runtime failure or no device */
#define FK_ENOMEM 3

#define FK_ABI_VERSION 1

typedef struct fk_handle fk_handle; /* one GPU: canonical tap LUT, streams, scratch */
typedef struct fk_plan fk_plan;     /* device-resident plans for up to max_frames frames */

/*
 * POD mirror of FoveationParams (retinal.py:34-44) plus the scalars the reference
 * evaluates on the host with Python's math module; they are passed in so that the
 * device sigma map is bit-identical to the reference's:
 *   log_inv_ct0 = math.log(1.0 / ct0)                      retinal.py:129
 *   two_pi      = 2.0 * math.pi                            retinal.py:155
 *   fmax        = params.max_cpd()                         retinal.py:63-65
 *   d_corner    = math.hypot(w / 2.0, h / 2.0)             retinal.py:111
 */
typedef struct fk_params {
    double alpha;
    double e2;
    double ct0;
    double e_corner;
    double strength;
    double log_inv_ct0;
    double two_pi;
    double fmax;
    double d_corner;
    int32_t fragment_size; /* >= 4 (blockwise.py:46-47) */
    /* 1: shift from the fixation (plan(..., use_shift=True), blockwise.py:207);
     * 0: no shift; 2: explicit (shift_x, shift_y), as build_sigma_field's `shift`
     * argument allows (retinal.py:159-161). */
    int32_t use_shift;
    int32_t shift_x, shift_y;
} fk_params;

/* Host-side view of one frame's plan, filled by fk_plan_read (arrays are caller-owned,
 * each with room for fk_plan_cell_capacity() entries; NULL pointers are skipped). */
typedef struct fk_plan_view {
    int32_t shift_x, shift_y; /* compute_fragment_shift, blockwise.py:39-51 */
    int32_t grid_w, grid_h;   /* len(fragment_spans(...)), tiling.py:15-28 */
    int32_t foveal_gy, foveal_gx; /* cell_of(...), tiling.py:36-39, blockwise.py:128 */
    int32_t max_length;       /* largest tap count used by the frame */
    int32_t status;           /* 0 ok; 1 fixation outside image (retinal.py:73-74) */
    double *sigma;            /* [grid_h*grid_w] SigmaField.sigma, retinal.py:159-177 */
    int32_t *raw_length;      /* filter_length(sigma), filters.py:20-27 */
    int32_t *length;          /* same with the foveal cell forced to 1, blockwise.py:129-130 */
} fk_plan_view;

typedef struct fk_device_info {
    int32_t device;
    int32_t sm_count;
    int32_t cc_major, cc_minor;
    int32_t clock_khz;       /* max SM clock */
    int32_t l2_bytes;
    int64_t global_mem_bytes;
    int32_t max_smem_optin;  /* bytes of shared memory per CTA (opt-in) */
    char name[64];
} fk_device_info;

/* ---- lifecycle ----------------------------------------------------------------- */
int fk_abi_version(void);
int fk_device_count(int *count);
int fk_create(int device, fk_handle **out);
int fk_destroy(fk_handle *h);
const char *fk_last_error(const fk_handle *h); /* h may be NULL: last error of this thread */
int fk_get_device_info(fk_handle *h, fk_device_info *out);

/* ---- Gaussian tap LUT ---------------------------------------------------------- */
/* Replaces gaussian_filter_1d / _bank_from_lengths (filters.py:30-38,77-85): builds, on
 * the device, the taps of every odd length L <= max_length at the representative
 * sigma = L / 6.  Filter L occupies [r*r, r*r + L) of the table, r = (L-1)/2.
 * fk_create builds the table up to 255 taps; planning grows it when needed. */
int fk_build_lut(fk_handle *h, int max_length, void *stream);
int fk_lut_max_length(fk_handle *h, int *max_length);
/* Copy the fp64 taps of one odd length to the host (FilterBank.filters). */
int fk_lut_read(fk_handle *h, int length, double *taps_host);

/* ---- planning: shift -> sigma field -> tap counts -> foveal cell ----------------- */
int fk_plan_create(fk_handle *h, int width, int height, int fragment_size,
                   int max_frames, fk_plan **out);
int fk_plan_destroy(fk_plan *p);
int fk_plan_cell_capacity(const fk_plan *p); /* per-frame stride of the cell arrays */

/* Replaces, for n_frames frames at once: compute_fragment_shift (blockwise.py:39-51),
 * fragment_spans / span_midpoints / cell_of (tiling.py:15-39), eccentricity_of,
 * cutoff_cpd, cutoff_cpp, sigma_at, build_sigma_field (retinal.py:97-177),
 * filter_length (filters.py:20-27) and the foveal forcing of build_blur_grid
 * (blockwise.py:107-133).  fix_xy holds n_frames (x, y) pairs, on the host
 * (fix_on_device = 0, copied stream-ordered) or already on the device. */
int fk_plan_model(fk_plan *p, const fk_params *params, int n_frames, const double *fix_xy,
                  int fix_on_device, void *stream);

/* Replaces ingest_density_map (retinal.py:180-231) and the density branch of plan
 * (blockwise.py:208-213): the 1-channel map (host memory, map_h x map_w bytes) is resampled
 * bilinearly at the fragment midpoints of every frame's shifted tiling and
 * sigma = sigma_max * (1 - v / 255); tap counts, foveal forcing and work items follow as in
 * fk_plan_model.  Of `params` only fragment_size, use_shift and shift_x/y are used. */
int fk_plan_density(fk_plan *p, const fk_params *params, int n_frames, const double *fix_xy,
                    int fix_on_device, const uint8_t *map_host, int map_w, int map_h,
                    double sigma_max, void *stream);

/* Replaces render()'s use of an arbitrary (BlurGrid, FilterBank) pair
 * (blockwise.py:156-186) for ONE frame: the caller supplies the shift, the per-cell tap
 * counts (odd, >= 1) and offsets into `coeffs` (FilterBank.cumulative_sizes layout,
 * filters.py:41-49).  All arrays are host memory; grid dims must match the tiling
 * (else FK_EINVAL, the reference's "does not match image" error). */
int fk_plan_set_grid(fk_plan *p, int shift_x, int shift_y, int grid_w, int grid_h,
                     const int32_t *length, const int32_t *offset, const double *coeffs,
                     int n_coeffs, void *stream);

/* Synchronising read-back of one frame's plan (for BlurGrid / SigmaField objects). */
int fk_plan_read(fk_plan *p, int frame, fk_plan_view *out, void *stream);
/* Read-back of tap counts for frames [first, first+count): lengths_host is
 * [count][cell_capacity], meta_host is [count][8] =
 * {shift_x, shift_y, grid_w, grid_h, foveal_gy, foveal_gx, max_length, status}. */
int fk_plan_read_lengths(fk_plan *p, int first, int count, int32_t *lengths_host,
                         int32_t *meta_host, void *stream);

/* The render kernels' work lists of the last plan, for accounting (bench.py reports the FLOPs
 * the merged strips execute next to the algorithmic count of costs.py).  A plan holds
 * fk_plan_item_classes() lists by tap count (the last one: identity fragments, plain copies);
 * an item is four uint32: frame, x0 | y0 << 16, width | taps << 8 | height << 21, tap offset --
 * a rectangle at most 32 pixels wide of vertically adjacent fragments that share one filter
 * (merging them is exact: an output pixel depends only on the image and its filter,
 * blockwise.py:136-153).  *count receives the list's length; up to `capacity` items are
 * copied to items_host (may be NULL to query the length).  Synchronises the stream. */
int fk_plan_item_classes(void);
int fk_plan_read_items(fk_plan *p, int klass, uint32_t *items_host, int capacity, int *count,
                       void *stream);

/* Frames of the last fk_plan_model / fk_plan_density call whose fixation lies outside the
 * image or is not a number (retinal.py:73-74 raises ValueError("fixation ... outside image")).
 * Host fixations are rejected before anything is launched; fixations that are already on
 * the device can only be checked there: the plan kernel counts them, copies those frames
 * through unchanged and this call reads the count (synchronises the stream). */
int fk_plan_status(fk_plan *p, int *bad_frames, void *stream);

/* ---- render: the per-fragment separable blur -------------------------------------- */
/* Replaces render / _render_cell (blockwise.py:136-186) + quantize_u8 (convolve.py:9-15)
 * for the n_frames frames planned in `p` (n_frames must equal the planned count: the work
 * lists cover every planned frame).  in/out are device pointers, [n][H][W][C]. */
int fk_render_u8(fk_handle *h, const fk_plan *p, const uint8_t *in_dev, uint8_t *out_dev,
                 int n_frames, int channels, void *stream);
/* Same arithmetic on float32 frames, result left unquantised (BASELINE config 5). */
int fk_render_f32(fk_handle *h, const fk_plan *p, const float *in_dev, float *out_dev,
                  int n_frames, int channels, void *stream);

/* Kernel selection for tests and profiling.  0 = default (RGB frames staged by TMA:
 * fk_blur_tma; RGB buffers TMA cannot describe: fk_blur_cols; gray: fk_blur_fast; generic
 * kernel where none of them takes a class), 1 = generic kernel only, 2 = fast kernels with
 * plain-load staging (no TMA), 3 = row-partitioned fk_blur_fast for RGB as well, 4 =
 * fk_blur_cols for every RGB class, 5 = same as 0, 6 = fk_blur_tma with one raw buffer.
 * Adding 16 launches the tap-count classes of a render one after the other on the caller's
 * stream instead of side by side on forked streams; adding 32 makes the plans built from then
 * on keep neighbouring fragments with different filters as separate work items instead of
 * one item with a filter per 8-pixel column.  All variants produce bit-identical output.
 * Returns the previous value. */
int fk_set_kernel_variant(fk_handle *h, int variant);
/* Number of kernel launches issued through this handle so far (bench "gpu_launches"). */
int64_t fk_launch_count(const fk_handle *h);

/* ---- request: one gaze-contingent frame as ONE graph launch ------------------------- */
/* The per-message work of the reference's streaming loop (service.py:192-238: apply the
 * fixation, render_frame service.py:73-81, send the frame) for an image that stays in HBM:
 * fixation upload -> plan (retinal model) -> render -> frame and plan summary to pinned host
 * memory, captured once as a CUDA graph for fixed parameters and buffers and replayed per
 * request, so a request costs one launch call and no synchronising read-back.
 *   fk_request_create  captures on `stream` (not the legacy default stream).  `p` must be a
 *                      one-frame-or-larger plan of the image's geometry and stays bound to the
 *                      request; in_dev / out_dev are [H][W][C] device buffers, out_host (may be
 *                      NULL) pinned host memory of the same size.  The graph holds the class
 *                      launches of the longest filter any fixation inside the image can need.
 *                      With out_host, frames of a megabyte and more are rendered in two
 *                      bands (the rows above and below FK_REQUEST_SPLIT percent of the height,
 *                      default 55, read at creation; 0: one band) from two plans of the same
 *                      fixation, and the upper band travels to out_host while the lower one
 *                      renders; out_dev and out_host hold the whole frame when the stream has
 *                      been synchronised, whatever the split.
 *   fk_request_launch  queues one request for fixation (fx, fy) -- which must lie inside the
 *                      image, the caller clamps as service.py:58-63 does -- on `stream`.
 *   fk_request_info    pinned host words, valid once the stream has been synchronised:
 *                      [0, 8) the frame's plan header (fk_plan_read_lengths), [8] frames whose
 *                      fixation was rejected on the device (0 or 1), [16, 16 + cells) the tap
 *                      counts of the fragments, row-major grid_h x grid_w. */
typedef struct fk_request fk_request;
int fk_request_create(fk_handle *h, fk_plan *p, const fk_params *params, const void *in_dev,
                      void *out_dev, void *out_host, int channels, int is_f32, void *stream,
                      fk_request **out);
int fk_request_launch(fk_request *r, double fx, double fy, void *stream);
const int32_t *fk_request_info(const fk_request *r);
int fk_request_destroy(fk_request *r);

/* ---- foveate: host frames in, host frames out (the call a foveakit user makes) ----- */
/* Replaces foveate() (blockwise.py:223-243) for a batch held in HOST memory: pipelines
 * H2D copy -> plan -> render -> D2H copy over internal streams in chunks of
 * `chunk_frames` (0 = pick).  Pinned buffers (fk_host_alloc) overlap fully. */
int fk_foveate_host_u8(fk_handle *h, const fk_params *params, int width, int height,
                       int channels, int n_frames, const double *fix_xy_host,
                       const uint8_t *in_host, uint8_t *out_host, int chunk_frames);
int fk_foveate_host_f32(fk_handle *h, const fk_params *params, int width, int height,
                        int channels, int n_frames, const double *fix_xy_host,
                        const float *in_host, float *out_host, int chunk_frames);
int fk_host_alloc(size_t bytes, void **out); /* pinned host memory */
int fk_host_free(void *ptr);

/* ---- measurement helpers ------------------------------------------------------------ */
/* Dependent-free FFMA loop on every SM; returns achieved FP32 TFLOP/s (2 flop per FMA)
 * measured with CUDA events.  The roofline denominator when it is FP32-bound. */
int fk_measure_fp32_peak(fk_handle *h, double *tflops, double *ms);

/* ---- validation: SSIM map on the device ---------------------------------------------- */
/* Replaces quality.ssim_map (quality.py:82-103): BT.601 luma of both images (quality.py:31-35),
 * the five separable windowed means over fully-valid windows (quality.py:45-48) and the SSIM
 * formula, fp64 throughout.  `ref_dev` / `test_dev`: device uint8 [height][width][channels],
 * channels 1 or 3.  `window_host`: the window_size (<= 15) normalised taps, evaluated by the
 * caller with the reference's expression (quality.py:38-42).  c1 = (K1 * range)^2,
 * c2 = (K2 * range)^2.  `values_dev`: device float64 [height - window_size + 1][width -
 * window_size + 1]; with accumulate != 0 the map is added onto what is there
 * (mean_ssim_map, quality.py:106-114). */
int fk_ssim_u8(fk_handle *h, const uint8_t *ref_dev, const uint8_t *test_dev, int width,
               int height, int channels, const double *window_host, int window_size, double c1,
               double c2, double *values_dev, int accumulate, void *stream);
/* Replaces _map_from_values (quality.py:70-79): divides the `count` values by `divisor`
 * in place (1.0: untouched), then stats_host[0..2] = mean, min, flat index of the first
 * minimum (np.argmin).  Synchronises the stream. */
int fk_ssim_stats(fk_handle *h, double *values_dev, int64_t count, double divisor,
                  double *stats_host, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FOVEA_H_ */
