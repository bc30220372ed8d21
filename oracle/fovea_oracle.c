/*
 * fovea_oracle.c -- CPU restatement of the blockwise foveation path of foveakit.
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_2012_08655_b200) never calls into it and has no CPU fallback.
 *
 * Parity status: PINNED.  tests/test_oracle_golden.py checks every function here
 * against vectors produced by the reference itself (tests/golden/make_golden.py,
 * run in the build container against /root/reference/pkg/src) and against the
 * known-answer values held by the reference's own tests.
 *
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/pkg/src/foveakit/).  All arithmetic is IEEE fp64 with one
 * rounding per operation (build with -ffp-contract=off), in the reference's
 * left-to-right order, because the sigma map has to agree bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define FO_OK 0
#define FO_EINVAL 1

typedef struct {
    double alpha;      /* retinal.py:37 */
    double e2;         /* retinal.py:38 */
    double ct0;        /* retinal.py:39 */
    double e_corner;   /* retinal.py:40 */
    double strength;   /* retinal.py:42 */
    int fragment_size; /* retinal.py:43 */
    int has_f_max;     /* retinal.py:41: f_max is None or a float */
    double f_max;
    /* Host scalars the reference evaluates with Python's math module
     * (retinal.py:111,129,155).  Python's math.hypot is not libm's hypot, so the
     * caller passes d_corner in; <= 0 means "compute it here with libm". */
    double d_corner;
} fo_params;

/* blockwise.py:39-51 -- ((floor(f) - F//2) mod F), Python's non-negative modulo. */
int fo_fragment_shift(double fx, double fy, int F, int *sx, int *sy)
{
    if (F < 4) return FO_EINVAL;
    long dx = (long)floor(fx) - F / 2;
    long dy = (long)floor(fy) - F / 2;
    long mx = dx % F, my = dy % F;
    if (mx < 0) mx += F;
    if (my < 0) my += F;
    *sx = (int)mx;
    *sy = (int)my;
    return FO_OK;
}

/* tiling.py:15-28 -- number of [start,end) spans covering [0,extent). */
int fo_span_count(int extent, int F, int offset)
{
    int n = 0;
    for (int s = offset; s < extent; s += F) n++;
    if (offset > 0) n++;
    return n;
}

/* tiling.py:15-28 -- spans[2*i], spans[2*i+1] = start, end of span i. */
int fo_fragment_spans(int extent, int F, int offset, int64_t *spans)
{
    if (extent < 1 || offset < 0 || offset >= F) return -1;
    int n = 0;
    if (offset > 0) spans[2 * n++] = 0;
    for (int s = offset; s < extent; s += F) spans[2 * n++] = s;
    for (int i = 0; i + 1 < n; i++) spans[2 * i + 1] = spans[2 * (i + 1)];
    spans[2 * (n - 1) + 1] = extent;
    return n;
}

/* tiling.py:36-39 -- searchsorted(starts, coord, side="right") - 1, clamped. */
static int fo_cell_of(const int64_t *spans, int n, double coord)
{
    int idx = 0;
    while (idx < n && (double)spans[2 * idx] <= coord) idx++;
    idx -= 1;
    if (idx < 0) idx = 0;
    if (idx > n - 1) idx = n - 1;
    return idx;
}

/* filters.py:20-27 -- ceil(6*sigma), at least 1, forced up to odd. */
int fo_filter_length(double sigma)
{
    long n = (long)ceil(6.0 * sigma);
    if (n < 1) n = 1;
    if (n % 2 == 0) n += 1;
    return (int)n;
}

/* filters.py:30-38,77-79 -- taps for the representative sigma = L/6. */
void fo_gaussian_taps(int L, double *w)
{
    if (L <= 1) { w[0] = 1.0; return; }
    double sigma = (double)L / 6.0;
    int r = (L - 1) / 2;
    double sum = 0.0;
    for (int i = 0; i < L; i++) {
        double k = (double)(i - r);
        w[i] = exp(-(k * k) / (2.0 * sigma * sigma));
    }
    /* numpy's w.sum() is a pairwise sum; for < 128 taps it is an 8-way unrolled
     * loop, so the last bit of the normaliser can differ from a plain running
     * sum.  The reference's tests pin taps to 1e-9/1e-12, not to the bit. */
    for (int i = 0; i < L; i++) sum += w[i];
    for (int i = 0; i < L; i++) w[i] = w[i] / sum;
}

/*
 * retinal.py:159-177 (build_sigma_field) + retinal.py:97-156 (eccentricity_of,
 * cutoff_cpd, cutoff_cpp, sigma_at) + filters.py:20-27 + blockwise.py:107-133
 * (foveal cell forced to the identity filter).
 *
 * Outputs (row-major gh x gw): sigma, raw_length (before foveal forcing, what
 * build_bank sees), length (after forcing, what render uses).
 * shift[2] = (sx, sy); dims[2] = (gw, gh); foveal[2] = (gy, gx).
 */
int fo_plan(const fo_params *p, int W, int H, double fx, double fy, int use_shift,
            int *shift, int *dims, int *foveal, double *sigma, int *raw_length,
            int *length)
{
    if (W < 1 || H < 1 || p->fragment_size < 4) return FO_EINVAL;
    if (!(fx >= 0 && fx < W && fy >= 0 && fy < H)) return FO_EINVAL; /* retinal.py:73 */
    const int F = p->fragment_size;
    int sx = 0, sy = 0;
    if (use_shift) fo_fragment_shift(fx, fy, F, &sx, &sy);
    int gw = fo_span_count(W, F, sx), gh = fo_span_count(H, F, sy);
    int64_t *spx = malloc(sizeof(int64_t) * 2 * gw);
    int64_t *spy = malloc(sizeof(int64_t) * 2 * gh);
    fo_fragment_spans(W, F, sx, spx);
    fo_fragment_spans(H, F, sy, spy);

    const double LOG = log(1.0 / p->ct0);           /* retinal.py:129 */
    const double TWO_PI = 2.0 * M_PI;               /* retinal.py:155 */
    const double fmax = p->has_f_max                /* retinal.py:63-65 */
        ? p->f_max
        : p->e2 / (p->alpha * (0.0 + p->e2)) * LOG;
    const double d_corner = p->d_corner > 0.0 ? p->d_corner
                                              : hypot(W / 2.0, H / 2.0);

    for (int gy = 0; gy < gh; gy++) {
        double my = (double)(spy[2 * gy] + spy[2 * gy + 1]) / 2.0; /* tiling.py:33 */
        for (int gx = 0; gx < gw; gx++) {
            double mx = (double)(spx[2 * gx] + spx[2 * gx + 1]) / 2.0;
            double d = hypot(mx - fx, my - fy);                  /* retinal.py:110 */
            double e = d / d_corner * p->e_corner;               /* retinal.py:112 */
            double fdeg = p->e2 / (p->alpha * (e + p->e2)) * LOG; /* retinal.py:129 */
            double fpix = 0.5 * fdeg / fmax;                     /* retinal.py:140 */
            double s = p->strength / (TWO_PI * fpix);            /* retinal.py:155 */
            sigma[gy * gw + gx] = s;
            int L = fo_filter_length(s);
            raw_length[gy * gw + gx] = L;
            length[gy * gw + gx] = L;
        }
    }
    int fgy = fo_cell_of(spy, gh, fy), fgx = fo_cell_of(spx, gw, fx);
    length[fgy * gw + fgx] = 1;                                   /* blockwise.py:128-130 */
    shift[0] = sx; shift[1] = sy;
    dims[0] = gw; dims[1] = gh;
    foveal[0] = fgy; foveal[1] = fgx;
    free(spx); free(spy);
    return FO_OK;
}

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/*
 * blockwise.py:136-153 (_render_cell): clamp-to-edge gather of the padded tile,
 * horizontal pass over every tile row, vertical pass over the real-valued
 * intermediate.  `in` is read through get(); result for the fragment goes to
 * frag[(y - y0) * fw * C + (x - x0) * C + c] as fp64 (unquantised).
 */
static void render_cell_f64(const void *in, int is_f32, int H, int W, int C,
                            int x0, int x1, int y0, int y1, const double *g, int L,
                            double *tile, double *interm, double *frag)
{
    const int r = (L - 1) / 2;
    const int fw = x1 - x0, fh = y1 - y0;
    const int tw = fw + 2 * r, th = fh + 2 * r;
    const uint8_t *in8 = (const uint8_t *)in;
    const float *in32 = (const float *)in;
    for (int ty = 0; ty < th; ty++) {
        int yy = clampi(y0 - r + ty, 0, H - 1);
        for (int tx = 0; tx < tw; tx++) {
            int xx = clampi(x0 - r + tx, 0, W - 1);
            size_t src = ((size_t)yy * W + xx) * C;
            for (int c = 0; c < C; c++)
                tile[((size_t)ty * tw + tx) * C + c] =
                    is_f32 ? (double)in32[src + c] : (double)in8[src + c];
        }
    }
    for (int ty = 0; ty < th; ty++)
        for (int x = 0; x < fw; x++)
            for (int c = 0; c < C; c++) {
                double acc = 0.0;
                for (int k = 0; k < L; k++)
                    acc += tile[((size_t)ty * tw + x + k) * C + c] * g[k];
                interm[((size_t)ty * fw + x) * C + c] = acc;
            }
    for (int y = 0; y < fh; y++)
        for (int x = 0; x < fw; x++)
            for (int c = 0; c < C; c++) {
                double acc = 0.0;
                for (int k = 0; k < L; k++)
                    acc += interm[((size_t)(y + k) * fw + x) * C + c] * g[k];
                frag[((size_t)y * fw + x) * C + c] = acc;
            }
}

/*
 * blockwise.py:156-186 (render) with convolve.py:9-15 (quantize_u8) for u8 output.
 *
 * cell_len / cell_off (gh x gw) give each fragment's tap count and the offset of
 * its taps inside coeffs (the flattened bank, FilterBank.cumulative_sizes
 * semantics, filters.py:41-49).  out_kind: 0 = uint8 quantised, 1 = float64
 * unquantised (the fp32-frame oracle: _render_cell with quantize_u8 removed).
 */
int fo_render(const void *in, int in_is_f32, void *out, int out_kind, int H, int W,
              int C, int F, int sx, int sy, const int *cell_len, const int *cell_off,
              const double *coeffs, int threads)
{
    if (C != 1 && C != 3) return FO_EINVAL;                       /* blockwise.py:160 */
    int gw = fo_span_count(W, F, sx), gh = fo_span_count(H, F, sy);
    int64_t *spx = malloc(sizeof(int64_t) * 2 * gw);
    int64_t *spy = malloc(sizeof(int64_t) * 2 * gh);
    if (fo_fragment_spans(W, F, sx, spx) != gw || fo_fragment_spans(H, F, sy, spy) != gh) {
        free(spx); free(spy);
        return FO_EINVAL;
    }
    int bad = 0;
    for (int i = 0; i < gw * gh; i++)
        if (cell_len[i] < 1 || cell_len[i] % 2 == 0) bad = 1;
    if (bad) { free(spx); free(spy); return FO_EINVAL; }
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel num_threads(threads)
#endif
    {
        double *tile = NULL, *interm = NULL, *frag = NULL;
        size_t cap_t = 0, cap_i = 0, cap_f = 0;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int cell = 0; cell < gw * gh; cell++) {
            int gy = cell / gw, gx = cell % gw;
            int x0 = (int)spx[2 * gx], x1 = (int)spx[2 * gx + 1];
            int y0 = (int)spy[2 * gy], y1 = (int)spy[2 * gy + 1];
            int L = cell_len[cell];
            int fw = x1 - x0, fh = y1 - y0;
            if (L == 1) {                                         /* blockwise.py:141-143 */
                for (int y = y0; y < y1; y++) {
                    size_t o = ((size_t)y * W + x0) * C;
                    if (out_kind == 0) {
                        memcpy((uint8_t *)out + o, (const uint8_t *)in + o, (size_t)fw * C);
                    } else {
                        for (int i = 0; i < fw * C; i++)
                            ((double *)out)[o + i] = in_is_f32
                                ? (double)((const float *)in)[o + i]
                                : (double)((const uint8_t *)in)[o + i];
                    }
                }
                continue;
            }
            int r = (L - 1) / 2;
            size_t nt = (size_t)(fw + 2 * r) * (fh + 2 * r) * C;
            size_t ni = (size_t)fw * (fh + 2 * r) * C;
            size_t nf = (size_t)fw * fh * C;
            if (nt > cap_t) { free(tile); tile = malloc(nt * sizeof(double)); cap_t = nt; }
            if (ni > cap_i) { free(interm); interm = malloc(ni * sizeof(double)); cap_i = ni; }
            if (nf > cap_f) { free(frag); frag = malloc(nf * sizeof(double)); cap_f = nf; }
            render_cell_f64(in, in_is_f32, H, W, C, x0, x1, y0, y1,
                            coeffs + cell_off[cell], L, tile, interm, frag);
            for (int y = 0; y < fh; y++) {
                size_t o = ((size_t)(y0 + y) * W + x0) * C;
                const double *src = frag + (size_t)y * fw * C;
                if (out_kind == 0) {
                    uint8_t *dst = (uint8_t *)out + o;
                    for (int i = 0; i < fw * C; i++) {            /* convolve.py:15 */
                        double v = floor(src[i] + 0.5);
                        v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
                        dst[i] = (uint8_t)v;
                    }
                } else {
                    memcpy((double *)out + o, src, (size_t)fw * C * sizeof(double));
                }
            }
        }
        free(tile); free(interm); free(frag);
    }
    free(spx); free(spy);
    return FO_OK;
}

/* Number of hardware threads OpenMP would use (for the cpu_baseline record). */
int fo_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
