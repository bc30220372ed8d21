/*
 * fk_hypot.h -- bit-exact replica of glibc >= 2.35 hypot() on x86-64 (the routine behind
 * numpy's np.hypot, which the reference calls at retinal.py:110).
 *
 * glibc's hypot is not correctly rounded; its result is defined by the operation sequence
 * below (the non-FMA "kernel" of sysdeps/ieee754/dbl-64/e_hypot.c as built for baseline
 * x86-64, after C. Borges, "An improved algorithm for hypot(a,b)").  Every operation is a
 * separately rounded IEEE fp64 operation; on the device we spell them with the
 * round-to-nearest intrinsics so the compiler can never contract them into FMAs.
 *
 * Included by the plan kernel (device) and by tests/c/test_hypot.c (host, gcc
 * -ffp-contract=off) which compares it with libm over millions of lattice points.
 */
#ifndef FK_HYPOT_H_
#define FK_HYPOT_H_

#ifdef __CUDA_ARCH__
#define FK_HD __host__ __device__ __forceinline__
#define FK_MUL(a, b) __dmul_rn((a), (b))
#define FK_ADD(a, b) __dadd_rn((a), (b))
#define FK_SUB(a, b) __dsub_rn((a), (b))
#define FK_DIV(a, b) __ddiv_rn((a), (b))
#define FK_SQRT(a) __dsqrt_rn((a))
#else
#include <math.h>
#ifdef __CUDACC__
#define FK_HD __host__ __device__ inline
#else
#define FK_HD static inline
#endif
#define FK_MUL(a, b) ((a) * (b))
#define FK_ADD(a, b) ((a) + (b))
#define FK_SUB(a, b) ((a) - (b))
#define FK_DIV(a, b) ((a) / (b))
#define FK_SQRT(a) sqrt((a))
#endif

/* Inputs: ax >= ay >= 0, no overflow/underflow when squared. */
FK_HD double fk_hypot_kernel(double ax, double ay)
{
    double h = FK_SQRT(FK_ADD(FK_MUL(ax, ax), FK_MUL(ay, ay)));
    double t1, t2;
    if (h <= FK_MUL(2.0, ay)) {
        double delta = FK_SUB(h, ay);
        t1 = FK_MUL(ax, FK_SUB(FK_MUL(2.0, delta), ax));
        t2 = FK_MUL(FK_SUB(delta, FK_MUL(2.0, FK_SUB(ax, ay))), delta);
    } else {
        double delta = FK_SUB(h, ax);
        t1 = FK_MUL(FK_MUL(2.0, delta), FK_SUB(ax, FK_MUL(2.0, ay)));
        t2 = FK_ADD(FK_MUL(FK_SUB(FK_MUL(4.0, delta), ay), ay), FK_MUL(delta, delta));
    }
    h = FK_SUB(h, FK_DIV(FK_ADD(t1, t2), FK_MUL(2.0, h)));
    return h;
}

/* Finite inputs only (pixel coordinates).  Huge/tiny rescaling branches of glibc are
 * reproduced for completeness although pixel distances never reach them. */
FK_HD double fk_hypot(double x, double y)
{
    const double SCALE = 0x1p-600, LARGE_VAL = 0x1p+511, TINY_VAL = 0x1p-459,
                 EPS = 0x1p-54;
    x = x < 0.0 ? -x : x;
    y = y < 0.0 ? -y : y;
    double ax = x < y ? y : x;
    double ay = x < y ? x : y;
    if (ax > LARGE_VAL) {
        if (ay <= FK_MUL(ax, EPS)) return FK_ADD(ax, ay);
        return FK_DIV(fk_hypot_kernel(FK_MUL(ax, SCALE), FK_MUL(ay, SCALE)), SCALE);
    }
    if (ay < TINY_VAL) {
        if (ax >= FK_DIV(ay, EPS)) return FK_ADD(ax, ay);
        ax = fk_hypot_kernel(FK_DIV(ax, SCALE), FK_DIV(ay, SCALE));
        return FK_MUL(ax, SCALE);
    }
    if (ax >= FK_DIV(ay, EPS)) return FK_ADD(ax, ay);
    return fk_hypot_kernel(ax, ay);
}

#endif /* FK_HYPOT_H_ */
