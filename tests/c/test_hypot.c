/* Host check of fk_hypot.h against libm hypot (the routine np.hypot resolves to).
 * Build: gcc -O2 -ffp-contract=off -I paper_2012_08655_b200/csrc tests/c/test_hypot.c -lm
 * Prints the number of mismatching bit patterns; exit status 0 iff none. */
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <math.h>
#include "fk_hypot.h"

static uint64_t s = 0x9E3779B97F4A7C15ull;
static uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
static double urand(void) { return (double)(rnd() >> 11) * 0x1p-53; }

static int differs(double a, double b) { return memcmp(&a, &b, 8) != 0; }

int main(void)
{
    long bad = 0, n = 0;
    /* lattice of half-integer midpoints against integer and fractional fixations */
    for (int i = 0; i < 4000000; i++) {
        double mx = 0.5 * (double)(rnd() % 7681), my = 0.5 * (double)(rnd() % 4321);
        double fx = (i & 1) ? (double)(rnd() % 3840) : urand() * 3840.0;
        double fy = (i & 2) ? (double)(rnd() % 2160) : urand() * 2160.0;
        double a = hypot(mx - fx, my - fy), b = fk_hypot(mx - fx, my - fy);
        bad += differs(a, b); n++;
    }
    /* exact zeros, axis-aligned and near-degenerate pairs */
    double sp[] = {0.0, 0.5, 1.0, 1e-13, 1.4e-14, 3.0, 4.0, 1e-300, 1e300, 2203.5, 5e-324};
    for (unsigned i = 0; i < sizeof sp / sizeof *sp; i++)
        for (unsigned j = 0; j < sizeof sp / sizeof *sp; j++) {
            double a = hypot(sp[i], -sp[j]), b = fk_hypot(sp[i], -sp[j]);
            bad += differs(a, b); n++;
        }
    /* wide dynamic range */
    for (int i = 0; i < 2000000; i++) {
        double x = ldexp(urand() + 0.5, (int)(rnd() % 120) - 60);
        double y = ldexp(urand() + 0.5, (int)(rnd() % 120) - 60);
        double a = hypot(x, y), b = fk_hypot(x, y);
        bad += differs(a, b); n++;
    }
    printf("%ld mismatches of %ld\n", bad, n);
    return bad != 0;
}
