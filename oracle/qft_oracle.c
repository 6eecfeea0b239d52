/*
 * oracle/qft_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C, scalar restatement of the reference quickfourier package's
 * transform recursions (improved and classical QFT) and of its two-tier
 * trigonometric-constant recipe.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library; the
 * product path (paper_1301_0763_b200) never links or calls it.
 *
 * Every function follows one reference function operation for operation:
 * same operands, same operand order for subtractions, one IEEE rounding per
 * add/sub/mul, no FMA contraction (built with -ffp-contract=off), no
 * reassociation.  The result is therefore bit-identical to the reference's
 * numpy evaluation (pinned by tests/test_oracle.py against the golden
 * vectors in tests/golden/, which were produced by the reference itself).
 *
 * Buffer convention: one signal per contiguous vector; complex signals are
 * interleaved (Re at 2n, Im at 2n+1), i.e. the memory order of complex64 /
 * complex128.  Batched entry points take batch-major arrays.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* counting.py:18 -- pi to more digits than an 80-bit long double holds */
static const long double WIDE_PI =
    3.14159265358979323846264338327950288419716939937510L;

/* ------------------------------------------------------------------ */
/* constants: counting.py:116-140 (TrigTable._wide_cos_of_turns,       */
/* _working_cos_of_turns, _value_for)                                   */
/* ------------------------------------------------------------------ */

/* two-tier, float64 working dtype: cos in x87 long double, 1/(2c) in long
 * double, rounded once to double (counting.py:120-121, 135-137) */
static double halfsec_two_tier_f64(long j, long d) {
    long double t = (long double)j / (long double)d;
    long double c = cosl(2.0L * WIDE_PI * t);
    return (double)(1.0L / (2.0L * c));
}
static double cos8_two_tier_f64(void) {
    long double t = 1.0L / 8.0L;
    return (double)cosl(2.0L * WIDE_PI * t); /* counting.py:130-132 */
}
/* two-tier, float32 working dtype: everything in double, rounded once to
 * float (counting.py:118-119, 135-137) */
static float halfsec_two_tier_f32(long j, long d) {
    double c = cos(2.0 * M_PI * ((double)j / (double)d));
    return (float)(1.0 / (2.0 * c));
}
static float cos8_two_tier_f32(void) {
    return (float)cos(2.0 * M_PI * (1.0 / 8.0));
}
/* single-tier, float64: every step in double (counting.py:123-127, 138-140) */
static double halfsec_single_tier_f64(long j, long d) {
    double ang = 2.0 * M_PI * ((double)j / (double)d);
    double c = cos(ang);
    return 1.0 / (2.0 * c);
}
static double cos8_single_tier_f64(void) {
    return cos(2.0 * M_PI * (1.0 / 8.0));
}

/* Natural table for periodization N: T[0] = cos(2pi/8) (the named entry),
 * T[m] = 1/(2 cos(2 pi m/N)) for m = 1..N/4-1.  Every value depends only on
 * the reduced fraction m/N (counting.py:152-158), and for power-of-two N the
 * quotient m/N is exact in every tier, so T[m * N/N'] is the constant the
 * reference uses at recursion level N'. */
int oracle_table_f64(int N, int pipeline, double *out) {
    if (N < 8 || (N & (N - 1))) return -1;
    out[0] = pipeline == 0 ? cos8_two_tier_f64() : cos8_single_tier_f64();
    for (int m = 1; m < N / 4; ++m)
        out[m] = pipeline == 0 ? halfsec_two_tier_f64(m, N)
                               : halfsec_single_tier_f64(m, N);
    return 0;
}
int oracle_table_f32(int N, float *out) {
    if (N < 8 || (N & (N - 1))) return -1;
    out[0] = cos8_two_tier_f32();
    for (int m = 1; m < N / 4; ++m) out[m] = halfsec_two_tier_f32(m, N);
    return 0;
}

/* ------------------------------------------------------------------ */
/* bump arena for the recursion temporaries (counting.py:60-67 rows_like) */
/* ------------------------------------------------------------------ */
typedef struct {
    char *base;
    size_t used, cap;
} arena_t;

static void *arena_alloc(arena_t *a, size_t bytes) {
    bytes = (bytes + 15) & ~(size_t)15;
    if (a->used + bytes > a->cap) abort();
    void *p = a->base + a->used;
    a->used += bytes;
    return p;
}

#define QFT_REAL double
#define QFT_SUF f64
#include "qft_oracle_impl.h"
#undef QFT_REAL
#undef QFT_SUF

#define QFT_REAL float
#define QFT_SUF f32
#include "qft_oracle_impl.h"
#undef QFT_REAL
#undef QFT_SUF

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
