/*
 * oracle/attend.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this code.  The product path (paper_2509_02121_b200/) never does, and shares
 * no code, header, table or helper with it.
 *
 * What it computes: UNSHARED softmax attention of one decode query per (request, q-head)
 * over the request's FULL context, in fp64.  The paper requires every optimisation to be
 * semantics-preserving -- "the final answers produced by an optimized execution are
 * identical to those from a naive execution" (§2.2 Scope, "Exact answers")
 * -- and presents prefix caching as pure reuse of precomputed state (§3.3
 * "Prefix caching").  So the oracle is the naive, unshared definition:
 *
 *   for q-head h:   j   = floor(h / g)                 (GQA group, reading R3)
 *                   s_t = scale * sum_i q[h][i] * k[t][j][i]           t = 0..T-1
 *                   m   = max_t s_t
 *                   Z   = sum_t exp(s_t - m)
 *                   o_h = (sum_t exp(s_t - m) * v[t][j]) / Z
 *                   lse = m + ln Z                       (natural log, reading R9)
 *
 * Inputs are bf16 bit patterns, widened exactly to double.  No blocking, no splitting, no
 * merging, no reordering: one straight pass per head.  Empty context (T == 0) returns the
 * identity of the log-sum-exp merge: o = 0, lse = -inf (reading R6).
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC (no -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double widen_bf16(uint16_t b)
{
    uint32_t u = (uint32_t)b << 16; /* bf16 is the upper half of an IEEE binary32 */
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

/* One (request): q [hq][d], k/v [T][hkv][d] (bf16 bits), out [hq][d], lse [hq] (fp64).
 * Returns 0, or -1 on invalid shapes. */
int oracle_attend(int64_t T, int hq, int hkv, int d,
                  const uint16_t *q, const uint16_t *k, const uint16_t *v,
                  double scale, double *out, double *lse, int nthreads)
{
    if (T < 0 || hq <= 0 || hkv <= 0 || d <= 0 || hq % hkv != 0)
        return -1;
    const int g = hq / hkv;
    if (T == 0) {
        for (int h = 0; h < hq; ++h) {
            lse[h] = -INFINITY;
            for (int i = 0; i < d; ++i)
                out[(int64_t)h * d + i] = 0.0;
        }
        return 0;
    }
    if (nthreads <= 0)
        nthreads = 1;
    int err = 0;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int h = 0; h < hq; ++h) {
        const int j = h / g;
        double *s = (double *)malloc((size_t)T * sizeof(double));
        if (!s) {
            err = -1;
            continue;
        }
        /* step 4: scores */
        double m = -INFINITY;
        for (int64_t t = 0; t < T; ++t) {
            double acc = 0.0;
            const uint16_t *kt = k + (t * hkv + j) * d;
            const uint16_t *qh = q + (int64_t)h * d;
            for (int i = 0; i < d; ++i)
                acc += widen_bf16(qh[i]) * widen_bf16(kt[i]);
            s[t] = scale * acc;
            if (s[t] > m)
                m = s[t];
        }
        /* step 5: softmax weights, normaliser, weighted sum of values */
        double Z = 0.0;
        for (int64_t t = 0; t < T; ++t) {
            s[t] = exp(s[t] - m);
            Z += s[t];
        }
        for (int i = 0; i < d; ++i) {
            double acc = 0.0;
            for (int64_t t = 0; t < T; ++t)
                acc += s[t] * widen_bf16(v[(t * hkv + j) * d + i]);
            out[(int64_t)h * d + i] = acc / Z;
        }
        lse[h] = m + log(Z);
        free(s);
    }
    return err;
}
