/*
 * Plain-C restatement of the reference's compiled incremental-update kernels.
 * TEST INFRASTRUCTURE ONLY (oracle): used by oracle/cgh_oracle.py to evaluate
 * SA/DBS proposals at reference speed and with the reference's arithmetic.
 *
 * Follows /root/reference/pkg/src/cghkit/kernels/_core.pyx:
 *   oracle_delta_error  <- delta_error   (_core.pyx:20-34)
 *   oracle_commit       <- commit_update (_core.pyx:37-44)
 *   oracle_best_delta   <- best_delta    (_core.pyx:47-83)
 * The reference compiles with -O3 -fcx-limited-range (pkg/setup.py:17), i.e.
 * complex products are the plain (ac-bd, ad+bc) form, and |z| is
 * sqrt(re*re + im*im) (_core.pyx:17-18). Complex arrays are interleaved
 * (re, im) doubles, exactly numpy's complex128 layout.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct { double re, im; } zc;

static inline zc zmul(zc a, zc b) {
    zc r;
    r.re = a.re * b.re - a.im * b.im;
    r.im = a.re * b.im + a.im * b.re;
    return r;
}

static inline double zabs(zc z) { return sqrt(z.re * z.re + z.im * z.im); }

/* Masked error-sum change of one pixel update (no commit). */
double oracle_delta_error(const zc *replay_m, const double *target_m,
                          const zc *row_tw, const zc *col_tw,
                          const int32_t *mu, const int32_t *mv, int64_t count,
                          double delta_re, double delta_im) {
    zc delta = {delta_re, delta_im};
    double total = 0.0;
    for (int64_t i = 0; i < count; ++i) {
        zc w = zmul(row_tw[mu[i]], col_tw[mv[i]]);
        zc dw = zmul(delta, w);
        zc upd = {replay_m[i].re + dw.re, replay_m[i].im + dw.im};
        double d0 = zabs(replay_m[i]) - target_m[i];
        double d1 = zabs(upd) - target_m[i];
        total += d1 * d1 - d0 * d0;
    }
    return total;
}

/* replay_m += delta * row_tw[mu] * col_tw[mv], in place. */
void oracle_commit(zc *replay_m, const zc *row_tw, const zc *col_tw,
                   const int32_t *mu, const int32_t *mv, int64_t count,
                   double delta_re, double delta_im) {
    zc delta = {delta_re, delta_im};
    for (int64_t i = 0; i < count; ++i) {
        zc dw = zmul(delta, zmul(row_tw[mu[i]], col_tw[mv[i]]));
        replay_m[i].re = replay_m[i].re + dw.re;
        replay_m[i].im = replay_m[i].im + dw.im;
    }
}

/* Best candidate level: zero deltas skipped, strict '<' from 0.0, lowest index
 * wins ties; returns -1 (and *best_change = 0.0) when nothing improves.
 * Returns -2 on allocation failure. */
int64_t oracle_best_delta(const zc *replay_m, const double *target_m,
                          const zc *row_tw, const zc *col_tw,
                          const int32_t *mu, const int32_t *mv, int64_t count,
                          const zc *deltas, int64_t levels, double *best_change) {
    zc *w = (zc *)malloc((size_t)(count > 0 ? count : 1) * sizeof(zc));
    double *base = (double *)malloc((size_t)(count > 0 ? count : 1) * sizeof(double));
    int64_t best = -1;
    double best_val = 0.0;
    if (!w || !base) {
        free(w);
        free(base);
        return -2;
    }
    for (int64_t i = 0; i < count; ++i) {
        w[i] = zmul(row_tw[mu[i]], col_tw[mv[i]]);
        double d = zabs(replay_m[i]) - target_m[i];
        base[i] = d * d;
    }
    for (int64_t j = 0; j < levels; ++j) {
        zc delta = deltas[j];
        if (delta.re == 0.0 && delta.im == 0.0) continue;
        double change = 0.0;
        for (int64_t i = 0; i < count; ++i) {
            zc dw = zmul(delta, w[i]);
            zc upd = {replay_m[i].re + dw.re, replay_m[i].im + dw.im};
            double d1 = zabs(upd) - target_m[i];
            change += d1 * d1 - base[i];
        }
        if (change < best_val) {
            best_val = change;
            best = j;
        }
    }
    free(w);
    free(base);
    *best_change = best_val;
    return best;
}
