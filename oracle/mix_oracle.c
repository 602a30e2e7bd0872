/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see perm_oracle.c header).
 *
 * Scalar C restatement of the reference's mixing arithmetic, written so the
 * rounding sequence is explicit and independent of which OpenBLAS kernel the
 * host CPU happens to select:
 *
 *  ring mix (reference mixing.py:106-125 `W @ T`, T = ring[p, p] from
 *  simulation.py:299-300): each output column j has exactly three nonzero
 *  weights fl(1/3) at rows {left[j], j, right[j]}.  OpenBLAS dgemm accumulates
 *  the k-loop in ascending k with FMA (zero products add exactly), so
 *      acc = fl(w[a]*t); acc = fma(w[b], t, acc); acc = fma(w[c], t, acc)
 *  with a < b < c the sorted neighbour triple.  Verified bit-identical to
 *  numpy 2.3.5 / OpenBLAS 0.3.30 (Haswell kernel) on this host by
 *  tests/test_oracle.py.
 *
 *  uniform mix (mixing.py:122-124 `W.mean(axis=1)` then tile): numpy's
 *  pairwise summation along the contiguous learner axis
 *  (numpy/_core/src/umath/loops_utils.h.src, DOUBLE_pairwise_sum), then
 *  true_divide by L.
 *
 *  SGD update (simulation.py:267 `apply_mixing(W, T) - lr * G`): numpy rounds
 *  lr*G first, then subtracts: y = mix - fl(lr*g).
 *
 * Layout here is the reference's: W, G, out are (d, L) row-major doubles.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

static double pairwise_sum(const double *a, int64_t n, int64_t stride) {
    if (n < 8) {
        /* numpy: res = 0.; for i: res += a[i]  (starts from -0.0 in newer
         * numpy to keep -0.0 sums; the first add makes it moot except for
         * all -0.0 inputs) */
        double res = -0.0;
        for (int64_t i = 0; i < n; i++) res += a[i * stride];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int k = 0; k < 8; k++) r[k] = a[k * stride];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; k++) r[k] += a[(i + k) * stride];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i * stride];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2, stride) + pairwise_sum(a + n2 * stride, n - n2, stride);
    }
}

double or_pairwise_sum(const double *a, int64_t n) { return pairwise_sum(a, n, 1); }

/* out = ringmix(W) - lr*G ; G may be NULL (pure apply_mixing). */
void or_ring_mix_sgd(const double *W, const double *G, double *out, const int32_t *left,
                     const int32_t *right, int64_t d, int64_t L, double lr) {
    const double t = 1.0 / 3.0;
    for (int64_t j = 0; j < L; j++) {
        int64_t x0 = left[j], x1 = j, x2 = right[j], tmp;
        if (x1 < x0) { tmp = x0; x0 = x1; x1 = tmp; }
        if (x2 < x1) { tmp = x1; x1 = x2; x2 = tmp; }
        if (x1 < x0) { tmp = x0; x0 = x1; x1 = tmp; }
        for (int64_t r = 0; r < d; r++) {
            const double *w = W + r * L;
            double acc = w[x0] * t;
            acc = fma(w[x1], t, acc);
            acc = fma(w[x2], t, acc);
            if (G) {
                volatile double s = lr * G[r * L + j];
                acc = acc - s;
            }
            out[r * L + j] = acc;
        }
    }
}

/* out = tile(mean_l W) - lr*G ; G may be NULL. */
void or_mean_sgd(const double *W, const double *G, double *out, int64_t d, int64_t L, double lr) {
    for (int64_t r = 0; r < d; r++) {
        double m = pairwise_sum(W + r * L, L, 1) / (double)L;
        for (int64_t j = 0; j < L; j++) {
            double y = m;
            if (G) {
                volatile double s = lr * G[r * L + j];
                y = m - s;
            }
            out[r * L + j] = y;
        }
    }
}
