/*
 * ORACLE — test infrastructure only (never linked into the product path).
 *
 * Plain-C restatement of the reference's complete-pivoting partial LU with
 * rank cut: /root/reference/pkg/src/mfhodlr/_kernels/_core.pyx:23-86
 * (pure twin: _kernels/_pure.py:26-89).
 *
 * Semantics restated:
 *   - pivot search over the trailing block in row-major order, strict '>'
 *     so the first maximum wins                       (_core.pyx:39-48)
 *   - k == 0: u11 = pivot, zero block -> rank 0       (_core.pyx:49-52)
 *   - k > 0: growth guard pivot > prev*2(1+1e-10) raises
 *     PivotMonotonicityError; rank cut when pivot/u11 < eps or
 *     pivot <= 1e-14*u11                              (_core.pyx:53-60)
 *   - k == kmax (= min(m, n, max_rank)) stops with ratio pivot/u11 (61-62)
 *   - physical row/column swaps of whole rows/cols, then the multipliers
 *     a[i,k] /= a[k,k] and a[i,j] -= v*a[k,j]           (_core.pyx:63-85)
 *
 * Compiled with -ffp-contract=off so the update is a separate multiply and
 * subtract, exactly like the Cython build (gcc -O3 on x86-64 does not
 * contract by default without -march flags either).
 *
 * Return: 0 ok; 1 pivot-monotonicity error (err_k, err_piv, err_prev set).
 */
#include <math.h>
#include <stdint.h>

#define ZERO_PIVOT_RATIO 1e-14
#define PIVOT_GROWTH_BOUND (2.0 * (1.0 + 1e-10))

int oracle_full_pivot_lu(double *a, int64_t m, int64_t n, double eps,
                         int64_t max_rank, int64_t *row_perm, int64_t *col_perm,
                         int64_t *rank_out, double *ratio_out, int64_t *err_k,
                         double *err_piv, double *err_prev) {
  int64_t kmin = m < n ? m : n;
  int64_t kmax = kmin < max_rank ? kmin : max_rank;
  double u11 = 0.0, prev = 0.0;
  for (int64_t i = 0; i < m; ++i) row_perm[i] = i;
  for (int64_t j = 0; j < n; ++j) col_perm[j] = j;
  *rank_out = 0;
  *ratio_out = 0.0;
  for (int64_t k = 0; k < kmin; ++k) {
    double piv = -1.0;
    int64_t bi = k, bj = k;
    for (int64_t i = k; i < m; ++i) {
      const double *row = a + i * n;
      for (int64_t j = k; j < n; ++j) {
        double v = fabs(row[j]);
        if (v > piv) {
          piv = v;
          bi = i;
          bj = j;
        }
      }
    }
    if (k == 0) {
      u11 = piv;
      if (u11 == 0.0) {
        *rank_out = 0;
        *ratio_out = 0.0;
        return 0;
      }
    } else {
      if (piv > prev * PIVOT_GROWTH_BOUND) {
        *err_k = k;
        *err_piv = piv;
        *err_prev = prev;
        return 1;
      }
      double next_ratio = piv / u11;
      if (next_ratio < eps || piv <= ZERO_PIVOT_RATIO * u11) {
        *rank_out = k;
        *ratio_out = next_ratio;
        return 0;
      }
    }
    if (k == kmax) {
      *rank_out = kmax;
      *ratio_out = piv / u11;
      return 0;
    }
    if (bi != k) {
      double *rk = a + k * n, *rb = a + bi * n;
      for (int64_t t = 0; t < n; ++t) {
        double tmp = rk[t];
        rk[t] = rb[t];
        rb[t] = tmp;
      }
      int64_t it = row_perm[k];
      row_perm[k] = row_perm[bi];
      row_perm[bi] = it;
    }
    if (bj != k) {
      for (int64_t t = 0; t < m; ++t) {
        double tmp = a[t * n + k];
        a[t * n + k] = a[t * n + bj];
        a[t * n + bj] = tmp;
      }
      int64_t it = col_perm[k];
      col_perm[k] = col_perm[bj];
      col_perm[bj] = it;
    }
    prev = fabs(a[k * n + k]);
    const double akk = a[k * n + k];
    const double *rowk = a + k * n;
    for (int64_t i = k + 1; i < m; ++i) {
      double *ri = a + i * n;
      ri[k] /= akk;
      double v = ri[k];
      for (int64_t j = k + 1; j < n; ++j) {
        double p = v * rowk[j];
        ri[j] = ri[j] - p;
      }
    }
    *rank_out = k + 1;
  }
  *ratio_out = 0.0;
  return 0;
}
