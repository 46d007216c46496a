/*
 * TEST INFRASTRUCTURE — CPU oracle for the MTNN hot path (float64 checkers).
 *
 * Used ONLY by tests/, __graft_entry__.smoke() and bench.py's CPU legs; the
 * product path never loads this library. Built WITHOUT fast-math and with
 * -ffp-contract=off so every operation rounds exactly like the reference's
 * float64 Python/numba arithmetic.
 *
 *  - oracle_nt_f64 / oracle_nn_f64: naive i-j-p loops, operands upcast to
 *    float64 before any arithmetic (reference tests/oracles.py:12-47).
 *  - oracle_nt_f64_rows: the same dot products for a chosen subset of rows and
 *    columns (large-shape spot checks; SURVEY.md §7 "oracle cost at scale").
 *  - oracle_walk_trees(_mnk): packed-tree walk (reference
 *    kernels/_numba_impl.py:197-222, layout selector.py:82-123), float64,
 *    raw = base; raw += eta * leaf — the selector's label oracle.
 */
#include <stdint.h>

int oracle_nt_f64(const float* a, const float* b, double* c, int64_t m, int64_t n,
                  int64_t k) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p) acc += (double)a[i * k + p] * (double)b[j * k + p];
      c[i * n + j] = acc;
    }
  return 0;
}

int oracle_nn_f64(const float* a, const float* b, double* c, int64_t m, int64_t n,
                  int64_t k) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p) acc += (double)a[i * k + p] * (double)b[p * n + j];
      c[i * n + j] = acc;
    }
  return 0;
}

/* out[r * ncols + s] = sum_p A[rows[r], p] * B[cols[s], p] in float64. */
int oracle_nt_f64_rows(const float* a, const float* b, const int64_t* rows, int64_t nrows,
                       const int64_t* cols, int64_t ncols, int64_t k, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < nrows; ++r)
    for (int64_t s = 0; s < ncols; ++s) {
      const float* ar = a + rows[r] * k;
      const float* br = b + cols[s] * k;
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p) acc += (double)ar[p] * (double)br[p];
      out[r * ncols + s] = acc;
    }
  return 0;
}

double oracle_walk_trees(const int64_t* feat, const double* thresh, const int64_t* left,
                         const int64_t* right, const double* leaf, int64_t n_trees,
                         int64_t width, const double* x, double base_score, double eta) {
  double raw = base_score;
  for (int64_t t = 0; t < n_trees; ++t) {
    const int64_t o = t * width;
    int64_t node = 0;
    while (feat[o + node] >= 0)
      node = x[feat[o + node]] < thresh[o + node] ? left[o + node] : right[o + node];
    raw += eta * leaf[o + node];
  }
  return raw;
}

double oracle_walk_trees_mnk(const int64_t* feat, const double* thresh, const int64_t* left,
                             const int64_t* right, const double* leaf, int64_t n_trees,
                             int64_t width, const double* prefix, double m, double n,
                             double k, double base_score, double eta) {
  double x[8];
  for (int i = 0; i < 5; ++i) x[i] = prefix[i];
  x[5] = m;
  x[6] = n;
  x[7] = k;
  return oracle_walk_trees(feat, thresh, left, right, leaf, n_trees, width, x, base_score,
                           eta);
}
