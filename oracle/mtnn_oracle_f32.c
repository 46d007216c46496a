/*
 * TEST INFRASTRUCTURE — CPU oracle for the MTNN hot path (float32 kernels).
 *
 * Plain-C restatement of the reference's compiled kernels
 * (/root/reference/pkg/src/mtnn/kernels/_numba_impl.py), used ONLY by tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm. The
 * product path (paper_1702_03192_b200) never loads this library.
 *
 * Each function follows the reference loop structure and arithmetic type
 * (float32 accumulation). The reference compiles these loops with
 * numba fastmath=True (reassociation allowed), so this file is built with
 * -ffast-math as well; results match the reference within reassociation,
 * not bit-for-bit (pinned by tests/test_oracle.py against tests/golden/).
 * The transpose is a pure copy and is bit-exact.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* _nn_panel (_numba_impl.py:31-100): one (j, p) panel of the blocked product
 * over rows [i_lo, i_hi): pack the B panel k-major, emit two C rows per pass,
 * 4-deep k unroll. c must be zero-initialised by the caller. */
static void nn_panel(const float* a, const float* b, float* c, int64_t k, int64_t n,
                     int64_t j0, int64_t j1, int64_t p0, int64_t p1, int64_t i_lo,
                     int64_t i_hi, float* pack_b, float* row0, float* row1,
                     int64_t block) {
  const int64_t nj = j1 - j0, npp = p1 - p0;
  for (int64_t pp = 0; pp < npp; ++pp)
    for (int64_t jj = 0; jj < nj; ++jj) pack_b[pp * block + jj] = b[(p0 + pp) * n + j0 + jj];
  int64_t i = i_lo;
  for (; i + 2 <= i_hi; i += 2) {
    const float* ar0 = a + i * k + p0;
    const float* ar1 = a + (i + 1) * k + p0;
    for (int64_t jj = 0; jj < nj; ++jj) row0[jj] = row1[jj] = 0.0f;
    int64_t pp = 0;
    for (; pp + 4 <= npp; pp += 4) {
      const float a00 = ar0[pp], a01 = ar0[pp + 1], a02 = ar0[pp + 2], a03 = ar0[pp + 3];
      const float a10 = ar1[pp], a11 = ar1[pp + 1], a12 = ar1[pp + 2], a13 = ar1[pp + 3];
      const float* q0 = pack_b + pp * block;
      const float* q1 = q0 + block;
      const float* q2 = q1 + block;
      const float* q3 = q2 + block;
      for (int64_t jj = 0; jj < nj; ++jj) {
        row0[jj] += a00 * q0[jj] + a01 * q1[jj] + a02 * q2[jj] + a03 * q3[jj];
        row1[jj] += a10 * q0[jj] + a11 * q1[jj] + a12 * q2[jj] + a13 * q3[jj];
      }
    }
    for (; pp < npp; ++pp) {
      const float a0 = ar0[pp], a1 = ar1[pp];
      const float* q = pack_b + pp * block;
      for (int64_t jj = 0; jj < nj; ++jj) {
        row0[jj] += a0 * q[jj];
        row1[jj] += a1 * q[jj];
      }
    }
    float* c0 = c + i * n + j0;
    float* c1 = c + (i + 1) * n + j0;
    for (int64_t jj = 0; jj < nj; ++jj) {
      c0[jj] += row0[jj];
      c1[jj] += row1[jj];
    }
  }
  for (; i < i_hi; ++i) {
    const float* ar0 = a + i * k + p0;
    for (int64_t jj = 0; jj < nj; ++jj) row0[jj] = 0.0f;
    int64_t pp = 0;
    for (; pp + 4 <= npp; pp += 4) {
      const float a00 = ar0[pp], a01 = ar0[pp + 1], a02 = ar0[pp + 2], a03 = ar0[pp + 3];
      const float* q0 = pack_b + pp * block;
      for (int64_t jj = 0; jj < nj; ++jj)
        row0[jj] += a00 * q0[jj] + a01 * q0[block + jj] + a02 * q0[2 * block + jj] +
                    a03 * q0[3 * block + jj];
    }
    for (; pp < npp; ++pp) {
      const float a0 = ar0[pp];
      const float* q = pack_b + pp * block;
      for (int64_t jj = 0; jj < nj; ++jj) row0[jj] += a0 * q[jj];
    }
    float* c0 = c + i * n + j0;
    for (int64_t jj = 0; jj < nj; ++jj) c0[jj] += row0[jj];
  }
}

/* gemm_nn / gemm_nn_parallel (_numba_impl.py:103-136): C = A x B, B k x n.
 * threads > 1 parallelises over disjoint column panels like the prange. */
int oracle_gemm_nn(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                   int64_t block, int threads) {
  if (block < 4) return 22;
  memset(c, 0, sizeof(float) * (size_t)(m * n));
  const int64_t n_panels = (n + block - 1) / block;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : 1)
#endif
  for (int64_t panel = 0; panel < n_panels; ++panel) {
    float* pack_b = (float*)malloc(sizeof(float) * (size_t)(block * block));
    float* row0 = (float*)malloc(sizeof(float) * (size_t)block);
    float* row1 = (float*)malloc(sizeof(float) * (size_t)block);
    const int64_t j0 = panel * block;
    const int64_t j1 = j0 + block < n ? j0 + block : n;
    for (int64_t p0 = 0; p0 < k; p0 += block) {
      const int64_t p1 = p0 + block < k ? p0 + block : k;
      nn_panel(a, b, c, k, n, j0, j1, p0, p1, 0, m, pack_b, row0, row1, block);
    }
    free(pack_b);
    free(row0);
    free(row1);
  }
  (void)threads;
  return 0;
}

/* gemm_nt / gemm_nt_parallel (_numba_impl.py:139-166): one float32 dot
 * product per output over the contiguous rows of a and b; rows in parallel. */
int oracle_gemm_nt(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                   int threads) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
#endif
  for (int64_t i = 0; i < m; ++i) {
    const float* ar = a + i * k;
    for (int64_t j = 0; j < n; ++j) {
      const float* br = b + j * k;
      float acc = 0.0f;
      for (int64_t p = 0; p < k; ++p) acc += ar[p] * br[p];
      c[i * n + j] = acc;
    }
  }
  (void)threads;
  return 0;
}

/* transpose_oop (_numba_impl.py:169-182): square tiles, contiguous output
 * runs; a pure 32-bit copy (moved as uint32 so NaN payloads survive). */
int oracle_transpose(const float* bf, float* outf, int64_t n, int64_t k, int64_t tile,
                     int threads) {
  if (tile < 1) return 22;
  const uint32_t* b = (const uint32_t*)bf;
  uint32_t* out = (uint32_t*)outf;
  const int64_t tiles_j = (k + tile - 1) / tile;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
#endif
  for (int64_t tj = 0; tj < tiles_j; ++tj) {
    const int64_t j0 = tj * tile, j1 = j0 + tile < k ? j0 + tile : k;
    for (int64_t i0 = 0; i0 < n; i0 += tile) {
      const int64_t i1 = i0 + tile < n ? i0 + tile : n;
      for (int64_t j = j0; j < j1; ++j)
        for (int64_t i = i0; i < i1; ++i) out[j * n + i] = b[i * k + j];
    }
  }
  (void)threads;
  return 0;
}

/* gemm_tnn / gemm_tnn_parallel (_numba_impl.py:185-194): allocate B^T,
 * transpose, NN, release — all inside the call. */
int oracle_gemm_tnn(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                    int64_t block, int64_t tile, int threads) {
  float* bt = (float*)malloc(sizeof(float) * (size_t)(n * k > 0 ? n * k : 1));
  if (!bt) return 12;
  int rc = oracle_transpose(b, bt, n, k, tile, 1);
  if (rc == 0) rc = oracle_gemm_nn(a, bt, c, m, n, k, block, threads);
  free(bt);
  return rc;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
