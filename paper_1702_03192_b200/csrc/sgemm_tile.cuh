// One 128 x 128 output tile of the exact-order FFMA GEMM (gemm_ffma.cu), shared
// by the SIMT GEMM kernel and the residual fix-up's recompute path (fixup.cu).
//
// 256 threads, 8 x 8 register micro-tile (two 4-wide halves 64 apart so LDS.128
// reads are conflict-free), register-staged double buffer of the next 8-deep
// k-slice. Each output is one FFMA chain over k ascending in [kbeg, kend), so
// identity products stay bit-exact (test_kernels.py:32-40, 87-89).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace mtnn {
namespace sgemm {

constexpr int BM = 128, BN = 128, BK = 8;

// A: m x k (row stride k). B_NK: B n x k (row stride k); else B^T k x n (row stride ldb).
template <bool B_NK>
__device__ __forceinline__ void tile(const float* __restrict__ A, const float* __restrict__ B,
                                     int64_t ldb, int64_t m, int64_t n, int64_t k, int64_t bm0,
                                     int64_t bn0, int64_t kbeg, int64_t kend,
                                     float (&As)[2][BK][BM], float (&Bs)[2][BK][BN],
                                     float (&acc)[8][8]) {
  const int tid = threadIdx.x;
  const int a_row = tid >> 1, a_k = (tid & 1) * 4;   // A: 128 rows x 8 k
  const int bt_k = tid >> 5, bt_c = (tid & 31) * 4;  // B^T: 8 k x 128 cols

  float ra[4], rb[4];
  auto load_tile = [&](int64_t k0) {
    {
      const int64_t r = bm0 + a_row;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t kk = k0 + a_k + j;
        ra[j] = (r < m && kk < kend) ? __ldg(A + r * k + kk) : 0.f;
      }
    }
    if (B_NK) {
      const int64_t r = bn0 + a_row;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t kk = k0 + a_k + j;
        rb[j] = (r < n && kk < kend) ? __ldg(B + r * k + kk) : 0.f;
      }
    } else {
      const int64_t kk = k0 + bt_k;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t c = bn0 + bt_c + j;
        rb[j] = (kk < kend && c < n) ? __ldg(B + kk * ldb + c) : 0.f;
      }
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 4; ++j) As[buf][a_k + j][a_row] = ra[j];
    if (B_NK) {
#pragma unroll
      for (int j = 0; j < 4; ++j) Bs[buf][a_k + j][a_row] = rb[j];
    } else {
      *reinterpret_cast<float4*>(&Bs[buf][bt_k][bt_c]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
    }
  };

  const int tx = tid & 15, ty = tid >> 4;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  int buf = 0;
  if (kbeg < kend) {
    load_tile(kbeg);
    store_tile(0);
  }
  __syncthreads();
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    const bool has_next = k0 + BK < kend;
    if (has_next) load_tile(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[8], b[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (has_next) {
      store_tile(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
}

// Writes the tile (rows of `ldc` elements).
__device__ __forceinline__ void store(const float (&acc)[8][8], float* out, int64_t ldc, int64_t m,
                                      int64_t n, int64_t bm0, int64_t bn0) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = bm0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (r >= m) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t c = bn0 + h * 64 + tx * 4;
      float* dst = out + r * ldc + c;
      if (c + 3 < n && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        *reinterpret_cast<float4*>(dst) = make_float4(acc[i][h * 4 + 0], acc[i][h * 4 + 1],
                                                      acc[i][h * 4 + 2], acc[i][h * 4 + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c + j < n) dst[j] = acc[i][h * 4 + j];
      }
    }
  }
}

// store(), or (accumulate) add the tile to what `out` holds. Each output is
// read and written by the one thread that owns it.
__device__ __forceinline__ void store_acc(const float (&acc)[8][8], float* out, int64_t ldc,
                                          int64_t m, int64_t n, int64_t bm0, int64_t bn0,
                                          bool accumulate) {
  if (!accumulate) {
    store(acc, out, ldc, m, n, bm0, bn0);
    return;
  }
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = bm0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (r >= m) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t c = bn0 + h * 64 + tx * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (c + j < n) out[r * ldc + c + j] += acc[i][h * 4 + j];
    }
  }
}

}  // namespace sgemm
}  // namespace mtnn
