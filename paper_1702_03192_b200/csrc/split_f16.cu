// Operand split for the FP16x3-scaled tensor-core GEMM (variant tc3xf16s).
//
// Each FP32 operand row (a row of A, a row of B for NT, a column of B^T for NN)
// gets an exact power-of-two scale s = 2^(14 - ceil(log2(max|x|))) that puts its
// largest magnitude in [2^13, 2^14] — inside FP16 range with headroom — and every
// element is written as two FP16 halves:
//     h = fp16_rn(x * s),   l = fp16_rn(x * s - h)        (x*s - h is exact in fp32)
// so x*s = h + l + r with |r| <= 2^-24 |x*s|. The GEMM accumulates h*h + h*l + l*h
// (the dropped l*l is ~2^-24 relative) in FP32 and multiplies each output by
// 1/(s_row * s_col), which is exact. FP16 carries the same 11-bit significand as
// TF32 but runs at twice the tensor-core rate, and the per-row scale removes its
// range limit (subnormal tails sit ~2^-38 below the row maximum).
//
// MN-major operands (B^T of NN, k x n) get one scale per (256-row chunk,
// column) instead of one per column: the GEMM's epilogue applies it to each
// FP32-promotion chunk (gemm_tc.cu), which makes the column split a single
// local pass.
//
// Traffic: the row splits (K-major operands) read each element from DRAM once
// and write its halves once — 4 B + 4 B; the column split does the same.
//
// Kernels by shape: rows — register warp (k <= 512, 1024 < k <= 2048), looped
// warp (k = 1024), register CTA (2048 < k <= 16384), smem CTA (longer rows);
// columns — one CTA per (256-row chunk, 32 columns).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "common.h"
#include "fix.h"
#include "pdl.h"

namespace mtnn {
namespace {

// 2^(14 - ceil(log2(mx))) for finite mx > 0; 1 for 0; 1 for non-finite (the
// Inf/NaN then propagates through the FP16 halves as it would in FP32). The
// exponent is capped at 2^126 so rows whose max is below 2^-112 keep a finite
// scale (and 1/s stays a normal float); their halves then lose low bits.
__device__ __forceinline__ float pow2_scale(float mx) {
  if (!(mx > 0.f) || !isfinite(mx)) return 1.f;
  int e;
  const float f = frexpf(mx, &e);  // mx = f * 2^e, f in [0.5, 1)
  const int c = (f == 0.5f) ? e - 1 : e;  // ceil(log2(mx))
  return ldexpf(1.f, min(14 - c, 126));
}

// Lets the GEMM launched next on the stream (programmatic stream serialization)
// start its prologue while this grid finishes; it waits for our completion
// before reading any output (gemm_tc.cu pdl_wait).
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// The split kernels are themselves launched with programmatic serialization
// (launch_chained), so they can be scheduled while the previous GEMM drains;
// they wait for it before reading anything.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }



constexpr int kUnroll = 4;  // independent 16-byte loads per lane in flight

__device__ __forceinline__ float4 ldg4(const float4* p) { return __ldg(p); }

// Smallest non-zero magnitude of v (+inf if all zero): a thread whose elements
// all sit at or above the row's residual candidate bound skips the check.
__device__ __forceinline__ float absmin_nz4(const float4& v) {
  const float ax = v.x != 0.f ? fabsf(v.x) : INFINITY, ay = v.y != 0.f ? fabsf(v.y) : INFINITY;
  const float az = v.z != 0.f ? fabsf(v.z) : INFINITY, aw = v.w != 0.f ? fabsf(v.w) : INFINITY;
  return fminf(fminf(ax, ay), fminf(az, aw));
}

__device__ __forceinline__ float absmax4(const float4& v) {
  if (isnan(v.x) || isnan(v.y) || isnan(v.z) || isnan(v.w)) return INFINITY;
  return fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
}

// split4 with residual tracking (fix.h): elements whose halves miss them by
// more than 2^-19 are listed for the fix-up; col0 = k index of v.x; cand =
// f16s_candidate_bound(1/s), or 0 for an untracked row.
__device__ __forceinline__ void split4c(const float4& v, float s, float inv_s, float cand,
                                        uint2& hw, uint2& lw, const FixList& fl, int64_t row,
                                        int64_t col0) {
  __half h0, h1, h2, h3, l0, l1, l2, l3;
  f16s_split_checked(v.x, s, inv_s, cand, h0, l0, fl, row, col0);
  f16s_split_checked(v.y, s, inv_s, cand, h1, l1, fl, row, col0 + 1);
  f16s_split_checked(v.z, s, inv_s, cand, h2, l2, fl, row, col0 + 2);
  f16s_split_checked(v.w, s, inv_s, cand, h3, l3, fl, row, col0 + 3);
  __half2 hp0 = __halves2half2(h0, h1), hp1 = __halves2half2(h2, h3);
  __half2 lp0 = __halves2half2(l0, l1), lp1 = __halves2half2(l2, l3);
  hw = make_uint2(*reinterpret_cast<uint32_t*>(&hp0), *reinterpret_cast<uint32_t*>(&hp1));
  lw = make_uint2(*reinterpret_cast<uint32_t*>(&lp0), *reinterpret_cast<uint32_t*>(&lp1));
}
__device__ __forceinline__ void split4(const float4& v, float s, uint2& hw, uint2& lw) {
  const __half2 h01 = __floats2half2_rn(v.x * s, v.y * s), h23 = __floats2half2_rn(v.z * s, v.w * s);
  const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
  const __half2 l01 = __floats2half2_rn(v.x * s - f01.x, v.y * s - f01.y);
  const __half2 l23 = __floats2half2_rn(v.z * s - f23.x, v.w * s - f23.y);
  hw = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
  lw = make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
}
// chk: this thread holds a residual candidate (see absmin_nz4).
__device__ __forceinline__ void split4x(bool chk, const float4& v, float s, float inv_s, float cand,
                                        uint2& hw, uint2& lw, const FixList& fl, int64_t row,
                                        int64_t col0) {
  if (chk) split4c(v, s, inv_s, cand, hw, lw, fl, row, col0);
  else split4(v, s, hw, lw);
}
// Residual check only (operands the GEMM splits in-kernel from raw rows: the
// halves it builds are bit-identical to these). One compare per element unless
// an element is a candidate.
__device__ __forceinline__ void check4(const float4& v, float s, float inv_s, float cand,
                                       const FixList& fl, int64_t row, int64_t col0) {
  f16s_check(v.x, s, inv_s, cand, fl, row, col0);
  f16s_check(v.y, s, inv_s, cand, fl, row, col0 + 1);
  f16s_check(v.z, s, inv_s, cand, fl, row, col0 + 2);
  f16s_check(v.w, s, inv_s, cand, fl, row, col0 + 3);
}
__device__ __forceinline__ void split_col4(const float4& v, const float4& sc, const float4& inv,
                                           uint2& hw, uint2& lw, const FixList& fl, int64_t col,
                                           int64_t krow) {
  __half h0, h1, h2, h3, l0, l1, l2, l3;
  f16s_split_checked(v.x, sc.x, inv.x, f16s_candidate_bound(inv.x), h0, l0, fl, col, krow);
  f16s_split_checked(v.y, sc.y, inv.y, f16s_candidate_bound(inv.y), h1, l1, fl, col + 1, krow);
  f16s_split_checked(v.z, sc.z, inv.z, f16s_candidate_bound(inv.z), h2, l2, fl, col + 2, krow);
  f16s_split_checked(v.w, sc.w, inv.w, f16s_candidate_bound(inv.w), h3, l3, fl, col + 3, krow);
  __half2 hp0 = __halves2half2(h0, h1), hp1 = __halves2half2(h2, h3);
  __half2 lp0 = __halves2half2(l0, l1), lp1 = __halves2half2(l2, l3);
  hw = make_uint2(*reinterpret_cast<uint32_t*>(&hp0), *reinterpret_cast<uint32_t*>(&hp1));
  lw = make_uint2(*reinterpret_cast<uint32_t*>(&lp0), *reinterpret_cast<uint32_t*>(&lp1));
}
// Columns: per-component minimum of the non-zero magnitudes seen.
__device__ __forceinline__ float4 absmin_nz_each(const float4& m, const float4& v) {
  return make_float4(v.x != 0.f ? fminf(m.x, fabsf(v.x)) : m.x, v.y != 0.f ? fminf(m.y, fabsf(v.y)) : m.y,
                     v.z != 0.f ? fminf(m.z, fabsf(v.z)) : m.z, v.w != 0.f ? fminf(m.w, fabsf(v.w)) : m.w);
}
__device__ __forceinline__ bool col_candidates(const float4& mn, const float4& inv) {
  return mn.x < f16s_candidate_bound(inv.x) || mn.y < f16s_candidate_bound(inv.y) ||
         mn.z < f16s_candidate_bound(inv.z) || mn.w < f16s_candidate_bound(inv.w);
}
__device__ __forceinline__ void split_col4x(bool chk, const float4& v, const float4& sc,
                                            const float4& inv, uint2& hw, uint2& lw,
                                            const FixList& fl, int64_t col, int64_t krow) {
  if (chk) {
    split_col4(v, sc, inv, hw, lw, fl, col, krow);
    return;
  }
  const __half2 h01 = __floats2half2_rn(v.x * sc.x, v.y * sc.y), h23 = __floats2half2_rn(v.z * sc.z, v.w * sc.w);
  const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
  const __half2 l01 = __floats2half2_rn(v.x * sc.x - f01.x, v.y * sc.y - f01.y);
  const __half2 l23 = __floats2half2_rn(v.z * sc.z - f23.x, v.w * sc.w - f23.y);
  hw = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
  lw = make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
}
// 1/s for the residual check, 0 (= untracked) for a row or column whose max is
// Inf/NaN: its output is non-finite anyway and its scale (1) says nothing
// about the other entries' range.
__device__ __forceinline__ float track_inv(float mx, float inv) { return mx <= 3.402823466e38f ? inv : 0.f; }
__device__ __forceinline__ float4 track_inv4(const float4& m, const float4& sc) {
  return make_float4(track_inv(m.x, 1.f / sc.x), track_inv(m.y, 1.f / sc.y),
                     track_inv(m.z, 1.f / sc.z), track_inv(m.w, 1.f / sc.w));
}

// A launch serves up to two K-major operands (A and B of one GEMM, same k):
// job 0 owns virtual rows [0, j0.rows), job 1 the next j1.rows. A job with
// hi == nullptr only computes its row scales (the GEMM splits it in-kernel).
struct RowJob {
  const float* x;
  __half* hi;
  __half* lo;
  float* inv_scale;
  int64_t rows;
  FixList fix;  // residual list (fix.h); ctr == nullptr: none
};

__device__ __forceinline__ RowJob pick(const RowJob& j0, const RowJob& j1, int64_t v, int64_t& r) {
  // field-wise select (a reference to either parameter would force both into local memory)
  const bool first = v < j0.rows;
  r = first ? v : v - j0.rows;
  RowJob j;
  j.x = first ? j0.x : j1.x;
  j.hi = first ? j0.hi : j1.hi;
  j.lo = first ? j0.lo : j1.lo;
  j.inv_scale = first ? j0.inv_scale : j1.inv_scale;
  j.rows = first ? j0.rows : j1.rows;
  j.fix.ctr = first ? j0.fix.ctr : j1.fix.ctr;
  j.fix.e = first ? j0.fix.e : j1.fix.e;
  j.fix.cap = first ? j0.fix.cap : j1.fix.cap;
  j.fix.row0 = first ? j0.fix.row0 : j1.fix.row0;
  return j;
}

// One warp per row: max, then (split jobs) split. Both passes keep kUnroll
// independent 16-byte loads per lane in flight; the second pass re-reads the
// row from L1/L2 (a row is at most 8 KiB here).
__global__ void __launch_bounds__(256)
split_rows_f16_kernel(const RowJob j0, const RowJob j1, int64_t k) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x % 32;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) / 32;
  const int64_t k4 = k / 4;
  constexpr int kStep = 32 * kUnroll;
  for (int64_t v = warp; v < j0.rows + j1.rows; v += nwarps) {
    int64_t r;
    const RowJob j = pick(j0, j1, v, r);
    const float4* row = reinterpret_cast<const float4*>(j.x + r * k);
    float mx = 0.f, mn = INFINITY;
    int64_t i = lane;
    for (; i + 32 * (kUnroll - 1) < k4; i += kStep) {
      float4 x[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) x[u] = ldg4(row + i + 32 * u);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        mx = fmaxf(mx, absmax4(x[u]));
        mn = fminf(mn, absmin_nz4(x[u]));
      }
    }
    for (; i < k4; i += 32) {
      const float4 x = ldg4(row + i);
      mx = fmaxf(mx, absmax4(x));
      mn = fminf(mn, absmin_nz4(x));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float s = pow2_scale(mx);
    const float inv = 1.f / s;
    const float cand = j.fix.ctr ? f16s_candidate_bound(track_inv(mx, inv)) : 0.f;
    const bool chk = mn < cand;  // this thread holds a residual candidate
    if (lane == 0) j.inv_scale[r] = inv;
    if (j.hi == nullptr) {  // row scales only (+ the residual check, from L1/L2)
      if (chk)
        for (i = lane; i < k4; i += 32) check4(ldg4(row + i), s, inv, cand, j.fix, r, 4 * i);
      continue;
    }
    uint2* hrow = reinterpret_cast<uint2*>(j.hi + r * k);
    uint2* lrow = reinterpret_cast<uint2*>(j.lo + r * k);
    i = lane;
    for (; i + 32 * (kUnroll - 1) < k4; i += kStep) {
      float4 x[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) x[u] = ldg4(row + i + 32 * u);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        uint2 hw, lw;
        split4x(chk, x[u], s, inv, cand, hw, lw, j.fix, r, 4 * (i + 32 * u));
        hrow[i + 32 * u] = hw;
        lrow[i + 32 * u] = lw;
      }
    }
    for (; i < k4; i += 32) {
      uint2 hw, lw;
      split4x(chk, ldg4(row + i), s, inv, cand, hw, lw, j.fix, r, 4 * i);
      hrow[i] = hw;
      lrow[i] = lw;
    }
  }
}

// Rows of up to 32 * kR float4 (k <= 128 * kR): one warp per row with the whole
// row held in registers — every load is issued before the first use, so a row
// costs one DRAM round trip and one read (the looped kernel above re-reads the
// row for the split pass and waits on each unrolled batch).
template <int kR>
__global__ void __launch_bounds__(256)
split_rows_f16_reg_kernel(const RowJob j0, const RowJob j1, int64_t k) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x % 32;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) / 32;
  const int64_t k4 = k / 4;
  for (int64_t v = warp; v < j0.rows + j1.rows; v += nwarps) {
    int64_t r;
    const RowJob j = pick(j0, j1, v, r);
    const float4* row = reinterpret_cast<const float4*>(j.x + r * k);
    float4 x[kR];
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const int64_t i = lane + 32 * u;
      x[u] = i < k4 ? ldg4(row + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float mx = 0.f, mn = INFINITY;
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      mx = fmaxf(mx, absmax4(x[u]));
      mn = fminf(mn, absmin_nz4(x[u]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float s = pow2_scale(mx);
    const float inv = 1.f / s;
    const float cand = j.fix.ctr ? f16s_candidate_bound(track_inv(mx, inv)) : 0.f;
    const bool chk = mn < cand;  // this thread holds a residual candidate
    if (lane == 0) j.inv_scale[r] = inv;
    if (j.hi == nullptr) {  // row scales only (+ the residual check)
      if (chk) {
#pragma unroll
        for (int u = 0; u < kR; ++u) {
          const int64_t i = lane + 32 * u;
          if (i < k4) check4(x[u], s, inv, cand, j.fix, r, 4 * i);
        }
      }
      continue;
    }
    uint2* hrow = reinterpret_cast<uint2*>(j.hi + r * k);
    uint2* lrow = reinterpret_cast<uint2*>(j.lo + r * k);
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const int64_t i = lane + 32 * u;
      if (i < k4) {
        uint2 hw, lw;
        split4x(chk, x[u], s, inv, cand, hw, lw, j.fix, r, 4 * i);
        hrow[i] = hw;
        lrow[i] = lw;
      }
    }
  }
}

// One CTA per row for rows too long for registers (16384 < k, row <= 160 KiB;
// all k > kWarpRowMax with MTNN_SPLIT_CTAREG=0): split jobs stage the row in
// shared memory during the max pass, so DRAM sees exactly one read and one write
// per element (8 B) — with warp-per-row the ~600 MB of long rows in flight
// overflow L2 and the split pass re-reads them from DRAM (12 B per element).
// Row-scale-only jobs just read (4 B per element).
constexpr int kWarpRowMax = 2048;
constexpr int kRowThreads = 512;

__global__ void __launch_bounds__(kRowThreads)
split_rows_f16_smem_kernel(const RowJob j0, const RowJob j1, int64_t k) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float4 row_s[];
  __shared__ float red[kRowThreads / 32];
  const int64_t k4 = k / 4;
  const int t = threadIdx.x;
  for (int64_t v = blockIdx.x; v < j0.rows + j1.rows; v += gridDim.x) {
    int64_t r;
    const RowJob j = pick(j0, j1, v, r);
    const bool stage = j.hi != nullptr || j.fix.ctr != nullptr;
    const float4* row = reinterpret_cast<const float4*>(j.x + r * k);
    float mx = 0.f, mn = INFINITY;
    int64_t i = t;
    for (; i + kRowThreads * (kUnroll - 1) < k4; i += kRowThreads * kUnroll) {
      float4 x[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) x[u] = ldg4(row + i + kRowThreads * u);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        if (stage) row_s[i + kRowThreads * u] = x[u];
        mx = fmaxf(mx, absmax4(x[u]));
        mn = fminf(mn, absmin_nz4(x[u]));
      }
    }
    for (; i < k4; i += kRowThreads) {
      const float4 x = ldg4(row + i);
      if (stage) row_s[i] = x;
      mx = fmaxf(mx, absmax4(x));
      mn = fminf(mn, absmin_nz4(x));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (t % 32 == 0) red[t / 32] = mx;
    __syncthreads();
    if (t < 32) {
      float m2 = t < kRowThreads / 32 ? red[t] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m2 = fmaxf(m2, __shfl_xor_sync(0xffffffffu, m2, o));
      if (t == 0) red[0] = m2;
    }
    __syncthreads();
    const float s = pow2_scale(red[0]);
    const float inv = 1.f / s;
    const float cand = j.fix.ctr ? f16s_candidate_bound(track_inv(red[0], inv)) : 0.f;
    const bool chk = mn < cand;  // this thread holds a residual candidate
    if (t == 0) j.inv_scale[r] = inv;
    if (stage && j.hi != nullptr) {
      uint2* hrow = reinterpret_cast<uint2*>(j.hi + r * k);
      uint2* lrow = reinterpret_cast<uint2*>(j.lo + r * k);
      for (int64_t q = t; q < k4; q += kRowThreads) {
        uint2 hw, lw;
        split4x(chk, row_s[q], s, inv, cand, hw, lw, j.fix, r, 4 * q);
        hrow[q] = hw;
        lrow[q] = lw;
      }
    } else if (stage && chk) {
      for (int64_t q = t; q < k4; q += kRowThreads) check4(row_s[q], s, inv, cand, j.fix, r, 4 * q);
    }
    __syncthreads();  // row_s and red are reused by the next row
  }
}

// One CTA per row with the row in registers (2048 < k <= 256 * 4 * kV): every
// thread issues its kV 16-byte loads before the first use, the row max goes
// through one shared-memory round (double-buffered by row parity, so one
// barrier per row), and the halves are written from the same registers. Several
// CTAs per SM keep 80-128 KiB of loads in flight per SM; the smem-staged kernel
// above serialises load, reduce and store phases inside one CTA.
constexpr int kCtaRowThreads = 256;

template <int kV>
__global__ void __launch_bounds__(kCtaRowThreads)
split_rows_f16_ctareg_kernel(const RowJob j0, const RowJob j1, int64_t k) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[2][kCtaRowThreads / 32];
  const int64_t k4 = k / 4;
  const int t = threadIdx.x;
  int parity = 0;
  for (int64_t v = blockIdx.x; v < j0.rows + j1.rows; v += gridDim.x, parity ^= 1) {
    int64_t r;
    const RowJob j = pick(j0, j1, v, r);
    const float4* row = reinterpret_cast<const float4*>(j.x + r * k);
    float4 x[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int64_t i = t + kCtaRowThreads * u;
      x[u] = i < k4 ? ldg4(row + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float mx = 0.f, mn = INFINITY;
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      mx = fmaxf(mx, absmax4(x[u]));
      mn = fminf(mn, absmin_nz4(x[u]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (t % 32 == 0) red[parity][t / 32] = mx;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kCtaRowThreads / 32; ++w) mx = fmaxf(mx, red[parity][w]);
    const float s = pow2_scale(mx);
    const float inv = 1.f / s;
    const float cand = j.fix.ctr ? f16s_candidate_bound(track_inv(mx, inv)) : 0.f;
    const bool chk = mn < cand;  // this thread holds a residual candidate
    if (t == 0) j.inv_scale[r] = inv;
    if (j.hi == nullptr) {  // row scales only (+ the residual check)
      if (chk) {
#pragma unroll
        for (int u = 0; u < kV; ++u) {
          const int64_t i = t + kCtaRowThreads * u;
          if (i < k4) check4(x[u], s, inv, cand, j.fix, r, 4 * i);
        }
      }
      continue;
    }
    uint2* hrow = reinterpret_cast<uint2*>(j.hi + r * k);
    uint2* lrow = reinterpret_cast<uint2*>(j.lo + r * k);
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int64_t i = t + kCtaRowThreads * u;
      if (i < k4) {
        uint2 hw, lw;
        split4x(chk, x[u], s, inv, cand, hw, lw, j.fix, r, 4 * i);
        hrow[i] = hw;
        lrow[i] = lw;
      }
    }
  }
}

template <int kV>
int launch_ctareg(const RowJob& j0, const RowJob& j1, int64_t rows, int64_t k, int sm_count,
                  cudaStream_t s) {
  static const int per_sm = [] {  // same on every device of a node (B200 only)
    int v = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, split_rows_f16_ctareg_kernel<kV>,
                                                      kCtaRowThreads, 0) != cudaSuccess) {
      (void)cudaGetLastError();
      v = 1;
    }
    return std::max(v, 1);
  }();
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)sm_count * per_sm));
  MTNN_TRY(launch_chained(split_rows_f16_ctareg_kernel<kV>, dim3((unsigned)blocks), dim3(kCtaRowThreads),
                           0, s, j0, j1, k));
  return MTNN_OK;
}

bool ctareg_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("MTNN_SPLIT_CTAREG");  // 0: smem-staged kernel (A/B runs)
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// Column split (MN-major B^T, k x n) with one scale per 256-row chunk of each
// column (kScaleChunkK, the GEMM's FP32-promotion period): the GEMM epilogue
// multiplies each TMEM chunk partial by its chunk's exact 1/s (gemm_tc.cu), so
// a chunk's scale only needs that chunk's maximum. Every (chunk, 32-column)
// block is then independent: one CTA reads its 256 x 32 block once (8 16-byte
// loads per thread, all issued before the first use), reduces the column
// maxima (shuffles + one shared-memory round), and writes the halves from
// registers — 8 B of DRAM traffic per element, no cross-CTA exchange, no second
// read, and (k/256) x (n/32) CTAs in flight instead of the cluster strips'
// serialised load/reduce/store phases (k = n = 4096: 43 us at 1.6 TB/s of reads
// -> this kernel). inv_scale is [ceil(k/256)][n].
__device__ __forceinline__ float nanmax(float m, float v) {
  return isnan(v) ? INFINITY : fmaxf(m, fabsf(v));
}

constexpr int kColBlockCols = 32;
constexpr int kColRowLanes = 32;
constexpr int kColRowsPerLane = kScaleChunkK / kColRowLanes;  // 8

// The A rows of the same NN call (K-major, one scale per row) ride along in the
// same launch (`rows`, blocks past the column grid: one CTA per row, max pass
// then split from an L1/L2 re-read — the same per-element operations as the
// row kernels, so the halves are identical), so the two splits overlap instead
// of running as two chained launches.
__device__ void split_row_cta(const RowJob& j, int64_t r, int64_t k, float* red) {
  const float4* row = reinterpret_cast<const float4*>(j.x + r * k);
  const int64_t k4 = k / 4;
  const int t = threadIdx.x;
  float mx = 0.f, mn = INFINITY;
#pragma unroll 4
  for (int64_t i = t; i < k4; i += 256) {
    const float4 v = ldg4(row + i);
    mx = fmaxf(mx, absmax4(v));
    mn = fminf(mn, absmin_nz4(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (t % 32 == 0) red[t / 32] = mx;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < 8; ++w) mx = fmaxf(mx, red[w]);
  const float s = pow2_scale(mx);
  const float inv = 1.f / s;
  const float cand = j.fix.ctr ? f16s_candidate_bound(track_inv(mx, inv)) : 0.f;
  const bool chk = mn < cand;
  if (t == 0) j.inv_scale[r] = inv;
  uint2* hrow = reinterpret_cast<uint2*>(j.hi + r * k);
  uint2* lrow = reinterpret_cast<uint2*>(j.lo + r * k);
#pragma unroll 4
  for (int64_t i = t; i < k4; i += 256) {
    uint2 hw, lw;
    split4x(chk, ldg4(row + i), s, inv, cand, hw, lw, j.fix, r, 4 * i);
    hrow[i] = hw;
    lrow[i] = lw;
  }
}

__global__ void __launch_bounds__(8 * kColRowLanes)
split_cols_chunk_kernel(const float* __restrict__ x, __half* __restrict__ hi,
                        __half* __restrict__ lo, float* __restrict__ inv_scale, int64_t k,
                        int64_t n, const FixList fl, const RowJob rows) {
  pdl_trigger();
  pdl_wait();
  __shared__ float4 wmax[8][8];  // [warp][16-byte column]
  __shared__ float4 scale[8];
  __shared__ float4 tinv_s[8];
  const int64_t nbx = (n + kColBlockCols - 1) / kColBlockCols;
  const int64_t ncol_blocks = nbx * ((k + kScaleChunkK - 1) / kScaleChunkK);
  if ((int64_t)blockIdx.x >= ncol_blocks) {
    split_row_cta(rows, (int64_t)blockIdx.x - ncol_blocks, k, reinterpret_cast<float*>(wmax));
    return;
  }
  const int64_t bx = (int64_t)blockIdx.x % nbx, by = (int64_t)blockIdx.x / nbx;
  const int c4 = threadIdx.x % 8;
  const int rl = threadIdx.x / 8;      // 0..31; a warp holds row lanes 4w..4w+3
  const int warp = threadIdx.x / 32;
  const int64_t col = bx * kColBlockCols + 4 * c4;
  const bool active = col < n;  // n % 4 == 0: the whole float4 is in range
  const int64_t r0 = by * kScaleChunkK + rl;
  float4 v[kColRowsPerLane];
#pragma unroll
  for (int u = 0; u < kColRowsPerLane; ++u) {
    const int64_t r = r0 + kColRowLanes * u;
    v[u] = (active && r < k) ? ldg4(reinterpret_cast<const float4*>(x + r * n + col))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float4 mx = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 mn = make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
#pragma unroll
  for (int u = 0; u < kColRowsPerLane; ++u) {
    mx.x = nanmax(mx.x, v[u].x); mx.y = nanmax(mx.y, v[u].y);
    mx.z = nanmax(mx.z, v[u].z); mx.w = nanmax(mx.w, v[u].w);
    mn = absmin_nz_each(mn, v[u]);
  }
  // lanes 8 and 16 apart hold the same columns
#pragma unroll
  for (int off = 8; off < 32; off <<= 1) {
    mx.x = fmaxf(mx.x, __shfl_xor_sync(0xffffffffu, mx.x, off));
    mx.y = fmaxf(mx.y, __shfl_xor_sync(0xffffffffu, mx.y, off));
    mx.z = fmaxf(mx.z, __shfl_xor_sync(0xffffffffu, mx.z, off));
    mx.w = fmaxf(mx.w, __shfl_xor_sync(0xffffffffu, mx.w, off));
  }
  if (threadIdx.x % 32 < 8) wmax[warp][c4] = mx;
  __syncthreads();
  if (threadIdx.x < 8) {
    float4 m = wmax[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      const float4 o = wmax[w][threadIdx.x];
      m.x = fmaxf(m.x, o.x); m.y = fmaxf(m.y, o.y); m.z = fmaxf(m.z, o.z); m.w = fmaxf(m.w, o.w);
    }
    const float4 sc = make_float4(pow2_scale(m.x), pow2_scale(m.y), pow2_scale(m.z), pow2_scale(m.w));
    scale[threadIdx.x] = sc;
    tinv_s[threadIdx.x] = track_inv4(m, sc);
    const int64_t c = bx * kColBlockCols + 4 * threadIdx.x;
    if (c < n)
      *reinterpret_cast<float4*>(inv_scale + by * n + c) =
          make_float4(1.f / sc.x, 1.f / sc.y, 1.f / sc.z, 1.f / sc.w);
  }
  __syncthreads();
  if (!active) return;
  const float4 sc = scale[c4];
  const float4 inv = tinv_s[c4];
  const bool chk = fl.ctr != nullptr && col_candidates(mn, inv);
#pragma unroll
  for (int u = 0; u < kColRowsPerLane; ++u) {
    const int64_t r = r0 + kColRowLanes * u;
    if (r < k) {
      uint2 hw, lw;
      split_col4x(chk, v[u], sc, inv, hw, lw, fl, col, r);
      const int64_t i = (r * n + col) / 4;
      reinterpret_cast<uint2*>(hi)[i] = hw;
      reinterpret_cast<uint2*>(lo)[i] = lw;
    }
  }
}


}  // namespace

// Splits (hi != nullptr) or row-scales (hi == nullptr) the rows of up to two
// K-major operands sharing k, in one launch.
int launch_split_rows_f16_pair(const float* x0, void* hi0, void* lo0, float* inv0, int64_t rows0,
                               const FixList& fix0, const float* x1, void* hi1, void* lo1,
                               float* inv1, int64_t rows1, const FixList& fix1, int64_t k,
                               cudaStream_t s) {
  if (rows0 < 0) rows0 = 0;
  if (rows1 < 0) rows1 = 0;
  if (rows0 + rows1 == 0) return MTNN_OK;
  const DeviceInfo* di = nullptr;
  MTNN_TRY(device_info(&di));
  const RowJob j0{x0, static_cast<__half*>(hi0), static_cast<__half*>(lo0), inv0, rows0, fix0};
  const RowJob j1{x1, static_cast<__half*>(hi1), static_cast<__half*>(lo1), inv1, rows1, fix1};
  const int64_t rows = rows0 + rows1;
  KernelTimer timer(MTNN_KCLASS_SPLIT,
                    ((hi0 ? 8.0 : 4.0) * (double)rows0 + (hi1 ? 8.0 : 4.0) * (double)rows1) * (double)k,
                    s);
  const size_t row_bytes = (size_t)k * sizeof(float);
  const bool any_split = ((hi0 || fix0.ctr) && rows0) || ((hi1 || fix1.ctr) && rows1);
  if (k > kWarpRowMax && k <= 16384 && ctareg_enabled()) {
    // measured (16384 x 8192 rows of 8192): 384 -> 280 us; 4096^2 x 4096: 101 -> 51 us
    if (k <= 4096)
      MTNN_TRY(launch_ctareg<4>(j0, j1, rows, k, di->sm_count, s));
    else if (k <= 8192)
      MTNN_TRY(launch_ctareg<8>(j0, j1, rows, k, di->sm_count, s));
    else
      MTNN_TRY(launch_ctareg<16>(j0, j1, rows, k, di->sm_count, s));
  } else if (k > kWarpRowMax && row_bytes <= 160 * 1024 && any_split) {
    MTNN_TRY(set_max_dynamic_smem((const void*)split_rows_f16_smem_kernel, 160 * 1024));
    const int per_sm = std::max<int>(1, std::min<int>(4, (int)((200 * 1024) / row_bytes)));
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)di->sm_count * per_sm));
    MTNN_TRY(launch_chained(split_rows_f16_smem_kernel, dim3((unsigned)blocks), dim3(kRowThreads),
                            row_bytes, s, j0, j1, k));
  } else {
    int64_t blocks = (rows + 7) / 8;
    // rows of <= 512 and 1024 < k <= 2048: whole row in registers, every load
    // issued before the first use (16384 x 2048: 5.5 -> 6.8 TB/s; 32768 rows of
    // 256: 18.3 -> 16.4 us). 512 < k < 1024 (the FCN's 784): the whole row in
    // registers too (FCN step +0.3%, interleaved A/B; MTNN_SPLIT_REG8=0 keeps the
    // looped kernel), and k = 1024 (split time of NT calls: 16384^2 x 1024 47.1 ->
    // 41.0 us, 2048 x 8192 x 1024 20.5 -> 16.4, 4096 x 784 x 1024 14.4 -> 12.3;
    // MTNN_SPLIT_REG1024=0 keeps the looped kernel there)
    static const bool reg8 = [] { const char* e = getenv("MTNN_SPLIT_REG8"); return !(e && e[0] == '0'); }();
    static const bool reg1024 = [] { const char* e = getenv("MTNN_SPLIT_REG1024"); return !(e && e[0] == '0'); }();
    const bool mid = reg8 && k > 512 && (k < 1024 || (k == 1024 && reg1024));
    const bool reg = k <= 512 || (k > 1024 && k <= 2048) || mid;  // (longer rows: past the smem limit)
    blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)di->sm_count * (reg && k <= 512 ? 8 : 16)));
    if (k <= 256)
      MTNN_TRY(launch_chained(split_rows_f16_reg_kernel<2>, dim3((unsigned)blocks), dim3(256), 0, s, j0, j1, k));
    else if (k <= 512)
      MTNN_TRY(launch_chained(split_rows_f16_reg_kernel<4>, dim3((unsigned)blocks), dim3(256), 0, s, j0, j1, k));
    else if (mid)
      MTNN_TRY(launch_chained(split_rows_f16_reg_kernel<8>, dim3((unsigned)blocks), dim3(256), 0, s, j0, j1, k));
    else if (reg)
      MTNN_TRY(launch_chained(split_rows_f16_reg_kernel<16>, dim3((unsigned)blocks), dim3(256), 0, s, j0, j1, k));
    else
      MTNN_TRY(launch_chained(split_rows_f16_kernel, dim3((unsigned)blocks), dim3(256), 0, s, j0, j1, k));
  }
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}

int launch_split_rows_f16(const float* x, void* hi, void* lo, float* inv_scale, int64_t rows,
                          int64_t k, const FixList& fix, cudaStream_t s) {
  return launch_split_rows_f16_pair(x, hi, lo, inv_scale, rows, fix, nullptr, nullptr, nullptr,
                                    nullptr, 0, FixList{}, k, s);
}

int launch_rowmax_f16(const float* x, float* inv_scale, int64_t rows, int64_t k,
                      const FixList& fix, cudaStream_t s) {
  return launch_split_rows_f16_pair(x, nullptr, nullptr, inv_scale, rows, fix, nullptr, nullptr,
                                    nullptr, nullptr, 0, FixList{}, k, s);
}

int launch_split_cols_f16(const float* x, void* hi, void* lo, float* inv_scale, int64_t k,
                          int64_t n, const FixList& fl, cudaStream_t s, const float* a,
                          void* a_hi, void* a_lo, float* a_inv, int64_t a_rows,
                          const FixList& a_fl) {
  if (k <= 0 || (n <= 0 && a_rows <= 0)) return MTNN_OK;
  if (n < 0) n = 0;
  if (a_rows < 0 || a == nullptr) a_rows = 0;
  const int64_t chunks = (k + kScaleChunkK - 1) / kScaleChunkK;
  const int64_t blocks = (n + kColBlockCols - 1) / kColBlockCols * chunks + a_rows;
  if (blocks > 0x7fffffff) return fail(MTNN_EINVAL, "column split: grid too large");
  const RowJob rj{a, static_cast<__half*>(a_hi), static_cast<__half*>(a_lo), a_inv, a_rows, a_fl};
  KernelTimer timer(MTNN_KCLASS_SPLIT, 8.0 * (double)k * (double)(n + a_rows), s);
  MTNN_TRY(launch_chained(split_cols_chunk_kernel, dim3((unsigned)blocks), dim3(8 * kColRowLanes),
                          0, s, x, static_cast<__half*>(hi), static_cast<__half*>(lo), inv_scale,
                          k, n, fl, rj));
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}

}  // namespace mtnn
