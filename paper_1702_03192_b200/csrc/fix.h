// Residual fix-up lists: the exactness guarantee of the split tensor-core paths.
//
// The FP32-accurate tensor-core GEMMs multiply a two-piece representation of
// each operand element (tc3xf16s: fp16 h + l under one power-of-two scale per
// row; tc3xtf32: trunc-tf32 hi + lo, subnormals flushed by the tensor core).
// For almost every element that representation is exact to <= 2^-23 (f16s) or
// 2^-20 (tf32) of the element itself. It is not for elements far below their
// row's largest value (f16s: the lo half turns subnormal ~2^-17 below the row
// max and both halves flush ~2^-39 below it) nor for FP32-subnormal inputs
// (tf32). Those are exactly the inputs where a row's large entries can be
// cancelled by zeros of the other operand, so the product is carried by the
// badly represented entries.
//
// The split kernels therefore compute each element's residual
//     r = x - represented(x)            (exact in FP32)
// and append (operand row, k index, r) to a per-operand list whenever
// |r| > 2^-19 |x| (every other element is represented within 2^-19, so even
// same-signed errors keep C within ~4e-6 of sum |a b|). After the GEMM one fix-up kernel
// (fixup.cu) adds the missing terms exactly:
//     C[i, :] += r_a(i, p) * B[:, p]            for every A entry
//     C[:, j] += rep(A[:, p]) * r_b(j, p)       for every B entry
// which makes C = A B^T up to FP32 rounding of each term, whatever the intra-
// row range. Uniform data lists ~2^-20 of its elements (a few hundred entries
// per 16384^2 operand), which the fix-up sorts on chip so every output is
// updated once, in a fixed order (deterministic). A list that overflows its
// capacity (adversarial data: a sizeable fraction of entries far below their
// row max) makes the fix-up recompute the whole output with FFMA instead.
//
// Counters: a per-device ring of zero-initialised {count, done} pairs. A call
// takes one per split operand; the fix-up's last CTA resets it, and an
// unconsumed pair (error exit) is reset by a stream-ordered memset.
#pragma once

#include <stdint.h>
#ifdef __CUDACC__
#include <cuda_fp16.h>
#endif

namespace mtnn {

struct FixEntry {
  int32_t row;  // operand row (a row of A, a row of B for NT, a column of B^T for NN)
  int32_t col;  // k index
  float r;      // x - represented(x), exact
};

struct FixCounter {
  unsigned count;  // entries appended (may exceed cap: overflow)
  unsigned done;   // fix-up CTAs that have read `count` (reset protocol)
};

// Device-side view of one operand's list, passed by value to the split kernels.
struct FixList {
  FixCounter* ctr = nullptr;  // null: no residual tracking for this operand
  FixEntry* e = nullptr;
  unsigned cap = 0;
  int32_t row0 = 0;  // global row index of the operand's row 0 (row-blocked splits)
};

// Residual thresholds (relative to |x|, resp. |x * s|).
constexpr float kFixRelF16S = 0x1p-19f;
constexpr float kFixRelTF32 = 0x1p-19f;

#ifdef __CUDACC__
__device__ __forceinline__ void fix_push(const FixList& fl, int64_t row, int64_t col, float r) {
  if (fl.ctr == nullptr) return;
  const unsigned i = atomicAdd(&fl.ctr->count, 1u);
  if (i < fl.cap) fl.e[i] = FixEntry{(int32_t)(fl.row0 + row), (int32_t)col, r};
}

// tc3xf16s: h = fp16(x s), l = fp16(x s - h); residual (x s - h - l) / s.
// Only elements with |x s| < 2^-6 can miss by more than 2^-19 (the residual
// is <= 2^-23 |x s| while l is normal and <= 2^-25 once it is subnormal), so
// the exact check runs behind the one-compare filter |x| < cand = 2^-6 / s.
// cand == 0: the row is not tracked (no list, or its max is Inf/NaN).
__device__ __forceinline__ float f16s_candidate_bound(float inv_s) { return 0x1p-6f * inv_s; }
__device__ __forceinline__ void f16s_check(float v, float s, float inv_s, float cand,
                                           const FixList& fl, int64_t row, int64_t col) {
  if (!(fabsf(v) < cand) || v == 0.f) return;
  const float xs = v * s;
  const float h = __half2float(__float2half_rn(xs));
  const float d = xs - h;
  const float rem = d - __half2float(__float2half_rn(d));
  if (fabsf(rem) > kFixRelF16S * fabsf(xs)) fix_push(fl, row, col, rem * inv_s);
}
__device__ __forceinline__ void f16s_split_checked(float v, float s, float inv_s, float cand,
                                                   __half& h, __half& l, const FixList& fl,
                                                   int64_t row, int64_t col) {
  const float xs = v * s;
  h = __float2half_rn(xs);
  const float d = xs - __half2float(h);
  l = __float2half_rn(d);
  if (fabsf(v) < cand && v != 0.f) {
    const float rem = d - __half2float(l);
    if (fabsf(rem) > kFixRelF16S * fabsf(xs)) fix_push(fl, row, col, rem * inv_s);
  }
}

// The value the f16s GEMM multiplies for x (row scale s = 1 / inv_s).
__device__ __forceinline__ float f16s_represented(float v, float inv_s) {
  const float xs = v * (1.f / inv_s);
  const __half h = __float2half_rn(xs);
  const __half l = __float2half_rn(xs - __half2float(h));
  return (__half2float(h) + __half2float(l)) * inv_s;
}

// tc3xtf32: the tensor core reads an fp32 operand as trunc-tf32 and flushes
// subnormals; hi is x itself (trunc mode) or rna_tf32(x) (MTNN_SPLIT=rna).
__device__ __forceinline__ float tf32_ftz_trunc(float x) {
  const float t = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  return fabsf(t) < 0x1p-126f ? 0.f : t;
}
template <bool kRna>
__device__ __forceinline__ float tf32_hi(float x) {
  if (kRna) {
    uint32_t t;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(x));
    return __uint_as_float(t);
  }
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
// lo as written by the split; represented = ftz(hi) + ftz(trunc(lo)).
template <bool kRna>
__device__ __forceinline__ float tf32_represented(float x) {
  const float hi = tf32_hi<kRna>(x);
  const float lo = x - hi;
  return (fabsf(hi) < 0x1p-126f ? 0.f : hi) + tf32_ftz_trunc(lo);
}
#endif

}  // namespace mtnn
