// Chunk-segment FP16 split for the fused-split tensor-core GEMM (tc3xf16s, NT).
//
// A K-major operand row is cut into segments of kScaleChunkK = 256 k-values
// (the GEMM's FP32-promotion chunk), and each (row, chunk) segment gets its own
// exact power-of-two scale s = 2^(14 - ceil(log2 max|x|)) over the segment:
//     h = fp16_rn(x s),  l = fp16_rn(x s - h),  1/s at inv[chunk * rows + row]
// — the same operations as split_f16.cu's per-row split, only the max is taken
// over 256 values instead of the whole row. The GEMM's epilogue applies each
// chunk's row and column scales to that chunk's TMEM partial (exact: powers of
// two), so no pass needs a whole row before splitting any of it: chunk 0 is
// split by a pre-pass, later chunks by spare warps inside the GEMM while the
// tensor cores work on the earlier ones (gemm_tc.cu, kConv == 3).
//
// One warp splits one segment: lane l owns k-values [8l, 8l + 8) (two 16-byte
// loads, one 16-byte store per half); the residual list (fix.h) takes every
// element the halves miss by more than 2^-19, as in the row split.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

#include "common.h"
#include "fix.h"

namespace mtnn {
namespace seg {

// 2^(14 - ceil(log2(mx))) for finite mx > 0, else 1 (split_f16.cu pow2_scale).
// Normal mx = 1.f * 2^(E-127): ceil(log2 mx) = E - 127 (+1 unless the
// mantissa is 0), so s = 2^(141 - E - (m != 0)) as float bits; subnormal mx
// takes the frexp path.
__device__ __forceinline__ float pow2_scale(float mx) {
  if (!(mx > 0.f) || !isfinite(mx)) return 1.f;
  const uint32_t b = __float_as_uint(mx);
  const int E = (int)(b >> 23);
  if (E > 0) {
    const int c = E - 127 + ((b & 0x7FFFFFu) != 0u ? 1 : 0);
    return __uint_as_float((uint32_t)(min(14 - c, 126) + 127) << 23);
  }
  int e;
  const float f = frexpf(mx, &e);
  const int c = (f == 0.5f) ? e - 1 : e;
  return ldexpf(1.f, min(14 - c, 126));
}

__device__ __forceinline__ float absmax4(const float4& v) {
  if (isnan(v.x) || isnan(v.y) || isnan(v.z) || isnan(v.w)) return INFINITY;
  return fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
}
__device__ __forceinline__ float absmin_nz4(const float4& v) {
  const float ax = v.x != 0.f ? fabsf(v.x) : INFINITY, ay = v.y != 0.f ? fabsf(v.y) : INFINITY;
  const float az = v.z != 0.f ? fabsf(v.z) : INFINITY, aw = v.w != 0.f ? fabsf(v.w) : INFINITY;
  return fminf(fminf(ax, ay), fminf(az, aw));
}

// The two K-major operands of one GEMM as one row space: virtual rows
// [0, rows0) are operand 0 (A), the next rows1 operand 1 (B).
struct Operand {
  const float* x;
  __half* h;
  __half* l;
  float* inv;  // [chunks][rows]
  int64_t rows;
  FixList fix;
};
struct Pair {
  Operand op[2];
  int64_t k;
};
// Field-wise select (indexing op[] with a run-time value would force the
// parameter into local memory).
__device__ __forceinline__ Operand sel(const Pair& pr, int o) {
  Operand r;
  r.x = o ? pr.op[1].x : pr.op[0].x;
  r.h = o ? pr.op[1].h : pr.op[0].h;
  r.l = o ? pr.op[1].l : pr.op[0].l;
  r.inv = o ? pr.op[1].inv : pr.op[0].inv;
  r.rows = o ? pr.op[1].rows : pr.op[0].rows;
  r.fix.ctr = o ? pr.op[1].fix.ctr : pr.op[0].fix.ctr;
  r.fix.e = o ? pr.op[1].fix.e : pr.op[0].fix.e;
  r.fix.cap = o ? pr.op[1].fix.cap : pr.op[0].fix.cap;
  r.fix.row0 = o ? pr.op[1].fix.row0 : pr.op[0].fix.row0;
  return r;
}

// 8 values -> packed halves (split_f16.cu split2 per element; the residual
// check runs only when an element is a candidate: |x| < 2^-6 / s).
__device__ __forceinline__ void split8(const float4& a, const float4& b, float s, float inv_s,
                                       float cand, const FixList& fl, int64_t row, int64_t k0,
                                       uint4& hw, uint4& lw) {
  const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  uint32_t hp[4], lp[4];
  const bool chk = fminf(absmin_nz4(a), absmin_nz4(b)) < cand;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __half2 h2, l2;
    if (chk) {
      __half h0, h1, l0, l1;
      f16s_split_checked(v[2 * i], s, inv_s, cand, h0, l0, fl, row, k0 + 2 * i);
      f16s_split_checked(v[2 * i + 1], s, inv_s, cand, h1, l1, fl, row, k0 + 2 * i + 1);
      h2 = __halves2half2(h0, h1);
      l2 = __halves2half2(l0, l1);
    } else {
      const float x0 = v[2 * i] * s, x1 = v[2 * i + 1] * s;
      h2 = __floats2half2_rn(x0, x1);
      const float2 hf = __half22float2(h2);
      l2 = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
    }
    hp[i] = *reinterpret_cast<const uint32_t*>(&h2);
    lp[i] = *reinterpret_cast<const uint32_t*>(&l2);
  }
  hw = make_uint4(hp[0], hp[1], hp[2], hp[3]);
  lw = make_uint4(lp[0], lp[1], lp[2], lp[3]);
}

// Splits the kNS segments (virtual rows v0 + i * stride, i < kNS, those below
// `vend`) of chunk `c`: all loads first (2 x 16 B per lane per segment in
// flight), then per segment the warp max, the scale and the halves.
template <int kNS>
__device__ __forceinline__ void split_segments(const Pair& pr, int c, int64_t v0, int64_t stride,
                                               int64_t vend, int lane) {
  const int64_t kx = (int64_t)c * kScaleChunkK + 8 * lane;
  const bool kin = kx < pr.k;  // k % 8 == 0: a lane's 8 values are all in or all out
  float4 a[kNS], b[kNS];
#pragma unroll
  for (int i = 0; i < kNS; ++i) {
    const int64_t v = v0 + i * stride;
    a[i] = b[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (v < vend && kin) {
      const int o = v < pr.op[0].rows ? 0 : 1;
      const int64_t r = o ? v - pr.op[0].rows : v;
      const float4* src = reinterpret_cast<const float4*>((o ? pr.op[1].x : pr.op[0].x) + r * pr.k + kx);
      a[i] = __ldcs(src);
      b[i] = __ldcs(src + 1);
    }
  }
#pragma unroll
  for (int i = 0; i < kNS; ++i) {
    const int64_t v = v0 + i * stride;
    if (v >= vend) break;  // warp-uniform
    float mx = kin ? fmaxf(absmax4(a[i]), absmax4(b[i])) : 0.f;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float s = pow2_scale(mx);
    const float inv_s = 1.f / s;
    const int o = v < pr.op[0].rows ? 0 : 1;
    const int64_t r = o ? v - pr.op[0].rows : v;
    const Operand op = sel(pr, o);
    if (lane == 0) op.inv[(int64_t)c * op.rows + r] = inv_s;
    if (!kin) continue;
    // untracked (cand 0): no list, or a non-finite max
    const float cand = (op.fix.ctr != nullptr && mx <= 3.402823466e38f) ? f16s_candidate_bound(inv_s) : 0.f;
    uint4 hw, lw;
    split8(a[i], b[i], s, inv_s, cand, op.fix, r, kx, hw, lw);
    *reinterpret_cast<uint4*>(op.h + r * pr.k + kx) = hw;
    *reinterpret_cast<uint4*>(op.l + r * pr.k + kx) = lw;
  }
}


// One (row, chunk) segment staged in shared memory (`len` <= 256 floats, a
// multiple of 8): lane l takes the float4s at 4l and 128 + 4l (conflict-free
// 16-byte shared loads), the warp max gives the segment's scale, and the
// halves go out as 8-byte stores (each instruction writes 256 contiguous
// bytes of h or l).
__device__ __forceinline__ void split4_checked(const float4& v, float s, float inv_s, float cand,
                                               const FixList& fl, int64_t row, int64_t k0, uint2& hw,
                                               uint2& lw) {
  __half h[4], l[4];
  const float x[4] = {v.x, v.y, v.z, v.w};
  if (fminf(absmin_nz4(v), INFINITY) < cand) {
#pragma unroll
    for (int i = 0; i < 4; ++i) f16s_split_checked(x[i], s, inv_s, cand, h[i], l[i], fl, row, k0 + i);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float xs = x[i] * s;
      h[i] = __float2half_rn(xs);
      l[i] = __float2half_rn(xs - __half2float(h[i]));
    }
  }
  const __half2 h01 = __halves2half2(h[0], h[1]), h23 = __halves2half2(h[2], h[3]);
  const __half2 l01 = __halves2half2(l[0], l[1]), l23 = __halves2half2(l[2], l[3]);
  hw = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
  lw = make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
}

__device__ __forceinline__ void split_staged_segment(const float* seg_smem, int len, const Operand& op,
                                                     int64_t r, int64_t k, int c, int lane) {
  const bool v0 = 4 * lane < len, v1 = 128 + 4 * lane < len;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 e0 = v0 ? reinterpret_cast<const float4*>(seg_smem)[lane] : z;
  const float4 e1 = v1 ? reinterpret_cast<const float4*>(seg_smem)[32 + lane] : z;
  float mx = fmaxf(absmax4(e0), absmax4(e1));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  const float s = pow2_scale(mx);
  const float inv_s = 1.f / s;
  if (lane == 0) op.inv[(int64_t)c * op.rows + r] = inv_s;
  const float cand = (op.fix.ctr != nullptr && mx <= 3.402823466e38f) ? f16s_candidate_bound(inv_s) : 0.f;
  const int64_t k0 = (int64_t)c * kScaleChunkK;
  uint2 hw, lw;
  if (v0) {
    split4_checked(e0, s, inv_s, cand, op.fix, r, k0 + 4 * lane, hw, lw);
    *reinterpret_cast<uint2*>(op.h + r * k + k0 + 4 * lane) = hw;
    *reinterpret_cast<uint2*>(op.l + r * k + k0 + 4 * lane) = lw;
  }
  if (v1) {
    split4_checked(e1, s, inv_s, cand, op.fix, r, k0 + 128 + 4 * lane, hw, lw);
    *reinterpret_cast<uint2*>(op.h + r * k + k0 + 128 + 4 * lane) = hw;
    *reinterpret_cast<uint2*>(op.l + r * k + k0 + 128 + 4 * lane) = lw;
  }
}

}  // namespace seg
}  // namespace mtnn
