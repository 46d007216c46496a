// SIMT FP32 GEMM (FFMA) — the "exact-order" variant of both MTNN paths.
//
// Reference semantics: kernels/_numba_impl.py:139-152 (gemm_nt: C[i,j] = sum_p
// A[i,p] B[j,p], fp32 accumulator) and :31-117 (gemm_nn over B^T, blocked 128,
// fp32). Both accumulate in float32; so does this kernel (one FFMA chain per
// output, k ascending within a split), which keeps the reference's bit-exact
// identity KATs exact (test_kernels.py:32-40, 87-89): every product against an
// identity matrix is exact and the chain adds only zeros around it.
//
// Used for: shapes the tensor-core path cannot take (TMA needs 16-byte row
// strides), small problems where launch latency dominates, and as the explicit
// MTNN_VARIANT_FFMA. B200 notes: 128x128x8 CTA tile, 256 threads, 8x8 register
// micro-tile (two 4-wide halves 64 apart so LDS.128 reads are conflict-free),
// register-staged double buffering of the next k-slice, optional split-K with a
// deterministic second-pass reduction for few-tile / long-k shapes so the grid
// reaches the 148 SMs.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.h"
#include "pdl.h"
#include "sgemm_tile.cuh"
#include "workspace.h"

namespace mtnn {
namespace {

// B_NK: B stored n x k (NT). Else B^T stored k x n (NN).
template <bool B_NK>
__global__ void __launch_bounds__(256)
sgemm_kernel(const float* __restrict__ A, const float* __restrict__ B,
             float* __restrict__ C, int64_t m, int64_t n, int64_t k, int64_t k_chunk,
             int64_t split_stride) {
  pdl_enter();
  __shared__ __align__(16) float As[2][sgemm::BK][sgemm::BM];
  __shared__ __align__(16) float Bs[2][sgemm::BK][sgemm::BN];
  const int64_t bm0 = (int64_t)blockIdx.y * sgemm::BM;
  const int64_t bn0 = (int64_t)blockIdx.x * sgemm::BN;
  const int64_t kbeg = (int64_t)blockIdx.z * k_chunk;
  const int64_t kend = min(k, kbeg + k_chunk);
  float acc[8][8];
  sgemm::tile<B_NK>(A, B, n, m, n, k, bm0, bn0, kbeg, kend, As, Bs, acc);
  sgemm::store(acc, C + (int64_t)blockIdx.z * split_stride, n, m, n, bm0, bn0);
}

// Skinny NT (GEMV-class): one side of the output <= kSkinnyMax (the FCN's
// 10-class layer, batch-1 products). A CTA (8 warps) owns rows of the long
// operand in groups of R and splits k into W slices, one per warp (W = 8 for
// k >= 4096; shorter k gives several row groups per CTA). Per 16-byte k-step a
// lane first issues all its loads — R long-operand pieces (DRAM, read once) and
// the s short-row pieces (L2-resident, reused across the R rows) — then runs
// s x R FFMA chains. The R x SMAX = 32 partial sums are folded across the warp
// by a butterfly that halves the values per lane each step (31 shuffles, lane l
// ends with value l), then across the W slices through shared memory. Output
// (long row r, short row j) goes to C[r * s + j] when the short side is B,
// C[j * L + r] when it is A. No operand split and no 128-wide tensor-core tile
// for a 10-wide output.
constexpr int kSkinnyMax = 16;

__device__ __forceinline__ void butterfly32(float* w, int lane) {
  // w[0..32): afterwards w[0] of lane l holds the warp-wide sum of value l
#pragma unroll
  for (int o = 16, n = 32; o >= 1; o >>= 1, n >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const float send = upper ? w[i] : w[i + n / 2];
      const float keep = upper ? w[i + n / 2] : w[i];
      w[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

template <int SMAX>
__global__ void __launch_bounds__(256, 2)
gemm_skinny_kernel(const float* __restrict__ big, const float* __restrict__ small,
                   float* __restrict__ C, int64_t L, int s, int64_t k, bool small_is_b, int W) {
  pdl_enter();
  constexpr int R = 32 / SMAX;  // long rows per warp: R x SMAX <= 32 partial sums
  __shared__ float red[8][32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int groups = 8 / W;
  const int slice = warp % W, grp = warp / W;
  const int64_t k4 = k / 4;
  const int64_t per = (k4 + W - 1) / W;
  const int64_t q_begin = (int64_t)slice * per, q_end = min(k4, q_begin + per);
  const int64_t rows_per_cta = (int64_t)groups * R;
  const float4* big4 = reinterpret_cast<const float4*>(big);
  const float4* small4 = reinterpret_cast<const float4*>(small);
  for (int64_t base = (int64_t)blockIdx.x * rows_per_cta; base < L;
       base += (int64_t)gridDim.x * rows_per_cta) {
    const int64_t r0 = base + (int64_t)grp * R;
    float acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.f;
    for (int64_t q = q_begin + lane; q < q_end; q += 32) {
      float4 a[R], b[SMAX];
#pragma unroll
      for (int r = 0; r < R; ++r)
        a[r] = r0 + r < L ? __ldg(big4 + (r0 + r) * k4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < SMAX; ++j)
        b[j] = j < s ? __ldg(small4 + (int64_t)j * k4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < SMAX; ++j) {
          float& c = acc[r * SMAX + j];  // (slots past R x SMAX stay 0)
          c = fmaf(a[r].w, b[j].w, fmaf(a[r].z, b[j].z, fmaf(a[r].y, b[j].y, fmaf(a[r].x, b[j].x, c))));
        }
    }
    butterfly32(acc, lane);
    red[warp][lane] = acc[0];
    __syncthreads();
    // fold the W slices of each row group: thread t -> (group, value)
    if (threadIdx.x < groups * 32) {
      const int g2 = threadIdx.x / 32, val = threadIdx.x % 32;
      const int r = val / SMAX, j = val % SMAX;
      const int64_t row = base + (int64_t)g2 * R + r;
      if (r < R && j < s && row < L) {
        float sum = 0.f;
        for (int w = 0; w < W; ++w) sum += red[g2 * W + w][val];
        C[small_is_b ? row * s + j : (int64_t)j * L + row] = sum;
      }
    }
    __syncthreads();  // red is reused by the next row block
  }
}


// Staged skinny NT (round 2): the same products, restructured for memory-level
// parallelism. A CTA (16 warps, up to 4 per SM) owns a block of long rows and pulls
// all of them into shared memory with one bulk copy per row as its first act,
// so the whole long operand is in flight across the chip at once (the 1 TB/s of
// the kernel above was latency: 1.16 waves of CTAs, a few 16-byte loads in
// flight per lane). Warps split k into kwarps slices (lane l of slice w owns
// float4 column w*32 + l; used when kwarps x 32 float4s cover k) and the
// remaining warps take further row groups; each lane holds its short-operand
// columns in registers for every row, and the R x SMAX partial sums fold across
// the warp (butterfly) and the slices (shared memory) in a fixed order, per
// batch of groups x R rows.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int kStagedWarps = 16;

template <int SMAX>
__global__ void __launch_bounds__(kStagedWarps * 32, 1)
gemm_skinny_staged_kernel(const float* __restrict__ big, const float* __restrict__ small,
                          float* __restrict__ C, int64_t L, int s, int64_t k, bool small_is_b,
                          int kwarps, int nb) {
  constexpr int R = 32 / SMAX;
  extern __shared__ __align__(128) float4 rows4[];  // [rows of this CTA][k / 4]
  __shared__ float red[kStagedWarps][32];
  __shared__ __align__(8) unsigned long long bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int groups = kStagedWarps / kwarps;
  const int slice = warp % kwarps, grp = warp / kwarps;
  const int64_t k4 = k / 4;
  const int rows_per_cta = nb * groups * R;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int nr = (int)min((int64_t)rows_per_cta, L - r0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_enter();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar)),
                 "r"((uint32_t)(nr * k * 4))
                 : "memory");
    for (int r = 0; r < nr; ++r)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr(rows4 + (int64_t)r * k4)),
          "l"(big + (r0 + r) * k), "r"((uint32_t)(k * 4)), "r"(smem_addr(&bar))
          : "memory");
  }
  const float4* small4 = reinterpret_cast<const float4*>(small);
  const int64_t q = (int64_t)slice * 32 + lane;  // this lane's float4 column (kwarps x 32 >= k / 4)
  const bool valid = q < k4;
  float4 bv[SMAX];  // its short-operand columns, for every row
#pragma unroll
  for (int j = 0; j < SMAX; ++j)
    bv[j] = (valid && j < s) ? __ldg(small4 + (int64_t)j * k4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(&bar))
        : "memory");
  for (int b = 0; b < nb; ++b) {
    float acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int rl = (b * groups + grp) * R + r;
      const float4 a = (valid && rl < nr) ? rows4[(int64_t)rl * k4 + q] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < SMAX; ++j) {
        float& c = acc[r * SMAX + j];  // (slots past R x SMAX stay 0)
        c = fmaf(a.w, bv[j].w, fmaf(a.z, bv[j].z, fmaf(a.y, bv[j].y, fmaf(a.x, bv[j].x, c))));
      }
    }
    butterfly32(acc, lane);
    red[warp][lane] = acc[0];
    __syncthreads();
    if (threadIdx.x < groups * 32) {
      const int g2 = threadIdx.x / 32, val = threadIdx.x % 32;
      const int r = val / SMAX, j = val % SMAX;
      const int rl = (b * groups + g2) * R + r;
      if (r < R && j < s && rl < nr) {
        float sum = 0.f;
        for (int w = 0; w < kwarps; ++w) sum += red[g2 * kwarps + w][val];
        const int64_t row = r0 + rl;
        C[small_is_b ? row * s + j : (int64_t)j * L + row] = sum;
      }
    }
    __syncthreads();  // red is reused by the next batch
  }
}

// Streaming skinny NT (round 2, session 4). The register kernel above re-reads
// the short operand from L2 for every R long rows (3.3x the long operand's
// bytes at s = 10) and keeps ~4 loads per lane in flight; the staged kernel
// needs the CTA's rows in shared memory. Here a CTA owns a k-range of
// kStreamQ float4 columns (warp w, lane l: column 32w + l) and a block of
// long rows: each lane loads its short-operand columns into registers once,
// then streams the rows — every warp load is 512 contiguous bytes of one row,
// the next R rows' loads are in flight while the current R are multiplied —
// and folds each R x SMAX batch across the warp by the halving butterfly. Per
// chunk of kStreamBatches batches the 8 warps fold through shared memory (warp
// order), then the k-ranges: the CTAs of one cluster along k (up to 8, DSMEM,
// rank order) and, when k has more ranges than a cluster, the clusters'
// partial outputs in a second pass (splitk_reduce, group order).
// Grid: x = k-ranges (clusters of cs consecutive ranges), y = row blocks.
constexpr int kStreamQ = 256;       // float4 columns per CTA k-range (1024 floats)
constexpr int kStreamWarps = 8;
constexpr int kStreamBatches = 8;   // butterfly batches per shared-memory fold of the warps
constexpr int kStreamMaxBatches = 256;  // batches per CTA
constexpr int64_t kStreamMaxBytes = 32ll << 20;  // long operand bytes it is used up to

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

#ifdef MTNN_TRACE
// per-CTA globaltimer stamps (trace builds only: tools/build_variant.sh)
__device__ unsigned long long g_skinny_trace[8192 * 8];
__device__ __forceinline__ void skinny_mark(int pt) {
  if (threadIdx.x != 0) return;
  const int64_t cta = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  if (cta >= 8192) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_skinny_trace[cta * 8 + pt] = t;
}
#define SKINNY_MARK(p) skinny_mark(p)
#else
#define SKINNY_MARK(p)
#endif

template <int SMAX>
__global__ void __launch_bounds__(kStreamWarps * 32, 2)
gemm_skinny_stream_kernel(const float* __restrict__ big, const float* __restrict__ small,
                          float* __restrict__ out, int64_t L, int s, int64_t k, bool small_is_b,
                          int64_t rows_per_cta) {
  constexpr int R = 32 / SMAX;
  __shared__ float red[kStreamWarps][kStreamBatches][32];
  extern __shared__ float part[];  // [batches of this CTA][32]: its k-range's sums
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t cs, rank;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int64_t k4 = k / 4;
  const int64_t q = (int64_t)blockIdx.x * kStreamQ + warp * 32 + lane;  // this lane's column
  const bool valid = q < k4;
  float* C = out + (int64_t)(blockIdx.x / cs) * L * s;  // this cluster's output (or partial)
  const int64_t rbeg = (int64_t)blockIdx.y * rows_per_cta;
  const int64_t rend = min(L, rbeg + rows_per_cta);
  SKINNY_MARK(0);
  pdl_enter();
  SKINNY_MARK(1);
  const float4* col = reinterpret_cast<const float4*>(big) + q;
  float4 bv[SMAX];
#pragma unroll
  for (int j = 0; j < SMAX; ++j)
    bv[j] = (valid && j < s) ? __ldg(reinterpret_cast<const float4*>(small) + (int64_t)j * k4 + q)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
  auto load = [&](float4* a, int64_t r) {
#pragma unroll
    for (int i = 0; i < R; ++i)
      a[i] = (valid && r + i < rend) ? __ldg(col + (r + i) * k4) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  // batches r (cur), r + R (nxt) and r + 2R (nx2) in flight
  float4 cur[R], nxt[R], nx2[R];
  load(cur, rbeg);
  load(nxt, rbeg + R);
  SKINNY_MARK(2);
  for (int64_t c0 = rbeg; c0 < rend; c0 += (int64_t)kStreamBatches * R) {  // chunks
    const int nb = (int)min((int64_t)kStreamBatches, (rend - c0 + R - 1) / R);
    for (int b = 0; b < nb; ++b) {
      const int64_t r = c0 + (int64_t)b * R;
      load(nx2, r + 2 * R);  // (across chunk ends)
      float acc[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = 0.f;
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = 0; j < SMAX; ++j) {
          float& t = acc[i * SMAX + j];
          t = fmaf(cur[i].w, bv[j].w, fmaf(cur[i].z, bv[j].z, fmaf(cur[i].y, bv[j].y, fmaf(cur[i].x, bv[j].x, t))));
        }
      butterfly32(acc, lane);  // lane l: value l of the batch (row l / SMAX, short row l % SMAX)
      red[warp][b][lane] = acc[0];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        cur[i] = nxt[i];
        nxt[i] = nx2[i];
      }
    }
    SKINNY_MARK(3);
    __syncthreads();
    const int b0 = (int)((c0 - rbeg) / R);
    for (int i = threadIdx.x; i < nb * 32; i += kStreamWarps * 32) {
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < kStreamWarps; ++w) v += red[w][i / 32][i % 32];
      part[b0 * 32 + i] = v;
    }
    __syncthreads();  // red is reused by the next chunk
  }
  if (cs > 1) cluster_barrier();  // every CTA's part[] is posted
  SKINNY_MARK(5);
  // CTA `rank` finishes items i = rank, rank + cs, ...: the cluster's k-range
  // partial sums in rank order (DSMEM)
  const int nbt = (int)((rend - rbeg + R - 1) / R);
  for (int i = threadIdx.x * (int)cs + (int)rank; i < nbt * 32; i += kStreamWarps * 32 * (int)cs) {
    const int l = i % 32, ri = l / SMAX, j = l % SMAX;
    const int64_t row = rbeg + (int64_t)(i / 32) * R + ri;
    if (ri >= R || j >= s || row >= rend) continue;
    float v = part[i];
    if (cs > 1) {
      v = 0.f;
      const uint32_t la = smem_addr(part + i);
      for (uint32_t cc = 0; cc < cs; ++cc) {
        float x;
        asm volatile(
            "{\n\t.reg .u32 ra;\n\tmapa.shared::cluster.u32 ra, %1, %2;\n\t"
            "ld.shared::cluster.f32 %0, [ra];\n\t}"
            : "=f"(x)
            : "r"(la), "r"(cc)
            : "memory");
        v += x;
      }
    }
    C[small_is_b ? row * s + j : (int64_t)j * L + row] = v;
  }
  SKINNY_MARK(6);
  if (cs > 1) cluster_barrier();  // peers are done reading this CTA's part[]
  SKINNY_MARK(7);
}

// NN with a tiny inner dimension (k <= 16; the FCN's 1024 x 4096 x 10 backward
// product): C = A B^T is an outer-product sum bound by writing C. A thread owns
// 4 adjacent columns and kNnRows rows: its k float4s of B^T (L2) are loaded
// once, the CTA's rows of A (k floats each) are staged in shared memory, and
// each output float4 is one fixed-order FFMA chain over k, stored with STG.128
// (64 threads write 1 KiB of a row contiguously).
constexpr int kNnSmallK = 16, kNnRows = 8;

template <int K>
__global__ void __launch_bounds__(256)
gemm_nn_smallk_kernel(const float* __restrict__ A, const float* __restrict__ BT,
                      float* __restrict__ C, int64_t m, int64_t n, int k) {
  // exactly K terms (one instantiation per k: no predicated-off iterations —
  // these products are instruction-bound, not memory-bound); A rows padded to
  // 16 floats so a row's k values come in with 16-byte shared loads
  constexpr int KMAX = K;
  __shared__ __align__(16) float As[4 * kNnRows][16];
  pdl_enter();
  const int tx = threadIdx.x % 64, ty = threadIdx.x / 64;  // 64 column groups x 4 row groups
  const int64_t c0 = ((int64_t)blockIdx.x * 64 + tx) * 4;
  const int64_t rbase = (int64_t)blockIdx.y * (4 * kNnRows);
  for (int i = threadIdx.x; i < 4 * kNnRows * 16; i += 256) {
    const int rr = i / 16, p = i % 16;
    As[rr][p] = (p < k && rbase + rr < m) ? __ldg(A + (rbase + rr) * k + p) : 0.f;
  }
  float4 bv[KMAX];
#pragma unroll
  for (int p = 0; p < KMAX; ++p)
    bv[p] = c0 < n ? __ldg(reinterpret_cast<const float4*>(BT + (int64_t)p * n + c0))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  if (c0 >= n) return;
#pragma unroll
  for (int r = 0; r < kNnRows; ++r) {
    const int rr = ty * kNnRows + r;
    const int64_t row = rbase + rr;
    if (row >= m) break;
    float av[16];
#pragma unroll
    for (int p4 = 0; p4 < (KMAX + 3) / 4; ++p4) {
      const float4 t = *reinterpret_cast<const float4*>(&As[rr][4 * p4]);
      av[4 * p4] = t.x; av[4 * p4 + 1] = t.y; av[4 * p4 + 2] = t.z; av[4 * p4 + 3] = t.w;
    }
    float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int p = 0; p < KMAX; ++p) {
      c.x = fmaf(av[p], bv[p].x, c.x);
      c.y = fmaf(av[p], bv[p].y, c.y);
      c.z = fmaf(av[p], bv[p].z, c.z);
      c.w = fmaf(av[p], bv[p].w, c.w);
    }
    *reinterpret_cast<float4*>(C + row * n + c0) = c;
  }
}
}  // namespace

// Deterministic split-K reduction: C[i] = sum_s part[s][i], s ascending.
__global__ void splitk_reduce_kernel(const float* __restrict__ part, float* __restrict__ C,
                                     int64_t count, int splits) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    float s = part[i];
    for (int z = 1; z < splits; ++z) s += part[(int64_t)z * count + i];
    C[i] = s;
  }
}

// The same over float4s (count % 4 == 0, 16-byte aligned): every partial of a
// thread's four outputs is loaded before the first add (up to 8 splits per
// round), so each thread has `splits` 16-byte loads in flight instead of one.
__global__ void splitk_reduce4_kernel(const float4* __restrict__ part, float4* __restrict__ C,
                                      int64_t count4, int splits) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count4; i += stride) {
    float4 s = __ldcs(part + i);
    for (int z0 = 1; z0 < splits; z0 += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (z0 + u < splits) v[u] = __ldcs(part + (int64_t)(z0 + u) * count4 + i);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (z0 + u < splits) {
          s.x += v[u].x;
          s.y += v[u].y;
          s.z += v[u].z;
          s.w += v[u].w;
        }
    }
    C[i] = s;
  }
}

int launch_splitk_reduce(const float* part, float* C, int64_t count, int splits,
                         cudaStream_t s) {
  const DeviceInfo* di = nullptr;
  MTNN_TRY(device_info(&di));
  KernelTimer timer(MTNN_KCLASS_REDUCE, 4.0 * (double)(splits + 1) * (double)count, s);
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (count % 4 == 0 && al16(part) && al16(C)) {
    const int64_t count4 = count / 4;
    const int64_t blocks = std::min<int64_t>((count4 + 255) / 256, (int64_t)di->sm_count * 8);
    MTNN_TRY(launch_chained(splitk_reduce4_kernel, dim3((unsigned)std::max<int64_t>(blocks, 1)),
                            dim3(256), 0, s, reinterpret_cast<const float4*>(part),
                            reinterpret_cast<float4*>(C), count4, splits));
  } else {
    int64_t blocks = (count + 255) / 256;
    blocks = std::min<int64_t>(blocks, (int64_t)di->sm_count * 8);
    MTNN_TRY(launch_chained(splitk_reduce_kernel, dim3((unsigned)std::max<int64_t>(blocks, 1)),
                            dim3(256), 0, s, part, C, count, splits));
  }
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}

int launch_gemm_ffma(const float* A, const float* B, float* C, int64_t m, int64_t n,
                     int64_t k, bool b_is_nk, cudaStream_t s) {
  if (m <= 0 || n <= 0) return MTNN_OK;
  const DeviceInfo* di = nullptr;
  MTNN_TRY(device_info(&di));
  const int64_t tiles_m = (m + sgemm::BM - 1) / sgemm::BM, tiles_n = (n + sgemm::BN - 1) / sgemm::BN;
  if (tiles_m > 65535) return fail(MTNN_EINVAL, "ffma gemm: m=%lld too large", (long long)m);
  // Split K when the tile grid cannot fill the chip and k is long enough.
  int splits = 1;
  const int64_t tiles = tiles_m * tiles_n;
  if (tiles < di->sm_count && k >= 512) {
    splits = (int)std::min<int64_t>((2 * di->sm_count + tiles - 1) / tiles, k / 256);
    splits = std::max(1, std::min(splits, 64));
  }
  int64_t k_chunk = (k + splits - 1) / splits;
  k_chunk = (k_chunk + sgemm::BK - 1) / sgemm::BK * sgemm::BK;
  splits = (int)((k + k_chunk - 1) / std::max<int64_t>(k_chunk, 1));
  if (k <= 0) { splits = 1; k_chunk = 0; }
  float* out = C;
  ScratchBuffer part;
  if (splits > 1) {
    MTNN_TRY(part.alloc((size_t)splits * m * n * sizeof(float), s));
    out = static_cast<float*>(part.ptr);
  }
  dim3 grid((unsigned)tiles_n, (unsigned)tiles_m, (unsigned)splits);
  {
  KernelTimer timer(MTNN_KCLASS_GEMM_FFMA, 2.0 * (double)m * (double)n * (double)k, s);
  if (b_is_nk)
    MTNN_TRY(launch_chained(sgemm_kernel<true>, grid, dim3(256), 0, s, A, B, out, m, n, k, k_chunk,
                            m * n));
  else
    MTNN_TRY(launch_chained(sgemm_kernel<false>, grid, dim3(256), 0, s, A, B, out, m, n, k, k_chunk,
                            m * n));
  }
  MTNN_CUDA_TRY(cudaGetLastError());
  if (splits > 1) MTNN_TRY(launch_splitk_reduce(out, C, m * n, splits, s));
  return MTNN_OK;
}


// Staged skinny NT when the CTA's long rows fit shared memory (<= 200 KiB for
// at least one batch) and the grid still covers most SMs; the register kernel
// above otherwise (MTNN_SKINNY_STAGED=0 forces it).
static bool skinny_staged_enabled() {
  static const bool on = [] {
    const char* e = getenv("MTNN_SKINNY_STAGED");
    return !(e && e[0] == '0');
  }();
  return on;
}

constexpr int kSkinnySmemMax = 200 * 1024;

template <int SMAX>
static int launch_skinny_staged(const float* big, const float* sml, float* C, int64_t L, int s,
                                int64_t k, bool small_is_b, int kwarps, int nb, int64_t grid,
                                size_t smem, cudaStream_t st) {
  auto kern = gemm_skinny_staged_kernel<SMAX>;
  MTNN_TRY(set_max_dynamic_smem((const void*)kern, kSkinnySmemMax));  // (set once: the cap)
  return launch_chained(kern, dim3((unsigned)grid), dim3(kStagedWarps * 32), smem, st, big, sml, C,
                        L, s, k, small_is_b, kwarps, nb);
}

static int try_skinny_staged(const float* big, const float* sml, float* C, int64_t L, int sm_rows,
                             int64_t k, bool small_is_b, int smax, const DeviceInfo* di,
                             cudaStream_t st, bool* done) {
  *done = false;
  if (!skinny_staged_enabled()) return MTNN_OK;
  const int64_t k4 = k / 4;
  int kwarps = 1;
  while (kwarps < kStagedWarps && (int64_t)kwarps * 32 < k4) kwarps *= 2;
  const int groups = kStagedWarps / kwarps, R = 32 / smax;
  const int64_t target = (L + di->sm_count - 1) / di->sm_count;
  int nb = (int)std::max<int64_t>(1, (target + groups * R - 1) / (groups * R));
  const size_t kSmemMax = kSkinnySmemMax;
  while (nb > 1 && (size_t)nb * groups * R * k * 4 > kSmemMax) --nb;
  const size_t smem = (size_t)nb * groups * R * k * 4;
  if (smem > kSmemMax || kSkinnySmemMax > di->max_smem_optin - 8 * 1024) return MTNN_OK;
  // (only where one k-step covers k: there the short operand stays in
  // registers for every row and the kernel measured faster — 10 x 4096 x 1024:
  // 12.5-13.0 vs 15.1 us under ncu; a multi-step version re-read the short
  // operand from L2 per batch and was no faster than the register kernel)
  if (k4 > (int64_t)kwarps * 32) return MTNN_OK;
  const int64_t rows = (int64_t)nb * groups * R;
  const int64_t grid = (L + rows - 1) / rows;
  if (grid > 8 * (int64_t)di->sm_count) return MTNN_OK;  // (long row sets: the register kernel)
  int rc;
  switch (smax) {
    case 4: rc = launch_skinny_staged<4>(big, sml, C, L, sm_rows, k, small_is_b, kwarps, nb, grid, smem, st); break;
    case 8: rc = launch_skinny_staged<8>(big, sml, C, L, sm_rows, k, small_is_b, kwarps, nb, grid, smem, st); break;
    case 10: rc = launch_skinny_staged<10>(big, sml, C, L, sm_rows, k, small_is_b, kwarps, nb, grid, smem, st); break;
    case 12: rc = launch_skinny_staged<12>(big, sml, C, L, sm_rows, k, small_is_b, kwarps, nb, grid, smem, st); break;
    default: rc = launch_skinny_staged<16>(big, sml, C, L, sm_rows, k, small_is_b, kwarps, nb, grid, smem, st); break;
  }
  MTNN_TRY(rc);
  MTNN_CUDA_TRY(cudaGetLastError());
  *done = true;
  return MTNN_OK;
}

// Streaming skinny NT (MTNN_SKINNY_STREAM=0 disables it).
static bool skinny_stream_enabled() {
  static const bool on = [] {
    const char* e = getenv("MTNN_SKINNY_STREAM");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int SMAX>
static int launch_skinny_stream(const float* big, const float* sml, float* C, int64_t L, int s,
                                int64_t k, bool small_is_b, const DeviceInfo* di, cudaStream_t st) {
  constexpr int R = 32 / SMAX;
  auto kern = gemm_skinny_stream_kernel<SMAX>;
  const int64_t nranges = (k / 4 + kStreamQ - 1) / kStreamQ;
  const unsigned cs = (unsigned)std::min<int64_t>(8, nranges);
  const int64_t groups = (nranges + cs - 1) / cs;
  // rows per CTA: two CTAs per SM over the whole grid, in whole batches
  // (capped so the CTA's folded sums, 128 B per batch, stay <= 32 KiB)
  const int64_t want = 2 * (int64_t)di->sm_count;
  int64_t rows = (L * nranges + want - 1) / want;
  rows = std::min<int64_t>(rows, (int64_t)kStreamMaxBatches * R);
  rows = std::max<int64_t>(R, (rows + R - 1) / R * R);
  int64_t nrb = (L + rows - 1) / rows;
  if (nrb > 65535)
    return fail(MTNN_ENOTSUP, "streaming skinny: %lld long rows exceed the grid", (long long)L);
  const size_t smem = (size_t)(rows / R) * 32 * sizeof(float);
  float* out = C;
  ScratchBuffer part;
  if (groups > 1) {
    MTNN_TRY(part.alloc((size_t)groups * L * s * sizeof(float), st));
    out = static_cast<float*>(part.ptr);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(groups * cs), (unsigned)nrb);
  cfg.blockDim = dim3(kStreamWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = chain_enabled() ? 2 : 1;
  MTNN_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, big, sml, out, L, s, k, small_is_b, rows));
  MTNN_CUDA_TRY(cudaGetLastError());
  if (groups > 1) MTNN_TRY(launch_splitk_reduce(out, C, L * s, (int)groups, st));
  return MTNN_OK;
}

static int try_skinny_stream(const float* big, const float* sml, float* C, int64_t L, int sm_rows,
                             int64_t k, bool small_is_b, int smax, const DeviceInfo* di,
                             cudaStream_t st, bool* done) {
  *done = false;
  // (measured faster only for the 10-or-fewer short rows of a one-wave long
  // operand — the FCN's 10-class products: 1024 x 10 x 4096 13.5 vs 16.4 us,
  // 10 x 4096 x 1024 12.3 vs 14.3 us; for longer streams its one k-step per
  // butterfly makes it instruction-bound and the register kernel wins)
  if (!skinny_stream_enabled() || smax > 10 || L * k * 4 > kStreamMaxBytes) return MTNN_OK;
  int rc;
  switch (smax) {
    case 4: rc = launch_skinny_stream<4>(big, sml, C, L, sm_rows, k, small_is_b, di, st); break;
    case 8: rc = launch_skinny_stream<8>(big, sml, C, L, sm_rows, k, small_is_b, di, st); break;
    case 10: rc = launch_skinny_stream<10>(big, sml, C, L, sm_rows, k, small_is_b, di, st); break;
    case 12: rc = launch_skinny_stream<12>(big, sml, C, L, sm_rows, k, small_is_b, di, st); break;
    default: rc = launch_skinny_stream<16>(big, sml, C, L, sm_rows, k, small_is_b, di, st); break;
  }
  MTNN_TRY(rc);
  *done = true;
  return MTNN_OK;
}

#ifdef MTNN_TRACE
extern "C" int mtnn_skinny_trace(void* host, int64_t n) {
  MTNN_CUDA_TRY(cudaMemcpyFromSymbol(host, g_skinny_trace, (size_t)std::min<int64_t>(n, 8192 * 8) * 8));
  return MTNN_OK;
}
#endif

bool nn_smallk_eligible(const float* BT, const float* C, int64_t m, int64_t n, int64_t k) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return k >= 1 && k <= kNnSmallK && m >= 1 && n >= 4 && n % 4 == 0 && al16(BT) && al16(C) &&
         (n / 4 + 63) / 64 <= 0x7fffffff && (m + 4 * kNnRows - 1) / (4 * kNnRows) <= 65535;
}

int launch_gemm_nn_smallk(const float* A, const float* BT, float* C, int64_t m, int64_t n, int64_t k,
                          cudaStream_t s) {
  if (!nn_smallk_eligible(BT, C, m, n, k))
    return fail(MTNN_ENOTSUP, "small-k NN: shape (%lld, %lld, %lld) not eligible", (long long)m,
                (long long)n, (long long)k);
  KernelTimer timer(MTNN_KCLASS_GEMM_FFMA, 2.0 * (double)m * (double)n * (double)k, s);
  const dim3 grid((unsigned)((n / 4 + 63) / 64), (unsigned)((m + 4 * kNnRows - 1) / (4 * kNnRows)));
  int rc = MTNN_OK;
  auto go = [&](auto kern) { return launch_chained(kern, grid, dim3(256), 0, s, A, BT, C, m, n, (int)k); };
  switch (k) {
    case 1: rc = go(gemm_nn_smallk_kernel<1>); break;
    case 2: rc = go(gemm_nn_smallk_kernel<2>); break;
    case 3: rc = go(gemm_nn_smallk_kernel<3>); break;
    case 4: rc = go(gemm_nn_smallk_kernel<4>); break;
    case 5: rc = go(gemm_nn_smallk_kernel<5>); break;
    case 6: rc = go(gemm_nn_smallk_kernel<6>); break;
    case 7: rc = go(gemm_nn_smallk_kernel<7>); break;
    case 8: rc = go(gemm_nn_smallk_kernel<8>); break;
    case 9: rc = go(gemm_nn_smallk_kernel<9>); break;
    case 10: rc = go(gemm_nn_smallk_kernel<10>); break;
    case 11: rc = go(gemm_nn_smallk_kernel<11>); break;
    case 12: rc = go(gemm_nn_smallk_kernel<12>); break;
    case 13: rc = go(gemm_nn_smallk_kernel<13>); break;
    case 14: rc = go(gemm_nn_smallk_kernel<14>); break;
    case 15: rc = go(gemm_nn_smallk_kernel<15>); break;
    default: rc = go(gemm_nn_smallk_kernel<16>); break;
  }
  MTNN_TRY(rc);
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}

bool skinny_eligible(const float* A, const float* B, int64_t m, int64_t n, int64_t k) {
  const int64_t sm = std::min(m, n);
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return sm >= 1 && sm <= kSkinnyMax && k % 4 == 0 && k > 0 && al16(A) && al16(B);
}

int launch_gemm_skinny(const float* A, const float* B, float* C, int64_t m, int64_t n, int64_t k,
                       cudaStream_t s) {
  if (!skinny_eligible(A, B, m, n, k))
    return fail(MTNN_ENOTSUP, "skinny gemm: shape (%lld, %lld, %lld) not eligible", (long long)m,
                (long long)n, (long long)k);
  const DeviceInfo* di = nullptr;
  MTNN_TRY(device_info(&di));
  const bool small_is_b = n <= m;
  const int sm_rows = (int)(small_is_b ? n : m);
  const int64_t L = small_is_b ? m : n;
  // k slices per row group: 32 lanes x >= 4 k-steps of 16 bytes per slice
  int W = (int)std::min<int64_t>(8, std::max<int64_t>(1, k / 512));
  while (8 % W) --W;
  // SMAX = short rows the kernel is compiled for (registers: SMAX + R float4
  // loads and 32 sums per lane, <= 128 registers for 2 CTAs per SM)
  const int smax = sm_rows <= 4 ? 4 : sm_rows <= 8 ? 8 : sm_rows <= 10 ? 10 : sm_rows <= 12 ? 12 : 16;
  const int64_t rows_per_cta = (int64_t)(8 / W) * (32 / smax);
  const int64_t blocks = std::max<int64_t>(
      1, std::min<int64_t>((L + rows_per_cta - 1) / rows_per_cta, (int64_t)di->sm_count * 8));
  KernelTimer timer(MTNN_KCLASS_GEMM_FFMA, 2.0 * (double)m * (double)n * (double)k, s);
  const float* big = small_is_b ? A : B;
  const float* sml = small_is_b ? B : A;
  bool staged = false;
  MTNN_TRY(try_skinny_stream(big, sml, C, L, sm_rows, k, small_is_b, smax, di, s, &staged));
  if (staged) return MTNN_OK;
  MTNN_TRY(try_skinny_staged(big, sml, C, L, sm_rows, k, small_is_b, smax, di, s, &staged));
  if (staged) return MTNN_OK;
  const unsigned g = (unsigned)blocks;
  switch (smax) {
    case 4: MTNN_TRY(launch_chained(gemm_skinny_kernel<4>, dim3(g), dim3(256), 0, s, big, sml, C, L, sm_rows, k, small_is_b, W)); break;
    case 8: MTNN_TRY(launch_chained(gemm_skinny_kernel<8>, dim3(g), dim3(256), 0, s, big, sml, C, L, sm_rows, k, small_is_b, W)); break;
    case 10: MTNN_TRY(launch_chained(gemm_skinny_kernel<10>, dim3(g), dim3(256), 0, s, big, sml, C, L, sm_rows, k, small_is_b, W)); break;
    case 12: MTNN_TRY(launch_chained(gemm_skinny_kernel<12>, dim3(g), dim3(256), 0, s, big, sml, C, L, sm_rows, k, small_is_b, W)); break;
    default: MTNN_TRY(launch_chained(gemm_skinny_kernel<16>, dim3(g), dim3(256), 0, s, big, sml, C, L, sm_rows, k, small_is_b, W)); break;
  }
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}

}  // namespace mtnn
