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
// 10-class layer and its weight gradient, batch-1 products): the long operand
// (L x k) is read from DRAM once and the product is bound by how much of it is
// in flight. One CTA per SM (512 threads), each owning a contiguous block of
// long rows; a row's k is split over the CTA's 16 warps when the block has few
// rows (1024 x 4096: 7 rows, 2 warps per row), else each warp walks whole rows.
// A lane issues U 16-byte long-operand loads before using any of them (U x 32
// x 16 warps = 64 KiB in flight per SM), then runs s four-term FFMA chains per
// piece against the short operand (L1/L2-resident, shared by the CTA's warps).
// Sums fold across lanes by shuffles and across a row's warps through shared
// memory in a fixed order (deterministic). Output (long row r, short row j)
// goes to C[r * s + j] when the short side is B, C[j * L + r] when it is A.
// (Round 1 ran one CTA per 3 rows: 1.16 waves of latency-bound CTAs, 15.8 us
// for 1024 x 10 x 4096.)
constexpr int kSkinnyMax = 16;
constexpr int kSkinnyWarps = 16;
constexpr int kSkinnyU = 8;

template <int SMAX>
__global__ void __launch_bounds__(32 * kSkinnyWarps, 1)
gemm_skinny_kernel(const float* __restrict__ big, const float* __restrict__ small,
                   float* __restrict__ C, int64_t L, int s, int64_t k, int64_t rows_per_cta,
                   bool small_is_b) {
  pdl_enter();
  __shared__ float part[kSkinnyWarps][SMAX];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t row0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t rows = min(rows_per_cta, L - row0);
  if (rows <= 0) return;
  const int64_t k4 = k / 4;
  // warps per row (k-parts) when the block is short, else rows per warp
  const int wpr = rows >= kSkinnyWarps ? 1 : kSkinnyWarps / (int)rows;
  const int64_t per = (k4 + wpr - 1) / wpr;  // 16-byte pieces per k-part
  const float4* big4 = reinterpret_cast<const float4*>(big);
  const float4* small4 = reinterpret_cast<const float4*>(small);
  const int64_t task_count = rows * wpr;
  const int tasks = task_count < kSkinnyWarps ? (int)task_count : kSkinnyWarps;
  for (int64_t rbase = 0; rbase < rows; rbase += kSkinnyWarps / wpr) {
    float acc[SMAX];
#pragma unroll
    for (int j = 0; j < SMAX; ++j) acc[j] = 0.f;
    const int64_t rr = rbase + warp / wpr;  // this warp's row (block-relative)
    const int part_k = warp % wpr;
    const bool active = warp < tasks && rr < rows;
    if (active) {
      const int64_t qb0 = (int64_t)part_k * per, qb1 = min(k4, qb0 + per);
      const float4* arow = big4 + (row0 + rr) * k4;
      for (int64_t qb = qb0; qb < qb1; qb += 32 * kSkinnyU) {
        float4 a[kSkinnyU];
#pragma unroll
        for (int u = 0; u < kSkinnyU; ++u) {
          const int64_t q = qb + lane + 32 * u;
          a[u] = q < qb1 ? __ldg(arow + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kSkinnyU; ++u) {
          const int64_t q = qb + lane + 32 * u;
          if (q >= qb1) break;
#pragma unroll
          for (int j = 0; j < SMAX; ++j) {
            if (j >= s) break;
            const float4 b = __ldg(small4 + (int64_t)j * k4 + q);
            acc[j] = fmaf(a[u].w, b.w, fmaf(a[u].z, b.z, fmaf(a[u].y, b.y, fmaf(a[u].x, b.x, acc[j]))));
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < SMAX; ++j)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < SMAX; ++j) part[warp][j] = acc[j];
    }
    __syncthreads();
    // the first warp of each row adds its row's k-parts in order and stores
    if (active && part_k == 0 && lane < s) {
      float sum = part[warp][lane];
      for (int w = 1; w < wpr; ++w) sum += part[warp + w][lane];
      const int64_t row = row0 + rr;
      C[small_is_b ? row * s + lane : (int64_t)lane * L + row] = sum;
    }
    __syncthreads();  // part is reused by the next rows
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

int launch_splitk_reduce(const float* part, float* C, int64_t count, int splits,
                         cudaStream_t s) {
  const DeviceInfo* di = nullptr;
  MTNN_TRY(device_info(&di));
  int64_t blocks = (count + 255) / 256;
  blocks = std::min<int64_t>(blocks, (int64_t)di->sm_count * 8);
  KernelTimer timer(MTNN_KCLASS_REDUCE, 4.0 * (double)(splits + 1) * (double)count, s);
  MTNN_TRY(launch_chained(splitk_reduce_kernel, dim3((unsigned)std::max<int64_t>(blocks, 1)),
                          dim3(256), 0, s, part, C, count, splits));
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
  // one CTA per SM, contiguous row blocks
  const int64_t rows_per_cta = (L + di->sm_count - 1) / di->sm_count;
  const int64_t blocks = (L + rows_per_cta - 1) / rows_per_cta;
  KernelTimer timer(MTNN_KCLASS_GEMM_FFMA, 2.0 * (double)m * (double)n * (double)k, s);
  const float* big = small_is_b ? A : B;
  const float* sml = small_is_b ? B : A;
  const dim3 g((unsigned)blocks), blk(32 * kSkinnyWarps);
  const int smax = sm_rows <= 4 ? 4 : sm_rows <= 8 ? 8 : sm_rows <= 10 ? 10 : sm_rows <= 12 ? 12 : 16;
  switch (smax) {
    case 4: MTNN_TRY(launch_chained(gemm_skinny_kernel<4>, g, blk, 0, s, big, sml, C, L, sm_rows, k, rows_per_cta, small_is_b)); break;
    case 8: MTNN_TRY(launch_chained(gemm_skinny_kernel<8>, g, blk, 0, s, big, sml, C, L, sm_rows, k, rows_per_cta, small_is_b)); break;
    case 10: MTNN_TRY(launch_chained(gemm_skinny_kernel<10>, g, blk, 0, s, big, sml, C, L, sm_rows, k, rows_per_cta, small_is_b)); break;
    case 12: MTNN_TRY(launch_chained(gemm_skinny_kernel<12>, g, blk, 0, s, big, sml, C, L, sm_rows, k, rows_per_cta, small_is_b)); break;
    default: MTNN_TRY(launch_chained(gemm_skinny_kernel<16>, g, blk, 0, s, big, sml, C, L, sm_rows, k, rows_per_cta, small_is_b)); break;
  }
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}

}  // namespace mtnn
