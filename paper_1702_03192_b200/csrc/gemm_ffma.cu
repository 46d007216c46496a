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
