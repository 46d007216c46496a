// Out-of-place FP32 transpose, BT[j, i] = B[i, j] — the TNN path's first half.
//
// Reference: kernels/_numba_impl.py:169-182 (`transpose_oop`: 32x32 tiles, the
// inner loop writes a contiguous run of the output row, strided reads). It is a
// pure copy, so the result is bit-exact by construction; every element moves as
// a 32-bit word (uint32/uint4), never through FP arithmetic, so NaN payloads and
// -0.0 survive.
//
// B200 design (HBM-bound: 8 bytes of DRAM traffic per element, 4 read + 4 write):
//   * 64x64-element tiles staged through 16 KiB of shared memory;
//   * 128-bit global loads and stores (LDG.128/STG.128), each warp touching
//     256 contiguous bytes per row on both sides;
//   * the 4x4 sub-block each thread loads is transposed in registers, so shared
//     memory traffic is 128-bit too, with an XOR swizzle on the 16-byte column
//     index that makes both the STS.128 and LDS.128 phases conflict-free;
//   * all four loads of a thread are issued before any use (16 KiB in flight per
//     CTA, 8 CTAs per SM) to cover HBM latency;
//   * a 1-D grid over tiles, so any shape up to 2^31 tiles launches.
// Shapes whose rows are not 16-byte multiples (cols % 4 or rows % 4 != 0, or
// unaligned base pointers) take a 4-byte-word 64x64 padded-tile kernel instead
// (32x32 below 64 rows or columns).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.h"
#include "pdl.h"

namespace mtnn {
namespace {

constexpr int kTile = 64;         // tile edge in elements
constexpr int kVecPerRow = 16;    // 64 floats = 16 x 16-byte vectors
constexpr int kThreads = 256;

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void stg_stream(uint4* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// rows, cols multiples of 4; in/out 16-byte aligned.
__global__ void __launch_bounds__(kThreads)
transpose_vec4_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                      int64_t rows, int64_t cols, int64_t tiles_c) {
  pdl_enter();
  // smem[r][v]: output-tile row r (= input column), 16-byte column v^swz(r).
  __shared__ uint4 smem[kTile][kVecPerRow];

  const int64_t tile = blockIdx.x;
  const int64_t tr = tile / tiles_c;  // tile row (input rows)
  const int64_t tc = tile - tr * tiles_c;
  const int64_t r0 = tr * kTile, c0 = tc * kTile;

  const int t = threadIdx.x;
  const int cv = t % kVecPerRow;      // input 16-byte column within the tile
  const int rg = t / kVecPerRow;      // input row group (4 rows) within the tile
  const int64_t gc = c0 + 4 * cv;     // global input column of this vector
  const int64_t gr = r0 + 4 * rg;     // first global input row of this group

  uint4 v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = gr + i;
    if (r < rows && gc < cols)
      v[i] = ldg_stream(reinterpret_cast<const uint4*>(in + r * cols + gc));
    else
      v[i] = make_uint4(0, 0, 0, 0);
  }
  // Register 4x4 transpose: w[j] = column (gc + j) over rows gr..gr+3.
  uint4 w[4];
  w[0] = make_uint4(v[0].x, v[1].x, v[2].x, v[3].x);
  w[1] = make_uint4(v[0].y, v[1].y, v[2].y, v[3].y);
  w[2] = make_uint4(v[0].z, v[1].z, v[2].z, v[3].z);
  w[3] = make_uint4(v[0].w, v[1].w, v[2].w, v[3].w);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int orow = 4 * cv + j;            // output-tile row
    const int ocol = rg ^ (orow >> 2);      // swizzled 16-byte column (= rg ^ cv)
    smem[orow][ocol & (kVecPerRow - 1)] = w[j];
  }
  __syncthreads();
  // Store phase: output rows c0 + orow, 16-byte columns r0/4 + ov.
  const int ov = t % kVecPerRow;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int orow = t / kVecPerRow + 16 * i;
    const int64_t go_r = c0 + orow;          // output row = input column
    const int64_t go_c = r0 + 4 * ov;        // output column = input row
    const uint4 val = smem[orow][(ov ^ (orow >> 2)) & (kVecPerRow - 1)];
    if (go_r < cols && go_c < rows)
      stg_stream(reinterpret_cast<uint4*>(out + go_r * rows + go_c), val);
  }
}

// Generic fallback: 32x32 tile, padded smem, 4-byte accesses, any shape.
__global__ void __launch_bounds__(256)
transpose_scalar_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                        int64_t rows, int64_t cols, int64_t tiles_c) {
  pdl_enter();
  __shared__ uint32_t smem[32][33];
  const int64_t tile = blockIdx.x;
  const int64_t tr = tile / tiles_c;
  const int64_t tc = tile - tr * tiles_c;
  const int64_t r0 = tr * 32, c0 = tc * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + ty + 8 * i, c = c0 + tx;
    if (r < rows && c < cols) smem[ty + 8 * i][tx] = in[r * cols + c];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t orow = c0 + ty + 8 * i, ocol = r0 + tx;
    if (orow < cols && ocol < rows) out[orow * rows + ocol] = smem[tx][ty + 8 * i];
  }
}

// Fallback for rows/cols that are not 16-byte multiples: 64x64 tiles of 4-byte
// words, 16 loads per thread issued before any use (16 KiB in flight per CTA),
// padded shared memory; each warp still reads and writes 128 contiguous bytes
// per row. Used for odd shapes of the transpose sweep (e.g. 4097 x 1023).
__global__ void __launch_bounds__(256)
transpose_scalar64_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                          int64_t rows, int64_t cols, int64_t tiles_c) {
  pdl_enter();
  __shared__ uint32_t smem[64][65];
  const int64_t tile = blockIdx.x;
  const int64_t tr = tile / tiles_c;
  const int64_t tc = tile - tr * tiles_c;
  const int64_t r0 = tr * 64, c0 = tc * 64;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
  uint32_t v[16];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t r = r0 + ty + 8 * i, c = c0 + tx + 32 * h;
      v[2 * i + h] = (r < rows && c < cols) ? __ldg(in + r * cols + c) : 0u;
    }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) smem[ty + 8 * i][tx + 32 * h] = v[2 * i + h];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t orow = c0 + ty + 8 * i, ocol = r0 + tx + 32 * h;
      if (orow < cols && ocol < rows) out[orow * rows + ocol] = smem[tx + 32 * h][ty + 8 * i];
    }
}

}  // namespace

int launch_transpose(const float* in, float* out, int64_t rows, int64_t cols,
                     cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return MTNN_OK;
  const bool vec = (rows % 4 == 0) && (cols % 4 == 0) &&
                   (reinterpret_cast<uintptr_t>(in) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  KernelTimer timer(MTNN_KCLASS_TRANSPOSE, 8.0 * (double)rows * (double)cols, s);
  if (vec) {
    const int64_t tiles_r = (rows + kTile - 1) / kTile;
    const int64_t tiles_c = (cols + kTile - 1) / kTile;
    const int64_t tiles = tiles_r * tiles_c;
    if (tiles > 0x7fffffffLL) return fail(MTNN_EINVAL, "transpose: matrix too large");
    MTNN_TRY(launch_chained(transpose_vec4_kernel, dim3((unsigned)tiles), dim3(kThreads), 0, s,
                            reinterpret_cast<const uint32_t*>(in), reinterpret_cast<uint32_t*>(out),
                            rows, cols, tiles_c));
  } else if (rows >= 64 && cols >= 64) {
    const int64_t tiles_r = (rows + 63) / 64;
    const int64_t tiles_c = (cols + 63) / 64;
    const int64_t tiles = tiles_r * tiles_c;
    if (tiles > 0x7fffffffLL) return fail(MTNN_EINVAL, "transpose: matrix too large");
    MTNN_TRY(launch_chained(transpose_scalar64_kernel, dim3((unsigned)tiles), dim3(256), 0, s,
                            reinterpret_cast<const uint32_t*>(in), reinterpret_cast<uint32_t*>(out),
                            rows, cols, tiles_c));
  } else {
    const int64_t tiles_r = (rows + 31) / 32;
    const int64_t tiles_c = (cols + 31) / 32;
    const int64_t tiles = tiles_r * tiles_c;
    if (tiles > 0x7fffffffLL) return fail(MTNN_EINVAL, "transpose: matrix too large");
    MTNN_TRY(launch_chained(transpose_scalar_kernel, dim3((unsigned)tiles), dim3(256), 0, s,
                            reinterpret_cast<const uint32_t*>(in), reinterpret_cast<uint32_t*>(out),
                            rows, cols, tiles_c));
  }
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}

}  // namespace mtnn

namespace mtnn {
namespace {
// rows x width floats from a dense device block to host-mapped pinned memory
// rows `pitch` floats apart: SM-driven PCIe writes (A/B against the copy
// engine's 2-D D2H in the blocked host pipeline, MTNN_PIPE_ZC=1)
__global__ void __launch_bounds__(256) store_rows_kernel(const float4* __restrict__ src, float4* dst,
                                                         int64_t rows, int64_t w4, int64_t p4) {
  const int64_t n4 = rows * w4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const int64_t r = i / w4, c = i - r * w4;
    dst[r * p4 + c] = __ldcs(src + i);
  }
}
}  // namespace

int launch_store_rows(const float* src, float* dst, int64_t rows, int64_t width, int64_t pitch,
                      cudaStream_t s) {
  if (rows <= 0 || width <= 0) return MTNN_OK;
  if (width % 4 || pitch % 4 || (reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15))
    return fail(MTNN_EINVAL, "store_rows: 16-byte rows required");
  store_rows_kernel<<<64, 256, 0, s>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), rows,
                                       width / 4, pitch / 4);
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}
}  // namespace mtnn
