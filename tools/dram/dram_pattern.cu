// DRAM access-pattern microbenchmark: the GEMM's TMA boxes (128 rows x 64 B, row
// pitch 2k bytes, walking k) vs the same bytes as contiguous 8 KiB bulk copies.
// One persistent CTA per SM streams panels through a 6-deep mbarrier ring; no
// compute. Prints GB/s per variant (run it on an idle GPU).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  uint32_t d = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(d) : "r"(bar), "r"(ph) : "memory");
  } while (!d);
}
constexpr int kDepth = 6, kBox = 8192;

// mode 0: 2D TMA boxes {32 halves, 128 rows} of a [rows][k] fp16 matrix, panel p = rows 128p..,
//         k-blocks walked in order (the GEMM's operand stream)
// mode 1: contiguous 8 KiB chunks, same total bytes, same per-CTA order
__global__ void __launch_bounds__(32, 1) stream_kernel(const __grid_constant__ CUtensorMap map,
                                                       const uint8_t* base, int panels, int kblocks,
                                                       int mode, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t buf[];
  __shared__ __align__(8) uint64_t bar[kDepth];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < kDepth; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long long total = (long long)panels * kblocks;
  long long issued = 0, done = 0;
  unsigned long long acc = 0;
  auto issue = [&](long long j) {
    const int slot = (int)(j % kDepth);
    const long long g = blockIdx.x + j * gridDim.x;  // this CTA's j-th box
    if (g >= total) return false;
    const int p = (int)(g / kblocks), kb = (int)(g % kblocks);
    const uint32_t b = s32(&bar[slot]), d = s32(buf + slot * kBox);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kBox) : "memory");
    if (mode == 0) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(d), "l"((uint64_t)&map), "r"(b), "r"(kb * 32), "r"(p * 128) : "memory");
    } else {
      const uint8_t* src = base + ((long long)p * kblocks + kb) * kBox;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(d), "l"(src), "r"(kBox), "r"(b) : "memory");
    }
    return true;
  };
  while (issued < kDepth && issue(issued)) ++issued;
  while (done < issued) {
    const int slot = (int)(done % kDepth);
    wait(s32(&bar[slot]), (uint32_t)((done / kDepth) & 1));
    acc += buf[slot * kBox];
    ++done;
    if (issue(issued)) ++issued;
  }
  sink[blockIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long rows = 16384, k = 16384;  // fp16 [rows][k] = 512 MiB
  const size_t bytes = rows * k * 2;
  uint8_t* d;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, sms * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows}, str[1] = {(cuuint64_t)k * 2};
  cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
  ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDepth * kBox);
  const int panels = (int)(rows / 128), kblocks = (int)(k / 32);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep)
    for (int mode = 0; mode < 2; ++mode) {
      for (int w = 0; w < 2; ++w) stream_kernel<<<sms, 32, kDepth * kBox>>>(map, d, panels, kblocks, mode, sink);
      cudaEventRecord(a);
      const int iters = 10;
      for (int it = 0; it < iters; ++it) stream_kernel<<<sms, 32, kDepth * kBox>>>(map, d, panels, kblocks, mode, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("mode %d (%s): %.0f GB/s\n", mode, mode ? "contiguous 8 KiB bulk" : "2D TMA 128 rows x 64 B",
             (double)bytes * iters / (ms * 1e-3) / 1e9);
    }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
