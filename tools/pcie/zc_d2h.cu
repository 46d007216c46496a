// Device->host bandwidth: copy-engine D2H vs SM-driven stores into mapped
// pinned host memory, contiguous and 2-D (6 KB rows at a 24 KB pitch: the
// blocked host pipeline's C column blocks), alone / beside an HBM-bound kernel /
// beside an H2D copy (duplex).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zc_d2h zc_d2h.cu -lcublas
#include <cstdio>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cuda_bf16.h>

// rows x width4 float4 from a dense source to dst rows `pitch4` apart
__global__ void zc_copy2d(const float4* __restrict__ src, float4* dst, size_t rows, size_t width4,
                          size_t pitch4) {
  const size_t n4 = rows * width4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const size_t r = i / width4, c = i - r * width4;
    dst[r * pitch4 + c] = __ldcs(src + i);
  }
}
__global__ void hbm_copy(const float4* __restrict__ src, float4* __restrict__ dst, size_t n4, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) dst[i] = src[i];
}

int main() {
  const size_t bytes = 256ull << 20;
  float4 *d, *h, *hin, *din, *x, *y;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 1, bytes);
  cudaMalloc(&din, bytes);
  cudaHostAlloc(&h, bytes * 4, cudaHostAllocDefault);  // (pitch room for 2-D)
  cudaHostAlloc(&hin, bytes, cudaHostAllocDefault);
  const size_t hb = 1ull << 30;
  cudaMalloc(&x, hb); cudaMalloc(&y, hb);
  cudaStream_t s1, s2, s3;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking);
  cudaEvent_t a, b, c0, c1;
  cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c0); cudaEventCreate(&c1);
  const size_t width = 6144, pitch = 24576, rows = bytes / width;  // (a 24 KB pitch keeps the pinned buffer at 1 GB)
  cublasHandle_t hbl;
  cublasCreate(&hbl);
  cublasSetStream(hbl, s2);
  const int G = 8192;
  __nv_bfloat16 *ga, *gb, *gc;
  cudaMalloc(&ga, (size_t)G * G * 2); cudaMalloc(&gb, (size_t)G * G * 2); cudaMalloc(&gc, (size_t)G * G * 2);
  cudaMemset(ga, 0, (size_t)G * G * 2); cudaMemset(gb, 0, (size_t)G * G * 2);
  const float one = 1.f, zero = 0.f;
  auto gemms = [&](int n) {
    for (int i = 0; i < n; ++i)
      cublasGemmEx(hbl, CUBLAS_OP_N, CUBLAS_OP_N, G, G, G, &one, ga, CUDA_R_16BF, G, gb, CUDA_R_16BF, G, &zero,
                   gc, CUDA_R_16BF, G, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  };
  gemms(2);
  const char* loads[] = {"alone", "beside HBM copy", "beside H2D (duplex)", "beside bf16 GEMMs"};
  for (int load = 0; load < 4; ++load)
    for (int two_d = 0; two_d < 2; ++two_d)
      for (int mode = 0; mode < 3; ++mode) {
        const int grids[] = {0, 32, 148};
        cudaDeviceSynchronize();
        if (load == 1) hbm_copy<<<148 * 4, 256, 0, s2>>>(x, y, hb / 16, 40);
        if (load == 3) gemms(30);
        if (load == 2) {
          cudaEventRecord(c0, s3);
          for (int r = 0; r < 3; ++r) cudaMemcpyAsync(din, hin, bytes, cudaMemcpyHostToDevice, s3);
          cudaEventRecord(c1, s3);
        }
        cudaEventRecord(a, s1);
        for (int r = 0; r < 3; ++r) {
          if (mode == 0) {
            if (two_d) cudaMemcpy2DAsync(h, pitch, d, width, width, rows, cudaMemcpyDeviceToHost, s1);
            else cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s1);
          } else if (two_d) {
            zc_copy2d<<<grids[mode], 256, 0, s1>>>(d, h, rows, width / 16, pitch / 16);
          } else {
            zc_copy2d<<<grids[mode], 256, 0, s1>>>(d, h, 1, bytes / 16, 0);
          }
        }
        cudaEventRecord(b, s1);
        cudaDeviceSynchronize();
        float ms = 0, ms2 = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (load == 2) cudaEventElapsedTime(&ms2, c0, c1);
        printf("%-20s %s %-16s grid %3d: D2H %6.1f GB/s", loads[load], two_d ? "2-D 6KB rows" : "contiguous  ",
               mode == 0 ? "copy engine" : "SM stores", grids[mode], 3.0 * bytes / ms / 1e6);
        if (load == 2) printf("   H2D %6.1f GB/s", 3.0 * bytes / ms2 / 1e6);
        printf("\n");
      }
  // the blocked pipeline's pattern: C column blocks of 4096 rows x 6 KB into a
  // 16384-wide row-major C (64 KB pitch), ten blocks side by side, alone and
  // beside ten 25 MB H2D copies
  {
    const size_t bw = 6144, bp = 65536, br = 4096;
    float4* hc;
    cudaHostAlloc(&hc, br * bp, cudaHostAllocDefault);
    for (int duplex = 0; duplex < 2; ++duplex)
      for (int mode = 0; mode < 2; ++mode) {
        cudaDeviceSynchronize();
        if (duplex) {
          cudaEventRecord(c0, s3);
          for (int j = 0; j < 10; ++j)
            cudaMemcpyAsync(reinterpret_cast<char*>(din) + j * br * bw, reinterpret_cast<char*>(hin) + j * br * bw,
                            br * bw, cudaMemcpyHostToDevice, s3);
          cudaEventRecord(c1, s3);
        }
        cudaEventRecord(a, s1);
        for (int j = 0; j < 10; ++j) {
          char* dst = reinterpret_cast<char*>(hc) + j * bw;
          const char* src = reinterpret_cast<const char*>(d) + j * br * bw;
          if (mode == 0) cudaMemcpy2DAsync(dst, bp, src, bw, bw, br, cudaMemcpyDeviceToHost, s1);
          else zc_copy2d<<<64, 256, 0, s1>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst),
                                             br, bw / 16, bp / 16);
        }
        cudaEventRecord(b, s1);
        cudaDeviceSynchronize();
        float ms = 0, ms2 = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (duplex) cudaEventElapsedTime(&ms2, c0, c1);
        printf("pipeline pattern %-8s %-12s: D2H %6.1f GB/s", duplex ? "duplex" : "alone", mode ? "SM stores" : "copy engine",
               10.0 * br * bw / ms / 1e6);
        if (duplex) printf("   H2D %6.1f GB/s", 10.0 * br * bw / ms2 / 1e6);
        printf("\n");
      }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
