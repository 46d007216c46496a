// Topology probe: which SMs share an L2 partition (die) with which addresses.
// Each of the 148 CTAs (one per SM, forced by shared-memory size) records its
// %smid and the average L2-hit latency of a dependent pointer chase over a small
// ring of lines; rings start at different offsets to sample both partitions.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void probe(const uint32_t* __restrict__ ring, int nrings, int ring_len, int iters,
                      int* smid_out, float* lat_out) {
  extern __shared__ uint8_t pad[];
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) {
    smid_out[blockIdx.x] = smid;
    pad[0] = 0;
    for (int r = 0; r < nrings; ++r) {
      const uint32_t* base = ring + (size_t)r * ring_len * 32;
      uint32_t idx = 0;
      // warm
      for (int i = 0; i < ring_len; ++i) idx = __ldcg(base + idx * 32);
      long long t0 = clock64();
      for (int i = 0; i < iters; ++i) idx = __ldcg(base + idx * 32);
      long long t1 = clock64();
      lat_out[blockIdx.x * nrings + r] = (float)(t1 - t0) / iters + (idx == 12345678 ? 1.f : 0.f);
    }
  }
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nrings = 16, ring_len = 16, iters = 2000;
  std::vector<uint32_t> h((size_t)nrings * ring_len * 32, 0);
  for (int r = 0; r < nrings; ++r)
    for (int i = 0; i < ring_len; ++i)  // each ring: lines 128 B apart, 4 KiB stride between rings' lines
      h[((size_t)r * ring_len + i) * 32] = (i + 1) % ring_len;
  uint32_t* d;
  cudaMalloc(&d, h.size() * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  int* smid; float* lat;
  cudaMalloc(&smid, sms * 4); cudaMalloc(&lat, sms * nrings * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  probe<<<sms, 32, 200 * 1024>>>(d, nrings, ring_len, iters, smid, lat);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<int> hs(sms); std::vector<float> hl(sms * nrings);
  cudaMemcpy(hs.data(), smid, sms * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hl.data(), lat, sms * nrings * 4, cudaMemcpyDeviceToHost);
  printf("block smid lat[ring0..%d]\n", nrings - 1);
  for (int b = 0; b < sms; ++b) {
    printf("%d %d", b, hs[b]);
    for (int r = 0; r < nrings; ++r) printf(" %.0f", hl[b * nrings + r]);
    printf("\n");
  }
  return 0;
}
