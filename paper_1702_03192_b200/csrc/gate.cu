// Host-released stream gate (measurement support; include/mtnn_b200.h).
//
// A benchmark that times one call with CUDA events on its stream opens the
// window (event), enqueues the call, closes it (event) — and if the host stalls
// while enqueueing (a page fault, the GIL, a first-use allocation) the GPU sits
// idle inside the open window and the stall is counted as device time
// (tools/probes/probe_outliers.py: such windows are the bench's rare 10-100x
// outliers). mtnn_gate puts a one-thread kernel ahead of the window that spins
// until the host has written `value` into a flag in pinned host memory, i.e.
// until the whole call is enqueued; the window then holds device work only.
// The spin is bounded (1 s of %globaltimer) so a forgotten release cannot hang
// the GPU.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.h"

namespace mtnn {
namespace {

__global__ void gate_kernel(const volatile int32_t* flag, int32_t value) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag < value) {
    __nanosleep(256);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 1000000000ull) break;
  }
}

}  // namespace
}  // namespace mtnn

using namespace mtnn;

extern "C" int mtnn_gate(const int32_t* host_flag, int32_t value, void* stream) {
  if (host_flag == nullptr) return fail(MTNN_EINVAL, "null gate flag");
  const DeviceInfo* di = nullptr;
  MTNN_TRY(device_info(&di));
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, host_flag) != cudaSuccess || attr.type != cudaMemoryTypeHost) {
    (void)cudaGetLastError();
    return fail(MTNN_EINVAL, "gate flag must be pinned (page-locked) host memory");
  }
  const int32_t* dflag = static_cast<const int32_t*>(attr.devicePointer);
  gate_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(dflag, value);
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}
