// Stream-ordered scratch allocations (cudaMallocAsync on the device's default
// memory pool, whose release threshold is raised once so freed blocks stay cached
// and steady-state calls do not touch the OS). The paper's TNN allocates and frees
// its B^T buffer inside the call (reference _numba_impl.py:16-19);
// stream ordering lets the free be issued right after the last kernel that reads it.
#pragma once

#include <cuda_runtime.h>

#include "common.h"

namespace mtnn {

int prepare_mempool();

struct ScratchBuffer {
  void* ptr = nullptr;
  cudaStream_t stream = nullptr;
  ScratchBuffer() = default;
  ScratchBuffer(const ScratchBuffer&) = delete;
  ScratchBuffer& operator=(const ScratchBuffer&) = delete;
  int alloc(size_t bytes, cudaStream_t s) {
    MTNN_TRY(prepare_mempool());
    stream = s;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&ptr, bytes, s);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      ptr = nullptr;
      if (e == cudaErrorMemoryAllocation)
        return fail(MTNN_ENOMEM, "device allocation of %zu bytes failed", bytes);
      return fail(MTNN_ECUDA, "cudaMallocAsync(%zu): %s", bytes, cudaGetErrorString(e));
    }
    return MTNN_OK;
  }
  void release() {
    if (ptr) (void)cudaFreeAsync(ptr, stream);
    ptr = nullptr;
  }
  ~ScratchBuffer() { release(); }
};

}  // namespace mtnn
