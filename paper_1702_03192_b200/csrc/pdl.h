// Programmatic dependent launch shared by the SIMT kernels (splits, skinny and
// FFMA GEMMs, transposes, split-K reduction): each is launched with
// programmatic stream serialization and executes launch_dependents on entry and
// wait before its first read, so consecutive kernels of one call — and of
// consecutive calls — overlap launch latency and prologues without reordering
// any memory access. MTNN_PDL=0 launches everything fully serialised.
#pragma once

#include <cuda_runtime.h>
#include <stdlib.h>

#include "common.h"

namespace mtnn {

__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

inline bool chain_enabled() {
  static const bool on = [] {
    const char* e = getenv("MTNN_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class Kern, class... Args>
int launch_chained(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = chain_enabled() ? 1 : 0;
  MTNN_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, args...));
  return MTNN_OK;
}

}  // namespace mtnn
