// Device-side cross-rank barrier for the fused all-gather.
//
// Every rank owns a small flag array `flags[world]` (uint32, device memory,
// exported with mtnn_ipc_handle and mapped by the other ranks). A barrier with
// epoch e is one single-warp kernel on the caller's stream:
//   lane j < npeers: st.release.sys  peer_flags[j][rank] = e
//   lane i < world, i != rank: spin ld.acquire.sys flags[i] >= e
// The release is cumulative, so everything the stream did before the barrier
// (the GEMM's peer TMA stores into the other ranks' C) is visible to a rank
// that has observed the flag; the acquire orders everything after the
// barrier on this stream behind the peers' pre-barrier work. Enqueued before
// and after mtnn_gemm_nt_allgather it keeps the whole exchange on the device:
// no host synchronisation, so the cross-rank completion sits inside the
// caller's timed CUDA-event window.
//
// A bounded spin (default 30 s, %globaltimer) turns a missing peer into an
// error word instead of a hung GPU: status[0] = 1 + the first rank not heard from.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.h"

namespace mtnn {
namespace {

struct PeerFlags {
  uint32_t* p[8];
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void peer_barrier_kernel(uint32_t* flags, PeerFlags peers, int npeers, int rank,
                                    int world, uint32_t epoch, uint32_t* status,
                                    uint64_t timeout_ns) {
  const int lane = threadIdx.x;
  if (lane < npeers) st_release_sys(peers.p[lane] + rank, epoch);
  if (lane < world && lane != rank) {
    const uint64_t t0 = globaltimer();
    // wrap-safe "flag has reached epoch"
    while (static_cast<int32_t>(ld_acquire_sys(flags + lane) - epoch) < 0) {
      if (globaltimer() - t0 > timeout_ns) {
        atomicCAS(status, 0u, static_cast<uint32_t>(lane + 1));
        break;
      }
      __nanosleep(64);
    }
  }
  __syncwarp();
}

}  // namespace
}  // namespace mtnn

using namespace mtnn;

extern "C" int mtnn_peer_barrier(uint32_t* flags, uint32_t* const* peer_flags, int npeers,
                                 int rank, int world, uint32_t epoch, uint32_t* status,
                                 double timeout_s, void* stream) {
  if (!flags || !status || (npeers > 0 && !peer_flags))
    return fail(MTNN_EINVAL, "null flag/status pointer");
  if (world < 1 || world > 8 || npeers != world - 1 || rank < 0 || rank >= world)
    return fail(MTNN_EINVAL, "bad world %d / rank %d / npeers %d (at most 8 ranks)", world, rank,
                npeers);
  PeerFlags pf = {};
  for (int j = 0; j < npeers; ++j) {
    if (!peer_flags[j]) return fail(MTNN_EINVAL, "null peer flag pointer %d", j);
    pf.p[j] = peer_flags[j];
  }
  const uint64_t timeout_ns =
      timeout_s > 0 ? static_cast<uint64_t>(timeout_s * 1e9) : 30ull * 1000000000ull;
  peer_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      flags, pf, npeers, rank, world, epoch, status, timeout_ns);
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}
