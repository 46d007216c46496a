// CUDA IPC plumbing for the fused all-gather: each rank exports
// its C buffer once (handle + offset of the pointer inside its allocation, so
// tensors from PyTorch's caching allocator work), the other ranks open it and
// get a device pointer they can store to directly (NVLink peer writes on an
// NVSwitch node; the same mechanism also maps between processes sharing a GPU).
#include <cuda.h>
#include <cuda_runtime.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>

#include "common.h"

namespace mtnn {
namespace {

struct Opened {
  void* base = nullptr;
  int refs = 0;
};
std::mutex g_mu;
std::map<std::string, Opened> g_open;      // handle bytes -> mapping
std::map<void*, std::string> g_by_ptr;     // returned pointer -> handle key

using GetRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

int base_of(const void* p, void** base) {
  static GetRangeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<GetRangeFn>(f);
  });
  if (!fn) return fail(MTNN_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr b = 0;
  size_t size = 0;
  if (fn(&b, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
    return fail(MTNN_EINVAL, "pointer %p is not device memory", p);
  *base = reinterpret_cast<void*>(b);
  return MTNN_OK;
}

}  // namespace
}  // namespace mtnn

using namespace mtnn;

extern "C" {

int mtnn_ipc_handle(const void* ptr, unsigned char handle[64], int64_t* offset) {
  if (!ptr || !handle || !offset) return fail(MTNN_EINVAL, "null argument");
  void* base = nullptr;
  MTNN_TRY(base_of(ptr, &base));
  cudaIpcMemHandle_t h;
  MTNN_CUDA_TRY(cudaIpcGetMemHandle(&h, base));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &h, 64);
  *offset = static_cast<const char*>(ptr) - static_cast<const char*>(base);
  return MTNN_OK;
}

int mtnn_ipc_open(const unsigned char handle[64], int64_t offset, void** ptr) {
  if (!handle || !ptr || offset < 0) return fail(MTNN_EINVAL, "bad argument");
  const std::string key(reinterpret_cast<const char*>(handle), 64);
  std::lock_guard<std::mutex> lk(g_mu);
  Opened& o = g_open[key];
  if (o.refs == 0) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    cudaError_t e = cudaIpcOpenMemHandle(&o.base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      g_open.erase(key);
      return fail(MTNN_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    }
  }
  o.refs += 1;
  *ptr = static_cast<char*>(o.base) + offset;
  g_by_ptr[*ptr] = key;
  return MTNN_OK;
}

int mtnn_ipc_close(void* ptr) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_by_ptr.find(ptr);
  if (it == g_by_ptr.end()) return fail(MTNN_EINVAL, "pointer %p was not opened by mtnn_ipc_open", ptr);
  auto o = g_open.find(it->second);
  g_by_ptr.erase(it);
  if (o != g_open.end() && --o->second.refs == 0) {
    cudaError_t e = cudaIpcCloseMemHandle(o->second.base);
    g_open.erase(o);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      return fail(MTNN_ECUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    }
  }
  return MTNN_OK;
}

}  // extern "C"
