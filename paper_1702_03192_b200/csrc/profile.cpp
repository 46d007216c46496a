// Kernel timing instrumentation for the benchmark (mtnn_profile_*; see
// include/mtnn_b200.h). Event pairs are recorded on the launch stream — the
// only way to time one kernel inside a stream of library launches — and
// resolved lazily in mtnn_profile_read, so recording never blocks the host.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "common.h"

namespace mtnn {
namespace {

struct Pending {
  int kclass;
  double work;
  cudaEvent_t start, stop;
};

std::atomic<unsigned> g_mask{0};  // bit c: time kernel class c
std::atomic<bool> g_counting{false};  // count launches and work of every class
std::atomic<double> g_min_work{0.0};  // time only launches with at least this much work
std::atomic<int> g_sample_every{1};   // of those, time every n-th (a rotating sample)
std::atomic<uint64_t> g_eligible{0};  // launches that passed the class and work filters
std::mutex g_mu;
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_free_events;
double g_ms[MTNN_KCLASS_COUNT];
int64_t g_launches[MTNN_KCLASS_COUNT];
double g_work[MTNN_KCLASS_COUNT];
int64_t g_timed_launches[MTNN_KCLASS_COUNT];  // the launches behind g_ms
double g_timed_work[MTNN_KCLASS_COUNT];

cudaEvent_t take_event() {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_free_events.empty()) {
      cudaEvent_t e = g_free_events.back();
      g_free_events.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  return e;
}

}  // namespace

KernelTimer::KernelTimer(int kc, double w, cudaStream_t s) : kclass(kc), work(w), stream(s) {
  if (!g_counting.load(std::memory_order_relaxed)) return;
  {
    std::lock_guard<std::mutex> lk(g_mu);  // every launch is counted while profiling
    g_launches[kc] += 1;
    g_work[kc] += w;
  }
  if (!((g_mask.load(std::memory_order_relaxed) >> kc) & 1u)) return;
  if (w < g_min_work.load(std::memory_order_relaxed)) return;
  const int every = g_sample_every.load(std::memory_order_relaxed);
  if (g_eligible.fetch_add(1, std::memory_order_relaxed) % (uint64_t)(every > 0 ? every : 1) != 0)
    return;
  start = take_event();
  if (start && cudaEventRecord(start, stream) != cudaSuccess) {
    (void)cudaGetLastError();
    start = nullptr;
  }
}

KernelTimer::~KernelTimer() {
  if (!start) return;
  cudaEvent_t stop = take_event();
  if (!stop || cudaEventRecord(stop, stream) != cudaSuccess) {
    (void)cudaGetLastError();
    return;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_pending.push_back({kclass, work, start, stop});
}

}  // namespace mtnn

using namespace mtnn;

extern "C" {

int mtnn_profile_trace(void* buf, int64_t ctas) {
  if (buf && ctas <= 0) return fail(MTNN_EINVAL, "trace buffer needs ctas > 0");
  return set_gemm_trace(buf, buf ? ctas : 0);
}

int mtnn_profile_enable(int on) {
  g_mask.store(on ? (1u << MTNN_KCLASS_COUNT) - 1u : 0u);
  g_counting.store(on != 0);
  return MTNN_OK;
}

int mtnn_profile_enable_classes(unsigned mask) {
  g_mask.store(mask & ((1u << MTNN_KCLASS_COUNT) - 1u));
  g_counting.store(true);
  return MTNN_OK;
}

int mtnn_profile_min_work(double work) {
  g_min_work.store(work > 0.0 ? work : 0.0);
  return MTNN_OK;
}

int mtnn_profile_sample_every(int n) {
  if (n < 1) return fail(MTNN_EINVAL, "sample period must be >= 1, got %d", n);
  g_sample_every.store(n);
  g_eligible.store(0);
  return MTNN_OK;
}

int mtnn_profile_read_timed(int kclass, double* total_ms, int64_t* launches, double* work) {
  MTNN_TRY(mtnn_profile_read(kclass, nullptr, nullptr, nullptr));  // resolves pending events
  std::lock_guard<std::mutex> lk(g_mu);
  if (total_ms) *total_ms = g_ms[kclass];
  if (launches) *launches = g_timed_launches[kclass];
  if (work) *work = g_timed_work[kclass];
  return MTNN_OK;
}

int mtnn_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& p : g_pending) {
    (void)cudaEventSynchronize(p.stop);
    g_free_events.push_back(p.start);
    g_free_events.push_back(p.stop);
  }
  g_pending.clear();
  for (int i = 0; i < MTNN_KCLASS_COUNT; ++i) {
    g_ms[i] = g_work[i] = g_timed_work[i] = 0.0;
    g_launches[i] = g_timed_launches[i] = 0;
  }
  (void)cudaGetLastError();
  return MTNN_OK;
}

int mtnn_profile_read(int kclass, double* total_ms, int64_t* launches, double* work) {
  if (kclass < 0 || kclass >= MTNN_KCLASS_COUNT)
    return fail(MTNN_EINVAL, "unknown kernel class %d", kclass);
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& p : g_pending) {
    float ms = 0.f;
    cudaError_t e = cudaEventSynchronize(p.stop);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, p.start, p.stop);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      return fail(MTNN_ECUDA, "profile event: %s", cudaGetErrorString(e));
    }
    g_ms[p.kclass] += ms;
    g_timed_launches[p.kclass] += 1;
    g_timed_work[p.kclass] += p.work;
    g_free_events.push_back(p.start);
    g_free_events.push_back(p.stop);
  }
  g_pending.clear();
  if (total_ms) *total_ms = g_ms[kclass];
  if (launches) *launches = g_launches[kclass];
  if (work) *work = g_work[kclass];
  return MTNN_OK;
}

}  // extern "C"
