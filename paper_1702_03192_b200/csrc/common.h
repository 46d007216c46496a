// Shared host-side helpers for the MTNN B200 library: error state, status codes,
// CUDA checks. Everything here is host code; device code lives in the .cu files.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/mtnn_b200.h"
#include "fix.h"

namespace mtnn {

// Thread-local last error message (mtnn_last_error).
void set_error(const std::string& msg);
const std::string& last_error();

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));

#define MTNN_CUDA_TRY(expr)                                                        \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      (void)cudaGetLastError();                                                    \
      if (_e == cudaErrorMemoryAllocation)                                         \
        return ::mtnn::fail(MTNN_ENOMEM, "%s: %s", #expr, cudaGetErrorString(_e)); \
      return ::mtnn::fail(MTNN_ECUDA, "%s: %s", #expr, cudaGetErrorString(_e));    \
    }                                                                              \
  } while (0)

#define MTNN_TRY(expr)         \
  do {                         \
    int _rc = (expr);          \
    if (_rc != MTNN_OK) return _rc; \
  } while (0)

// Per-device facts cached at first use.
struct DeviceInfo {
  int device = -1;
  int sm_count = 0;
  int cc_major = 0, cc_minor = 0;
  int max_smem_optin = 0;
  int l2_bytes = 0;
  int clock_khz = 0;
  int bus_width = 0;
  size_t total_mem = 0;
};
// Returns MTNN_ENOTSUP when no sm_100-class device is current.
int device_info(const DeviceInfo** out);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute belongs to the device's context, so a process driving several
// GPUs must set it on each. Pass the kernel's largest launch size (later calls
// for the same kernel are no-ops).
int set_max_dynamic_smem(const void* kernel, int bytes);

// Kernel timing instrumentation (mtnn_profile_*): a scope records a CUDA event
// pair around one launch when profiling is enabled, else does nothing.
struct KernelTimer {
  KernelTimer(int kclass, double work, cudaStream_t s);
  ~KernelTimer();
  int kclass;
  double work;
  cudaStream_t stream;
  cudaEvent_t start = nullptr;
};

// Kernel launchers (implemented in the .cu files). All asynchronous on `s`.
int launch_store_rows(const float* src, float* dst, int64_t rows, int64_t width, int64_t pitch,
                      cudaStream_t s);
int launch_transpose(const float* in, float* out, int64_t rows, int64_t cols,
                     cudaStream_t s);
// SIMT NT for outputs with a side <= 16 (k % 4 == 0, 16-byte aligned operands).
// ENOTSUP otherwise.
bool skinny_eligible(const float* A, const float* B, int64_t m, int64_t n, int64_t k);
// NN with a tiny inner dimension (k <= 16): output-bound outer-product kernel.
bool nn_smallk_eligible(const float* BT, const float* C, int64_t m, int64_t n, int64_t k);
int launch_gemm_nn_smallk(const float* A, const float* BT, float* C, int64_t m, int64_t n, int64_t k,
                          cudaStream_t s);
int launch_gemm_skinny(const float* A, const float* B, float* C, int64_t m, int64_t n, int64_t k,
                       cudaStream_t s);
int launch_gemm_ffma(const float* A, const float* B, float* C, int64_t m, int64_t n,
                     int64_t k, bool b_is_nk, cudaStream_t s);
// Tensor-core FP32-accurate GEMMs (three MMAs per product on hi/lo operand halves).
// TF32: hi = raw fp32 (truncated to tf32 by the tensor core), lo = x - trunc(x).
// F16S: per-row power-of-two scaled fp16 hi/lo (split_f16.cu), 2x the MMA rate.
// b_is_nk: B stored n x k (NT); else B^T stored k x n (NN).
// Returns MTNN_ENOTSUP when the shape/alignment is ineligible.
enum class TcKind { TF32, F16S };
int launch_gemm_tc(const float* A, const float* B, float* C, int64_t m, int64_t n,
                   int64_t k, bool b_is_nk, TcKind kind, cudaStream_t s);
bool tc_eligible_operands(const float* A, const float* B, int64_t m, int64_t n, int64_t k,
                          bool b_is_nk, TcKind kind);
bool tc_eligible(const float* A, const float* B, const float* C, int64_t m, int64_t n,
                 int64_t k, bool b_is_nk, TcKind kind);
// Prepared (split) tensor-core operand: hi/lo halves, plus 1/scale per row for F16S.
struct TcOperand {
  const void* hi = nullptr;
  const void* lo = nullptr;
  // F16S 1/s: per row (K-major), or [ceil(k / kScaleChunkK)][n] for MN-major B^T
  const float* inv_scale = nullptr;
  FixList fix;  // residual entries of this operand (fix.h)
};
struct ScratchBuffer;
// inkernel: the operand is split inside the GEMM from its raw rows (hi = X,
// lo = nullptr); F16S then only computes the row scales (read-only pass).
// fh: receives the operand's residual list (fix.h; nullptr = no tracking); it
// must live until the fix-up (launch_fixup) that consumes it is enqueued.
struct FixHandle;
int tc_prepare(const float* X, int64_t rows, int64_t k, bool mn_major, TcKind kind,
               bool inkernel, ScratchBuffer& ws, FixHandle* fh, TcOperand* out, cudaStream_t s);
// Both operands of one GEMM; F16S with K-major B runs a single split launch.
int tc_prepare_pair(const float* A, int64_t m, const float* B, int64_t n, int64_t k,
                    bool b_mn_major, TcKind kind, int conv, ScratchBuffer& wa, ScratchBuffer& wb,
                    FixHandle* fa, FixHandle* fb, TcOperand* a, TcOperand* b, cudaStream_t s);
// Which operand (1 = A, 2 = B, 0 = none) the GEMM splits in-kernel for this shape.
int tc_inkernel_operand(int64_t m, int64_t n, bool b_is_nk, TcKind kind);
// Run-time knob (mtnn_config_set): largest output short side split in-kernel.
int64_t f16s_inkernel_max_short();
void set_f16s_inkernel_max_short(int64_t v);
// Run-time knob (mtnn_config_set "tc_pair"): 256 x 256 CTA-pair tiles for large NT.
int tc_pair_mode();  // 0 off, 1 large problems (default), 2 always when possible
void set_tc_pair_mode(int v);
// mtnn_profile_trace: phase timestamps of the single-CTA tensor-core kernel.
int set_gemm_trace(void* buf, int64_t ctas);
// ldc: C row stride in elements (-1 = n); a larger one pads each C row.
int tc_run(const TcOperand& a, const TcOperand& b, float* C, int64_t m, int64_t n, int64_t k,
           bool b_is_nk, TcKind kind, cudaStream_t s, int64_t ldc = -1);
// Row block of a row-sharded NT with the all-gather fused into the epilogue
// (peers: the same rows of other ranks' C buffers, mapped into this process).
int gemm_nt_allgather(const float* A, const float* B, float* C_local, float* const* peers,
                      int npeers, int64_t m, int64_t n, int64_t k, cudaStream_t s);
// The library's AUTO NT dispatch (mtnn_abi.cpp), for internal fallbacks.
int gemm_dispatch_nt(const float* A, const float* B, float* C, int64_t m, int64_t n, int64_t k,
                     cudaStream_t s);
// F16S operand splits. `fix` receives the operand's residual entries (fix.h;
// FixList{} = none). hiN == nullptr -> row scales (and residual check) only.
int launch_split_rows_f16(const float* x, void* hi, void* lo, float* inv_scale, int64_t rows,
                          int64_t k, const FixList& fix, cudaStream_t s);
// Both K-major operands of one GEMM in one launch: rows of x0 then x1 (same k).
int launch_split_rows_f16_pair(const float* x0, void* hi0, void* lo0, float* inv0, int64_t rows0,
                               const FixList& fix0, const float* x1, void* hi1, void* lo1,
                               float* inv1, int64_t rows1, const FixList& fix1, int64_t k,
                               cudaStream_t s);
// 1/s per row (s = split_rows_f16's power-of-two row scale), reading x only.
int launch_rowmax_f16(const float* x, float* inv_scale, int64_t rows, int64_t k,
                      const FixList& fix, cudaStream_t s);
// Rows of an MN-major (k x n) F16S operand that share one column scale: the
// column split writes inv_scale[ceil(k / kScaleChunkK)][n], and the GEMM applies
// chunk c's scale to its FP32-promotion chunks covering k rows [256c, 256c+256).
constexpr int kScaleChunkK = 256;
// Optionally also splits a K-major operand `a` (a_rows x k, per-row scales) in
// the same launch (NN: A and B^T of one call).
int launch_split_cols_f16(const float* x, void* hi, void* lo, float* inv_scale, int64_t k,
                          int64_t n, const FixList& fl, cudaStream_t s, const float* a = nullptr,
                          void* a_hi = nullptr, void* a_lo = nullptr, float* a_inv = nullptr,
                          int64_t a_rows = 0, const FixList& a_fl = FixList{});

// Draws skip .. skip + count - 1 of numpy's PCG64 stream with initial
// (state_lo, state_hi, inc_lo, inc_hi), as uniform(low, high) doubles rounded to
// float32 (operands.cu; reference bench.py:104-114).
int fill_uniform_pcg64(float* out, int64_t count, const uint64_t state[4], int64_t skip,
                       double low, double high, cudaStream_t s);

// ------------------------------------------------------------ residual fix-up
// Residual list of one split operand (fix.h): a ring counter pair plus entries
// carved from the caller's workspace. Releasing an unconsumed list (error exit)
// resets its counter on the stream.
struct FixHandle {
  FixList list;
  cudaStream_t stream = nullptr;
  bool consumed = false;
  FixHandle() = default;
  FixHandle(const FixHandle&) = delete;
  FixHandle& operator=(const FixHandle&) = delete;
  ~FixHandle();
};
// Whether split operands track residuals (mtnn_config_set("fixup", 0/1); env MTNN_FIXUP=0).
bool fixup_enabled();
void set_fixup_enabled(bool on);
// Entries to reserve for an operand of `elems` elements, and their bytes.
unsigned fix_capacity(int64_t elems);
inline size_t fix_entry_bytes(unsigned cap) { return ((size_t)cap * sizeof(FixEntry) + 255) & ~size_t(255); }
// Takes a zeroed counter pair from the device ring and points the list at
// `entries` (cap entries). row0: global row of the operand's row 0.
int fix_attach(FixHandle* h, void* entries, unsigned cap, int32_t row0, cudaStream_t s);

enum class FixRep { F16S = 0, TF32_TRUNC = 1, TF32_RNA = 2 };
// Adds the listed residual terms to C (ndst copies: C and up to 7 peer
// buffers, same layout), or recomputes C with the exact-order FFMA tile loop
// if a list overflowed. A: m x k raw rows (global rows a_row0.. of its list),
// inv_a: its F16S row scales; B: n x k (b_is_nk) or k x n (ldb) raw; C rows of
// ldc. reset_*: this is the list's last consumer (its counter is reset).
struct FixupArgs {
  const float* A = nullptr;
  const float* inv_a = nullptr;  // F16S row scales of A (and of B): bound the
  const float* inv_b = nullptr;  // corrections so negligible ones are skipped
  const float* B = nullptr;
  int64_t ldb = 0;
  float* C[8] = {};
  int ndst = 1;
  int64_t ldc = 0;
  int64_t m = 0, n = 0, k = 0;
  bool b_is_nk = true;
  FixRep rep = FixRep::F16S;
  FixList fa, fb;
  int32_t a_row0 = 0, b_row0 = 0;
  bool reset_a = true, reset_b = true;
};
int launch_fixup(const FixupArgs& args, cudaStream_t s);
// How the tensor-core kind represents an operand element (the fix-up recomputes it).
FixRep tc_fix_rep(TcKind kind);

}  // namespace mtnn
