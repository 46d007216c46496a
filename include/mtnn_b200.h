/*
 * mtnn_b200.h — C-ABI of the B200-native MTNN hot path (arXiv 1702.03192).
 *
 * This is the drop-in boundary. The reference binds its kernels through the
 * `_impl` module protocol: a module exposing nine functions that is chosen once
 * at import by `_backend.BACKEND` and looked up by attribute at call time
 *   - /root/reference/pkg/src/mtnn/kernels/__init__.py:24-27  (kernel API binds _impl)
 *   - /root/reference/pkg/src/mtnn/selector.py:25-28          (selector binds _impl)
 *   - protocol signatures: kernels/_numba_impl.py:103-222, kernels/_numpy_impl.py:18-67
 * Every entry point below replaces one protocol function (or the selector step
 * that calls it); the comment on each names the reference interface it replaces.
 *
 * Conventions (mirroring the reference protocol):
 *   - matrices are dense, row-major (C-contiguous) float32; A is m x k, B is n x k,
 *     B^T is k x n, C is m x n; inputs are never written.
 *   - "device" entry points take device pointers and a cudaStream_t passed as
 *     void* (NULL = legacy default stream); they are asynchronous on that stream.
 *   - "_host" entry points take HOST pointers, copy in, compute, copy out and
 *     return synchronously — the reference's numpy-in/numpy-out semantics.
 *   - return value: 0 on success, else one of the MTNN_E* codes; the message
 *     is in mtnn_last_error() (thread-local). The Python shim maps
 *     MTNN_EINVAL -> ValueError, MTNN_ENOMEM -> MemoryError, others -> RuntimeError,
 *     matching the reference's error taxonomy (kernels/__init__.py:70-158).
 *   - no CPU fallback exists: a missing/unsupported GPU is an error.
 */
#ifndef MTNN_B200_H
#define MTNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MTNN_ABI_VERSION 1

/* status codes */
#define MTNN_OK 0
#define MTNN_EINVAL 22  /* bad argument            -> ValueError   */
#define MTNN_ENOMEM 12  /* allocation / budget     -> MemoryError  */
#define MTNN_ECUDA 5    /* CUDA runtime failure    -> RuntimeError */
#define MTNN_ENOTSUP 95 /* no sm_100 device / unsupported variant   */

/* GEMM variant selector (within one path; the NT-vs-TNN choice is the model's). */
#define MTNN_VARIANT_AUTO 0     /* heuristic: tc3xf16s, else tc3xtf32, else FFMA           */
#define MTNN_VARIANT_TC3XTF32 1 /* tcgen05 kind::tf32, hi/lo split, 3 MMAs per product     */
#define MTNN_VARIANT_FFMA 2     /* SIMT FP32 FFMA (exact-order fp32, any shape)            */
#define MTNN_VARIANT_TC3XF16S 3 /* tcgen05 kind::f16, per-row pow2-scaled fp16 hi/lo split */

/* dispatcher choices (reference selector.py:43-51) */
#define MTNN_CHOICE_NT 0
#define MTNN_CHOICE_TNN 1
#define MTNN_REASON_PREDICTED 0
#define MTNN_REASON_MEMORY_FALLBACK 1

typedef struct mtnn_model mtnn_model;

/* ---- library ---------------------------------------------------------- */
int mtnn_abi_version(void);
const char* mtnn_last_error(void);
/* 1 if a compute-capability-10.x device is usable, else 0 (never errors). */
int mtnn_device_available(void);
/* Free device memory in bytes (cudaMemGetInfo), cached for 1 s.
 * Replaces selector.py:76-79 / :158-169 (psutil available memory, 1 s cache). */
int mtnn_device_free_bytes(int64_t* out);
/* The five platform features (gm GiB, sm count, cc MHz, mbw bits, l2c KB) of the
 * current device. Replaces platform.py:113-139 probe_platform detection. */
int mtnn_device_features(double out5[5]);

/* ---- kernel timing (measurement instrumentation) ----------------------
 * When enabled, every launch of the library's main kernels is bracketed with
 * CUDA events on its launch stream and tagged with its algorithmic work:
 * class 0 = tc3xtf32 GEMM (2mnk flops), 1 = FFMA GEMM (2mnk flops),
 * 2 = transpose (8*rows*cols bytes), 3 = operand split (bytes moved: 8 per
 * element; 12 for the column-scaled fp16 split), 4 = split-K reduction
 * (4*(splits+1) bytes per output), 5 = tc3xf16s GEMM (2mnk flops),
 * 6 = residual fix-up after a split tensor-core GEMM (work = 0: its cost is
 * the time it adds).
 * mtnn_profile_read synchronizes the recorded events and returns the totals. */
#define MTNN_KCLASS_GEMM_TC 0
#define MTNN_KCLASS_GEMM_FFMA 1
#define MTNN_KCLASS_TRANSPOSE 2
#define MTNN_KCLASS_SPLIT 3
#define MTNN_KCLASS_REDUCE 4
#define MTNN_KCLASS_GEMM_TC_F16S 5
#define MTNN_KCLASS_FIXUP 6
#define MTNN_KCLASS_COUNT 7
int mtnn_profile_enable(int on);
/* Time only the classes whose bit (1 << class) is set: every timed launch is
 * bracketed by two timestamp events, which serialise the stream around it, so
 * a benchmark can time its dominant kernel without paying that on the rest.
 * While profiling is on (either call), launches and work of EVERY class are
 * counted; mtnn_profile_read's total_ms covers the timed classes only. */
int mtnn_profile_enable_classes(unsigned mask);
/* Time only launches whose work (flops or bytes) is at least `work`; the rest
 * are still counted. mtnn_profile_read_timed returns the timed subset: its
 * milliseconds, launch count and work (so rate = work / ms is consistent). */
int mtnn_profile_min_work(double work);
/* Of the launches that pass the class mask and the work filter, time every
 * n-th (n >= 1; resets the counter): a rotating sample, so the event pairs
 * (which serialise the stream around a launch and break the programmatic launch
 * chain) stay a small part of a step of many mid-size launches. */
int mtnn_profile_sample_every(int n);
/* Phase timestamps (globaltimer ns) of the single-CTA tensor-core GEMM: while
 * `buf` (device memory, ctas x 16 uint64) is set, every launch with at most
 * `ctas` CTAs writes, per CTA: 0 entry, 1 prologue done, 2 after the grid
 * dependency wait, 3 first TMA issued, 4 first stage landed (MMA warp), 5 last
 * MMA issued, 6 first accumulator chunk ready (epilogue), 7 last chunk ready,
 * 8 last C store issued, 9 C stores complete, 10 exit, 11 last TMA issued.
 * Diagnostics only, compiled in with -DMTNN_TRACE (tools/build_variant.sh);
 * other builds return MTNN_ENOTSUP for a non-NULL buffer. NULL turns it off. */
int mtnn_profile_trace(void* buf, int64_t ctas);
/* Stream gate for event-timed windows: enqueues a one-thread kernel that
 * holds `stream` until *host_flag >= value (host_flag: pinned host memory the
 * caller writes after enqueueing the work it times), so host stalls while
 * enqueueing are not counted as device time. Bounded to 1 s. */
int mtnn_gate(const int32_t* host_flag, int32_t value, void* stream);
int mtnn_profile_read_timed(int kclass, double* total_ms, int64_t* launches, double* work);
int mtnn_profile_reset(void);
int mtnn_profile_read(int kclass, double* total_ms, int64_t* launches, double* work);

/* ---- tuning knobs (no reference counterpart; the reference's block/tile
 * hints, kernels/__init__.py:41-42, are the closest analogue) -------------
 * "f16s_inkernel_max_short": tc3xf16s splits the long operand inside the GEMM
 *   (no split pass; a read-only row-max pass gives the row scales) when the
 *   output's short side is at most this and its long side >= 1024; 0 disables.
 *   Default 256, the best on the B200 sweep (env MTNN_F16S_INKERNEL_MAX,
 *   MTNN_F16S_INKERNEL=0 disables). The halves equal the split pass's; only
 *   the output tiling (and so the split-K order) may differ.
 * "tc_pair": 1 (default; env MTNN_TC_PAIR=0 turns it off): NT problems with
 *   >= 74 256x256 output tiles run on CTA pairs (tcgen05 cta_group::2, M = 256,
 *   each CTA loading half of B); 2 forces it whenever structurally possible
 *   (tests), 0 keeps the single-CTA 128x256 tiles. Bit-identical results at the
 *   same split-K.
 * "host_pipeline_blocked": 1 (default; env MTNN_PIPE_BLOCKED=0 turns it off):
 *   host-buffer NT calls on the tc3xf16s path with n >= 1024, k <= 4096 stream B in row
 *   blocks against A's first row block so C leaves while B arrives; 0 = copy B
 *   first, then pipeline A/C row chunks.
 * "host_pipeline_zc": 0 (default; env MTNN_PIPE_ZC=1 turns it on): in that
 *   blocked pipeline, C blocks leave by SM stores into the host C when it is
 *   pinned and device-mapped, instead of 2-D copy-engine copies (A/B: faster
 *   on the widest outputs, slower on others; net -0.6% over the sweep's cases;
 *   the store kernel needs SMs, so it can wait behind long GEMMs: with the
 *   pipeline forced to k = 16384 one case took 128 ms instead of 45).
 * "fixup": 1 (default; env MTNN_FIXUP=0 turns it off): the split tensor-core
 *   paths list every operand element their two-piece representation misses by
 *   more than 2^-19 (tc3xf16s: entries far below their row's max; tc3xtf32:
 *   FP32-subnormal parts) and add those terms to C exactly after the GEMM, so
 *   accuracy does not depend on the range inside a row; 0 skips it (A/B only).
 * Unknown keys -> MTNN_EINVAL. */
int mtnn_config_set(const char* key, int64_t value);
int mtnn_config_get(const char* key, int64_t* value);

/* ---- measurement support --------------------------------------------- */
/* out[i] = float32(low + (high - low) * u_{skip+i}) for i < count, u_j the j-th
 * double of numpy's PCG64 stream whose initial state is {state_lo, state_hi,
 * inc_lo, inc_hi} (np.random.default_rng(seed).bit_generator.state): bit-identical
 * to rng.uniform(low, high, count).astype(float32) after `skip` draws. With
 * skip = 0 for A and skip = m*k for B this is the reference harness's
 * make_operands(shape, seed) (pkg/src/mtnn/bench.py:104-114), generated on the
 * device. Asynchronous on `stream`. */
int mtnn_fill_uniform_pcg64(float* out, int64_t count, const uint64_t state[4], int64_t skip,
                            double low, double high, void* stream);

/* ---- device-resident kernels ----------------------------------------- */
/* C = A x B^T directly. Replaces _impl.gemm_nt / gemm_nt_parallel
 * (_numba_impl.py:139-166; caller kernels/__init__.py:105-116). */
int mtnn_gemm_nt(const float* A, const float* B, float* C, int64_t m, int64_t n,
                 int64_t k, int variant, void* stream);
/* C = A x BT with BT k x n. Replaces _impl.gemm_nn / gemm_nn_parallel
 * (_numba_impl.py:103-136; caller kernels/__init__.py:89-102). */
int mtnn_gemm_nn(const float* A, const float* BT, float* C, int64_t m, int64_t n,
                 int64_t k, int variant, void* stream);
/* Out-of-place transpose: BT[j,i] = B[i,j], B rows x cols. Bit-exact copy.
 * Replaces _impl.transpose_oop (_numba_impl.py:169-182; caller kernels/__init__.py:119-124). */
int mtnn_transpose(const float* B, float* BT, int64_t rows, int64_t cols, void* stream);
/* TNN: allocate B^T (4*n*k bytes, stream-ordered), transpose, NN, release — all
 * inside the call. mem_budget >= 0 caps the buffer and fails with MTNN_ENOMEM
 * before allocating (kernels/__init__.py:150-155); -1 = no cap.
 * Replaces _impl.gemm_tnn / gemm_tnn_parallel (_numba_impl.py:185-194). */
int mtnn_gemm_tnn(const float* A, const float* B, float* C, int64_t m, int64_t n,
                  int64_t k, int variant, int64_t mem_budget, void* stream);

/* ---- multi-GPU: row-sharded NT with the all-gather fused ----
 * Rank r owns rows [row0, row0 + m_local) of A and C (B replicated). The GEMM
 * epilogue stores each C tile into this rank's C (full m x n, row-major) AND
 * into every peer's C (peer_C[i]: the other ranks' full C buffers mapped into
 * this process with mtnn_ipc_open), so the gather runs tile by tile under the
 * MMAs over NVLink instead of an ncclAllGather after them. C is complete on a
 * rank once every rank's call has finished (the caller's barrier). Up to 7
 * peers; tc3xf16s on CTA pairs (shapes it cannot take: local GEMM + device-to-
 * device copies). No reference counterpart (the reference has no multi-GPU). */
int mtnn_gemm_nt_allgather(const float* A_local, const float* B, float* C, float* const* peer_C,
                           int npeers, int64_t row0, int64_t m_local, int64_t n, int64_t k,
                           void* stream);
/* CUDA IPC for the peer C buffers: export a device pointer (64-byte handle +
 * its offset inside its allocation) / map a peer's (ref-counted per handle) /
 * unmap. Errors: MTNN_EINVAL (not device memory, unknown pointer), MTNN_ECUDA. */
int mtnn_ipc_handle(const void* ptr, unsigned char handle[64], int64_t* offset);
int mtnn_ipc_open(const unsigned char handle[64], int64_t offset, void** ptr);
int mtnn_ipc_close(void* ptr);
/* Device-side barrier of `world` ranks (<= 8) on `stream`: this rank stores
 * `epoch` into slot `rank` of every peer's flag array (peer_flags[j], mapped
 * with mtnn_ipc_open; release at system scope, cumulative over everything the
 * stream did before) and waits until its own flags[i] >= epoch for every other
 * rank i (acquire). Enqueued before and after mtnn_gemm_nt_allgather it keeps
 * the exchange's completion on the device, inside the caller's event window.
 * A peer silent for timeout_s (<= 0: 30 s) sets *status = 1 + its rank instead
 * of hanging. Errors: MTNN_EINVAL. */
int mtnn_peer_barrier(uint32_t* flags, uint32_t* const* peer_flags, int npeers, int rank,
                      int world, uint32_t epoch, uint32_t* status, double timeout_s,
                      void* stream);

/* ---- host-buffer (drop-in) variants: synchronous, numpy semantics ------ */
int mtnn_gemm_nt_host(const float* A, const float* B, float* C, int64_t m, int64_t n,
                      int64_t k, int variant);
int mtnn_gemm_nn_host(const float* A, const float* BT, float* C, int64_t m, int64_t n,
                      int64_t k, int variant);
int mtnn_transpose_host(const float* B, float* BT, int64_t rows, int64_t cols);
int mtnn_gemm_tnn_host(const float* A, const float* B, float* C, int64_t m, int64_t n,
                       int64_t k, int variant, int64_t mem_budget);

/* ---- packed-tree walkers (host, float64) -------------------------------
 * Same flat layout as selector._pack_trees (selector.py:82-123): arrays of shape
 * (n_trees, width), feat = -1 marks a leaf, pre-order, root at 0. Routing
 * x[f] < t -> left else right; raw = base; raw += eta * leaf, tree order.
 * Replace _impl.walk_trees / walk_trees_mnk (_numba_impl.py:197-222). */
double mtnn_walk_trees(const int64_t* feat, const double* thresh, const int64_t* left,
                       const int64_t* right, const double* leaf, int64_t n_trees,
                       int64_t width, const double* x, double base_score, double eta);
double mtnn_walk_trees_mnk(const int64_t* feat, const double* thresh,
                           const int64_t* left, const int64_t* right,
                           const double* leaf, int64_t n_trees, int64_t width,
                           const double* prefix5, double m, double n, double k,
                           double base_score, double eta);

/* ---- model handle (immutable, thread-safe) ----------------------------- */
/* Parse the reference's model JSON v1 (gbdt.py:388-455). Errors -> MTNN_EINVAL. */
int mtnn_model_load_json(const char* text, size_t len, mtnn_model** out);
/* Build a model from packed arrays (the Dispatcher's one-time pack, selector.py:151). */
int mtnn_model_from_packed(const int64_t* feat, const double* thresh, const int64_t* left,
                           const int64_t* right, const double* leaf, int64_t n_trees,
                           int64_t width, double base_score, double eta,
                           int64_t n_features, mtnn_model** out);
void mtnn_model_free(mtnn_model* model);
int64_t mtnn_model_n_features(const mtnn_model* model);
int64_t mtnn_model_n_trees(const mtnn_model* model);
/* Raw score of one feature vector (gbdt.predict_raw, gbdt.py:242-254; finite check,
 * arity check -> MTNN_EINVAL). */
int mtnn_model_raw(const mtnn_model* model, const double* x, int64_t nx, double* raw);
/* Algorithm 2's decision (selector.py:181-190): 4*n*k > free_bytes -> NT with
 * reason MEMORY_FALLBACK and raw = NaN; else raw >= 0 -> NT, raw < 0 -> TNN.
 * free_bytes < 0 -> query the device (mtnn_device_free_bytes). */
int mtnn_select(const mtnn_model* model, const double prefix5[5], int64_t m, int64_t n,
                int64_t k, int64_t free_bytes, double* raw_out, int* choice_out,
                int* reason_out);
/* Host cost of one mtnn_select decision in C++ (no FFI), averaged over `iters`
 * decisions on sweep shapes with ample free memory: the paper's "0.005 ms"
 * predict budget measured on this build. */
int mtnn_select_cost_ns(const mtnn_model* model, const double prefix5[5], int64_t iters,
                        double* ns_per_call);
/* Dispatcher.gemm (selector.py:192-221): select, run TNN or NT; a TNN
 * allocation failure is retried as NT (choice_out reports what ran). */
int mtnn_dispatch_gemm(const mtnn_model* model, const double prefix5[5], const float* A,
                       const float* B, float* C, int64_t m, int64_t n, int64_t k,
                       int64_t free_bytes, int variant, void* stream, int* choice_out);
int mtnn_dispatch_gemm_host(const mtnn_model* model, const double prefix5[5],
                            const float* A, const float* B, float* C, int64_t m,
                            int64_t n, int64_t k, int64_t free_bytes, int variant,
                            int* choice_out);

#ifdef __cplusplus
}
#endif
#endif /* MTNN_B200_H */
