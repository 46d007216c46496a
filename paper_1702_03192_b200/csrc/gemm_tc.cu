// Tensor-core FP32-accurate GEMMs for sm_100a: tcgen05 MMAs on hi/lo operand
// halves, TMA-fed shared memory, TMEM accumulators. Serves both MTNN paths:
//   NT  C = A * B^T  with B stored n x k (K-major UMMA B operand)
//       — reference kernels/_numba_impl.py:139-166 (gemm_nt), PAPER.md:249-257;
//   NN  C = A * BT   with BT stored k x n (MN-major UMMA B operand)
//       — reference kernels/_numba_impl.py:31-136 (gemm_nn), the second half of
//         TNN.
//
// FP32 accuracy from 11-bit-significand tensor-core inputs: every operand x is
// split into hi + lo and the kernel accumulates hi*hi + hi*lo + lo*hi (the
// dropped lo*lo is ~2^-22 relative):
//   KindF16S (default): per-row power-of-two scale s, h = fp16(x*s),
//     l = fp16(x*s - h) (split_f16.cu); kind::f16 MMAs at twice the TF32 rate;
//     the epilogue multiplies by 1/(s_row * s_col), exact.
//   KindTF32: hi = the raw fp32 operand (the tensor core truncates it to tf32),
//     lo = x - trunc_tf32(x); kind::tf32 MMAs.
// The TMEM accumulator truncates (measured -0.5 ulp bias per accumulation), so
// each accumulation covers chunk_kb k-blocks (48 MMAs) and the epilogue adds
// the chunks into round-to-nearest FP32 registers (FP32 promotion).
//
// Kernels:
//   gemm_tc3x_kernel<BN, B_MN, Kind, kConv>: persistent, one CTA per SM,
//     warp-specialised — warp 0 TMA producer (4-stage ring), warp 1 one-lane
//     MMA issuer (M = 128, N = BN), warp 2 TMEM allocator (2 x BN columns:
//     double-buffered accumulator so the epilogue of tile i overlaps the MMAs of
//     tile i+1), epilogue warps (tcgen05.ld, FP32 promotion, swizzled staging,
//     TMA store). kConv != 0: one operand split in shared memory from raw fp32
//     tiles (skinny problems; see the kernel).
//   gemm_tc3x_pair_kernel<B_MN, Kind>: the CTA-pair (cta_group::2) variant,
//     256 x 256 tiles, optional peer stores (fused all-gather).
// Work units are (k-split, tile); with few output tiles and long k the host
// splits K so the grid reaches all SMs and a deterministic reduction kernel sums
// the fp32 partials.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <utility>
#include <atomic>
#include <cmath>
#include <mutex>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#include "common.h"
#include "workspace.h"

namespace mtnn {

int launch_splitk_reduce(const float* part, float* C, int64_t count, int splits,
                         cudaStream_t s);

namespace tc {

constexpr int BM = 128;          // UMMA M (one CTA, 128 TMEM lanes)
constexpr int kStages = 4;
constexpr int kEpiWarp0 = 4;      // warps 0..3: TMA, MMA, TMEM alloc, spare
constexpr int kEpiWarps = 16;     // 4 TMEM lane quarters x 4 column quarters
// Epilogue tail: 1 = the tile's output scales are loaded while its last chunk
// is still in the tensor core (the store loop then waits on no L2 load: the
// exposed tail of a tile drops ~0.8-1.2 us, 1024^3 45.0 -> 43.7 us per call);
// 0 = load them in the store loop (A/B builds: -DMTNN_TAIL=0). Staging the
// last tile in the idle operand ring so its stores issue back to back measured
// slower and was dropped.
#ifndef MTNN_TAIL
#define MTNN_TAIL 1
#endif
constexpr int kTail = MTNN_TAIL;
constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);
// Warp roles. F16S in-kernel conversion (kConv != 0, BN = 128): 8 epilogue
// warps (4 lane quarters x 2 column halves) and 8 converter warps (two groups
// of 4 taking alternate k-blocks, one thread per row of the converted tile).
constexpr int kF16ConvRows = 128;
template <bool kF16Conv>
struct Roles {
  static constexpr int kEpi = kF16Conv ? 8 : kEpiWarps;
  static constexpr int kConvWarps = kF16Conv ? 8 : 0;
  static constexpr int kConv0 = kEpiWarp0 + kEpi;  // first converter warp
  static constexpr int kThreads = 32 * (kEpiWarp0 + kEpi + kConvWarps);
};
constexpr uint32_t kLayoutSW64 = 4;      // UMMA SWIZZLE_64B

// Operand kinds. Both keep 64-byte K-major rows per k-block (SWIZZLE_64B, one
// UMMA K-step = 32 bytes), so the smem ring and the K-major descriptors are
// shared; they differ in element type, MMA kind and the MN-major B layout.
struct KindTF32 {  // hi = raw fp32 (read as trunc-tf32), lo = x - trunc(x)
  static constexpr int kElemBytes = 4;
  static constexpr int BK = 16;                 // elements per k-block
  static constexpr int UMMA_K = 8;              // kind::tf32
  static constexpr uint32_t kFmt = 2;           // instruction-descriptor TF32
  static constexpr bool kScaled = false;
  static constexpr CUtensorMapDataType kTmaType = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  // MN-major B^T: SWIZZLE_128B_BASE32B (the only MN-major tf32 layout), boxes of
  // 32 columns x 16 k-rows (2 KiB), 4-row groups 512 B apart, K-step 8 rows.
  static constexpr int kMnBox = 32;
  static constexpr uint32_t kMnLayout = 1, kMnLBO = 2048, kMnSBO = 512, kMnKStep = 1024;
  static constexpr CUtensorMapSwizzle kMnSwizzle = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
};
struct KindF16S {  // per-row power-of-2 scaled fp16 hi/lo (split_f16.cu)
  static constexpr int kElemBytes = 2;
  static constexpr int BK = 32;
  static constexpr int UMMA_K = 16;             // kind::f16
  static constexpr uint32_t kFmt = 0;           // instruction-descriptor F16
  static constexpr bool kScaled = true;
  static constexpr CUtensorMapDataType kTmaType = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  // MN-major B^T: SWIZZLE_128B, boxes of 64 columns x 32 k-rows (4 KiB), 8-row
  // groups 1 KiB apart, K-step 16 rows.
  static constexpr int kMnBox = 64;
  static constexpr uint32_t kMnLayout = 2, kMnLBO = 4096, kMnSBO = 1024, kMnKStep = 2048;
  static constexpr CUtensorMapSwizzle kMnSwizzle = CU_TENSOR_MAP_SWIZZLE_128B;
};

// kRawBytes: slot size of the raw fp32 tile of an operand converted in-kernel
// (F16S, kConv != 0): 128 rows x 32 k x 4 B, TMA SWIZZLE_128B. Those tiles get
// their own deeper ring (kRawStages) so more DRAM bytes are in flight per SM
// than the 3-stage h/l ring alone would allow — the converted operand streams
// from DRAM, the other one from L2.
// In-kernel split rings: 4 h/l stages (even, so each of the two converter
// groups — alternate k-blocks — always owns the same two slots) and 5 raw
// stages. Against 3 + 7: in-kernel shapes 2.5-3.6% faster (128x16384x16384
// 412 -> 399 us, 16384x256x4096 170 -> 167 us), and racecheck no longer sees two
// converter groups writing one slot (their hand-off went through the tensor
// core's commit-arrive, which it does not model). -D overrides for A/B builds.
#ifndef MTNN_HL_STAGES_RAW
#define MTNN_HL_STAGES_RAW 4
#endif
#ifndef MTNN_RAW_STAGES
#define MTNN_RAW_STAGES 5
#endif
template <int BN, int kRawBytes = 0, int kEpi = kEpiWarps>
struct Smem {
  static constexpr int kABytes = BM * 64;                // 8 KiB (64-byte k-block rows)
  static constexpr int kBBytes = BN * 64;                // 16 KiB at BN=256
  static constexpr int kStages = kRawBytes ? MTNN_HL_STAGES_RAW : 4;      // h/l ring
  static constexpr int kRawStages = kRawBytes ? MTNN_RAW_STAGES : 0;     // raw fp32 ring
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kStagingBytes = 32 * 16 * 4;      // one 32x16 fp32 tile
  static constexpr int kRingBytes = kStages * kStageBytes;
  static constexpr int kRawOff = kRingBytes;             // 1024-aligned
  static constexpr int kRawRingBytes = kRawStages * kRawBytes;
  static constexpr int kEpiBytes = kEpi * kStagingBytes;
  static constexpr int kBarBytes = 256;
  static constexpr int kTotal = 1024 + kRingBytes + kRawRingBytes + kEpiBytes + kBarBytes;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, const uint4& v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 r;\n\t.reg .pred p;\n\t"
      "elect.sync r|p, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map,
                                            uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map,
                                            uint32_t bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0,
                                             int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_store_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Programmatic dependent launch: the GEMMs are launched with programmatic stream
// serialization, so their prologue (barrier init, TMEM allocation, descriptor
// prefetch) overlaps the tail of the operand split that precedes them on the
// stream; every thread then waits for that grid's completion (and its memory)
// before anything reads an operand. Kernels that trigger early: the splits.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
template <bool kF16>
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  if constexpr (kF16) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}
// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
        "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
        "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]),
        "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
        "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
        "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor (sm_100 format: version 1 at bit 46).
// start/lbo/sbo in bytes; layout 4 = SWIZZLE_64B.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                               uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// Instruction descriptor: D=f32, A=B=fmt, A K-major, B K- or MN-major, M=128, N.
__host__ __device__ constexpr uint32_t make_idesc(int n, bool b_mn_major, uint32_t fmt) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

struct Params {
  int64_t m, n, k;
  int64_t ldc;   // C row stride in elements (>= n; > n for a row-padded output)
  int chunk_kb;  // k-blocks per TMEM accumulation chunk (FP32 promotion period)
  int tiles_m, tiles_n, splits, kblocks_per_split, total_kblocks;
  int tiles_mp;  // CTA-pair kernel: pairs of m-tiles
  int group_m;   // CTA-pair kernel: m-tile pairs per raster group
  int npeers;    // CTA-pair kernel: peer C buffers the epilogue also stores to
  int units;
  const float* inv_scale_a;  // KindF16S: 1/s per row of A (m) and of B (n)
  const float* inv_scale_b;
  unsigned long long* trace;    // mtnn_profile_trace: [CTA][kTracePoints] globaltimer ns
};
constexpr int kTracePoints = 16;

// Work-unit order: units are (k-split, tile); within a split, tiles walk
// groups of kGroupM m-tiles with the group's m-tiles fastest, so the ~148 units
// in flight cover a ~16 x 9 block of output tiles. Each A and B panel is then
// streamed from DRAM by few waves instead of every wave re-streaming all of A
// (m-fastest order), which cost ~15% at m = 16384.
constexpr int kGroupM = 16;
__device__ __forceinline__ void unit_coords(int u, const Params& p, int& split, int& tm,
                                            int& tn) {
  const int tiles = p.tiles_m * p.tiles_n;
  split = u / tiles;
  const int t = u - split * tiles;
  const int per_group = kGroupM * p.tiles_n;
  const int group = t / per_group;
  const int first_m = group * kGroupM;
  const int gm = min(kGroupM, p.tiles_m - first_m);
  const int r = t - group * per_group;
  tm = first_m + r % gm;
  tn = r / gm;
}

// One work item of a CTA: output tile (tm, tn), k-split index, k-block range
// (units are (k-split, tile), strided over the grid).
struct Work {
  int tm, tn, split, kb0, kb1;
};
__device__ __forceinline__ int work_count(const Params& p) {
  return blockIdx.x < (unsigned)p.units ? (p.units - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
}
__device__ __forceinline__ Work work_item(const Params& p, int i) {
  Work w;
  unit_coords(blockIdx.x + i * gridDim.x, p, w.split, w.tm, w.tn);
  w.kb0 = w.split * p.kblocks_per_split;
  w.kb1 = min(p.total_kblocks, w.kb0 + p.kblocks_per_split);
  return w;
}

// Phase timestamps of one CTA (mtnn_profile_trace; off = null pointer).
// Compiled in only with -DMTNN_TRACE (tools/build_variant.sh NAME -DMTNN_TRACE):
// even the untaken null check costs ~2 us per call on the one-wave GEMMs.
__device__ __forceinline__ void trace_mark(const Params& p, int point) {
#ifdef MTNN_TRACE
  if (p.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[(size_t)blockIdx.x * kTracePoints + point] = t;
  }
#else
  (void)p;
  (void)point;
#endif
}

// FP16 hi/lo of 8 consecutive k-values of one row with the row's exact
// power-of-two scale s — the same operations as split_f16.cu's split2, so the
// halves (and every C bit) equal the pre-split path's.
__device__ __forceinline__ void split8_f16(const float4& x0, const float4& x1, float s,
                                          uint4& hw, uint4& lw) {
  const float v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
  uint32_t hp[4], lp[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // packed round-to-nearest conversions: per element identical to
    // __float2half_rn, two per instruction
    const float a = v[2 * i] * s, b = v[2 * i + 1] * s;
    const __half2 h2 = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h2);
    const __half2 l2 = __floats2half2_rn(a - hf.x, b - hf.y);
    hp[i] = *reinterpret_cast<const uint32_t*>(&h2);
    lp[i] = *reinterpret_cast<const uint32_t*>(&l2);
  }
  hw = make_uint4(hp[0], hp[1], hp[2], hp[3]);
  lw = make_uint4(lp[0], lp[1], lp[2], lp[3]);
}

// MN-major F16S B: the exact column scales (powers of two) of one promotion
// chunk for an epilogue warp's kCols columns, lane l holding columns l, 32 + l,
// ... (coalesced loads, one per 32 columns; columns >= n get 0: never stored).
template <int kCols>
struct ChunkScales {
  float v[kCols / 32];
};
template <int kCols>
__device__ __forceinline__ ChunkScales<kCols> load_chunk_scales(const float* inv_b, int chunk,
                                                                int64_t n, int64_t col0, int lane) {
  const float* sc = inv_b + (int64_t)chunk * n + col0;
  ChunkScales<kCols> c;
#pragma unroll
  for (int i = 0; i < kCols / 32; ++i)
    c.v[i] = col0 + 32 * i + lane < n ? __ldg(sc + 32 * i + lane) : 0.f;
  return c;
}
// Adds 16 TMEM columns (the c16-th group of the warp's) of one chunk into the
// FP32 sums, each scaled by its column's chunk scale (x * 2^e is exact, so the
// sum rounds once per chunk exactly as the unscaled path does).
template <int kCols>
__device__ __forceinline__ void add_chunk_scaled(float* sum, const uint32_t (&r)[16],
                                                 const ChunkScales<kCols>& cs, int c16) {
  const float src = cs.v[c16 / 2];
  const int base = (c16 & 1) * 16;
#pragma unroll
  for (int j = 0; j < 16; ++j)
    sum[j] += __uint_as_float(r[j]) * __shfl_sync(0xffffffffu, src, base + j);
}

// ------------------------------------------------------------------- kernel
// kConv: 0 = both operands come split from the pre-pass; 1 / 2 = operand A / B
// is read raw (fp32, 4 B per element from DRAM, no split pass) and split
// in-kernel from the tile TMA just landed; the MMA warp then waits on conv_bar
// instead of full_bar.
//   KindTF32: lo = x - trunc_tf32(x) is elementwise, written at the same offsets
//     of the lo tile (the raw tile itself is hi); warps 2-3 (idle after TMEM
//     allocation) do it.
//   KindF16S: the raw tile lands in its own SWIZZLE_128B slot and 4 extra warps
//     (one thread per tile row, kF16ConvRows = 128 = the converted tile's rows)
//     write h/l into the operand's SWIZZLE_64B slots with the row scale from a
//     read-only row-max pre-pass (4 B per element instead of the split's 8).
template <int BN, bool B_MN, class Kind, int kConv>
__global__ void __launch_bounds__(Roles<(kConv == 1 || kConv == 2) && Kind::kScaled>::kThreads, 1)
gemm_tc3x_kernel(const __grid_constant__ CUtensorMap map_ahi,
                     const __grid_constant__ CUtensorMap map_alo,
                     const __grid_constant__ CUtensorMap map_bhi,
                     const __grid_constant__ CUtensorMap map_blo,
                     const __grid_constant__ CUtensorMap map_c, const Params p) {
  constexpr bool kF16Conv = (kConv == 1 || kConv == 2) && Kind::kScaled;
  static_assert(!kF16Conv || (kConv == 1 ? BM : BN) == kF16ConvRows,
                "F16S in-kernel conversion needs a 128-row converted tile");
  static_assert(!(kF16Conv && kConv == 2 && B_MN), "in-kernel F16S split of B needs K-major B (NT)");
  using R = Roles<kF16Conv>;
  using S = Smem<BN, kF16Conv ? kF16ConvRows * 128 : 0, R::kEpi>;
  constexpr int kColsPerWarp = BN / (R::kEpi / 4);  // each epilogue warp: a column slice
  // MN-major F16S B carries one scale per (kScaleChunkK rows, column): applied
  // per promotion chunk (the host keeps chunks and k-splits aligned to it)
  constexpr bool kChunkB = B_MN && Kind::kScaled;
  constexpr int kScaleKb = kScaleChunkK / Kind::BK;
  static_assert(kColsPerWarp % 32 == 0, "chunk scales: 32-column groups per epilogue warp");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStages = S::kStages;
  constexpr int kRawStages = S::kRawStages;
  static_assert(3 * kStages + 4 + 2 * kRawStages <= S::kBarBytes / 8 - 1, "barrier space");
  uint8_t* ring = smem;
  uint8_t* raw_ring = smem + S::kRawOff;
  uint8_t* epi = smem + S::kRingBytes + S::kRawRingBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi + S::kEpiBytes);
  uint64_t* full_bar = bars;                 // [kStages]
  uint64_t* empty_bar = bars + kStages;      // [kStages]
  uint64_t* tfull_bar = bars + 2 * kStages;  // [2]
  uint64_t* tempty_bar = bars + 2 * kStages + 2;  // [2]
  uint64_t* conv_bar = bars + 2 * kStages + 4;     // [kStages] (kConv != 0)
  uint64_t* rfull_bar = bars + 3 * kStages + 4;    // [kRawStages] (F16S conversion)
  uint64_t* rempty_bar = rfull_bar + kRawStages;   // [kRawStages]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty_bar + kRawStages);
  // TMA bytes per h/l stage: F16S conversion loads only the other operand's
  // halves (the raw tile arrives on its own ring); TF32 conversion skips the
  // converted lo slot.
  constexpr int kConvBytes = kConv == 1 ? S::kABytes : kConv == 2 ? S::kBBytes : 0;
  constexpr int kExpectBytes = kF16Conv ? S::kStageBytes - 2 * kConvBytes
                                        : S::kStageBytes - kConvBytes;
  constexpr int kRawTileBytes = kF16ConvRows * 128;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (threadIdx.x == 0) trace_mark(p, 0);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_c)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&tfull_bar[s]), 1);
      mbar_init(smem_u32(&tempty_bar[s]), R::kEpi);  // one arrive per epilogue warp
    }
    for (int s = 0; s < kStages; ++s)
      mbar_init(smem_u32(&conv_bar[s]), kF16Conv ? R::kConvWarps / 2 : 2);  // one converter group
    for (int s = 0; s < kRawStages; ++s) {
      mbar_init(smem_u32(&rfull_bar[s]), 1);
      mbar_init(smem_u32(&rempty_bar[s]), R::kConvWarps / 2);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) trace_mark(p, 1);
  pdl_wait();
  pdl_trigger();  // the next call's split may be scheduled (it waits for us)
  if (threadIdx.x == 0) trace_mark(p, 2);

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      const int nw = work_count(p);
      for (int wi = 0; wi < nw; ++wi) {
        const Work w = work_item(p, wi);
        const int tm = w.tm, tn = w.tn;
        if (wi == 0) trace_mark(p, 12);
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          mbar_expect_tx(fb, kExpectBytes);
          uint8_t* st = ring + stage * S::kStageBytes;
          const int kx = kb * Kind::BK;
          if (!(kF16Conv && kConv == 1)) {  // (raw A: warp 3)
            tma_load_2d(smem_u32(st), &map_ahi, fb, kx, tm * BM);
            if (kConv != 1) tma_load_2d(smem_u32(st + S::kABytes), &map_alo, fb, kx, tm * BM);
          }
          if (kF16Conv && kConv == 2) {
            // raw B: warp 3
          } else if (!B_MN) {
            tma_load_2d(smem_u32(st + 2 * S::kABytes), &map_bhi, fb, kx, tn * BN);
            if (kConv != 2)
              tma_load_2d(smem_u32(st + 2 * S::kABytes + S::kBBytes), &map_blo, fb, kx, tn * BN);
          } else {
            // BN/kMnBox boxes of [BK k-rows][kMnBox columns] (128-byte rows), each
            // one MN group of the canonical MN-major layout, kMnLBO bytes apart
#pragma unroll
            for (int g = 0; g < BN / Kind::kMnBox; ++g) {
              tma_load_2d(smem_u32(st + 2 * S::kABytes + g * Kind::kMnLBO), &map_bhi, fb,
                          tn * BN + g * Kind::kMnBox, kx);
              if (kConv != 2)
                tma_load_2d(smem_u32(st + 2 * S::kABytes + S::kBBytes + g * Kind::kMnLBO),
                            &map_blo, fb, tn * BN + g * Kind::kMnBox, kx);
            }
          }
          if (wi == 0 && kb == w.kb0) trace_mark(p, 3);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
      trace_mark(p, 11);
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc = make_idesc(BN, B_MN, Kind::kFmt);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const int nw = work_count(p);
    for (int wi = 0; wi < nw; ++wi) {
      const Work w = work_item(p, wi);
      const int kb1 = w.kb1;
      for (int kc = w.kb0, kce; kc < kb1; kc = kce) {
        kce = min(kb1, kc + p.chunk_kb);
        mbar_wait(smem_u32(&tempty_bar[acc]), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = kc; kb < kce; ++kb) {
          // TF32 conversion waits full_bar itself, so conv_bar implies it; the F16S
          // converters do not (the raw tile has its own ring)
          if (kConv == 0 || kF16Conv) mbar_wait(smem_u32(&full_bar[stage]), phase);
          if (kConv == 1 || kConv == 2) mbar_wait(smem_u32(&conv_bar[stage]), phase);
          if (wi == 0 && kb == w.kb0 && lane == 0) trace_mark(p, 4);
          tc_fence_after();
          if (elect_one()) {
            uint8_t* st = ring + stage * S::kStageBytes;
            const uint32_t a_hi = smem_u32(st);
            const uint32_t a_lo = a_hi + S::kABytes;
            const uint32_t b_hi = a_hi + 2 * S::kABytes;
            const uint32_t b_lo = b_hi + S::kBBytes;
#pragma unroll
            for (int ks = 0; ks < Kind::BK / Kind::UMMA_K; ++ks) {
              // A: K-major SW64 — 64-byte rows, 8-row groups 512 B apart; k-step +32 B.
              const uint64_t dah = make_sdesc(a_hi + ks * 32, 16, 512, kLayoutSW64);
              const uint64_t dal = make_sdesc(a_lo + ks * 32, 16, 512, kLayoutSW64);
              uint64_t dbh, dbl;
              if (!B_MN) {
                dbh = make_sdesc(b_hi + ks * 32, 16, 512, kLayoutSW64);
                dbl = make_sdesc(b_lo + ks * 32, 16, 512, kLayoutSW64);
              } else {
                // B: MN-major — column groups kMnLBO apart, k-row groups kMnSBO apart
                dbh = make_sdesc(b_hi + ks * Kind::kMnKStep, Kind::kMnLBO, Kind::kMnSBO,
                                 Kind::kMnLayout);
                dbl = make_sdesc(b_lo + ks * Kind::kMnKStep, Kind::kMnLBO, Kind::kMnSBO,
                                 Kind::kMnLayout);
              }
              const uint32_t accum = (kb == kc && ks == 0) ? 0u : 1u;
              tc_mma<Kind::kScaled>(tmem_d, dal, dbh, idesc, accum);
              tc_mma<Kind::kScaled>(tmem_d, dah, dbl, idesc, 1u);
              tc_mma<Kind::kScaled>(tmem_d, dah, dbh, idesc, 1u);
            }
            tc_commit(smem_u32(&empty_bar[stage]));
            if (kb == kce - 1) tc_commit(smem_u32(&tfull_bar[acc]));
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
    if (lane == 0) trace_mark(p, 5);
  } else if (kF16Conv && warp == 3) {
    // ===================== TMA producer of the raw (converted) operand =====================
    if (elect_one()) {
      int rs = 0;
      uint32_t rphase = 0;
      const int nw = work_count(p);
      for (int wi = 0; wi < nw; ++wi) {
        const Work w = work_item(p, wi);
        const int tm = w.tm, tn = w.tn;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(smem_u32(&rempty_bar[rs]), rphase ^ 1);
          const uint32_t fb = smem_u32(&rfull_bar[rs]);
          mbar_expect_tx(fb, kRawTileBytes);
          const uint32_t dst = smem_u32(raw_ring + rs * kRawTileBytes);
          if (kConv == 1) tma_load_2d(dst, &map_ahi, fb, kb * Kind::BK, tm * BM);
          else tma_load_2d(dst, &map_bhi, fb, kb * Kind::BK, tn * BN);
          if (++rs == kRawStages) { rs = 0; rphase ^= 1; }
        }
      }
    }
  } else if ((kConv == 1 || kConv == 2) && !Kind::kScaled && (warp == 2 || warp == 3)) {
    // ===================== in-kernel lo split (TF32, one operand) =====================
    const int t = threadIdx.x - 64;  // 0..63
    int stage = 0;
    uint32_t phase = 0;
    const int nw = work_count(p);
    for (int wi = 0; wi < nw; ++wi) {
      const Work w = work_item(p, wi);
      for (int kb = w.kb0; kb < w.kb1; ++kb) {
        mbar_wait(smem_u32(&full_bar[stage]), phase);
        uint8_t* raw = ring + stage * S::kStageBytes + (kConv == 1 ? 0 : 2 * S::kABytes);
        uint8_t* lo = raw + kConvBytes;
#pragma unroll 4
        for (int i = t; i < kConvBytes / 16; i += 64) {
          float4 v = *reinterpret_cast<const float4*>(raw + 16 * i);
          v.x -= __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          v.y -= __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          v.z -= __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          v.w -= __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          *reinterpret_cast<float4*>(lo + 16 * i) = v;
        }
        fence_proxy_async_smem();  // generic-proxy smem writes -> visible to UMMA
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&conv_bar[stage]));
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (kF16Conv && warp >= R::kConv0) {
    // ===================== in-kernel FP16 split (F16S, one operand) =====================
    // Two groups of 4 warps take alternate k-blocks, so each group's serial
    // chain (raw wait, LDS, convert, h/l-slot wait, STS, proxy fence, arrive)
    // has two MMA k-blocks of time. Thread r of a group owns row r of the
    // converted tile: reads its 128-byte raw row (SWIZZLE_128B: 16-byte chunk c at
    // c ^ (r & 7)) and writes 64-byte h and l rows (SWIZZLE_64B: chunk c at
    // c ^ ((r >> 1) & 3)); both patterns keep each warp's 16-byte accesses
    // conflict-free.
    const int t = threadIdx.x - 32 * R::kConv0;
    const int r = t % kF16ConvRows;             // tile row
    const int grp = t / kF16ConvRows;           // k-block parity this thread converts
    const int sw128 = r & 7, sw64 = (r >> 1) & 3;
    const float* inv = kConv == 1 ? p.inv_scale_a : p.inv_scale_b;
    const int64_t nrows = kConv == 1 ? p.m : p.n;
    int stage = 0, rs = 0, parity = 0;
    uint32_t phase = 0, rphase = 0;
    const int nw = work_count(p);
    for (int wi = 0; wi < nw; ++wi) {
      const Work w = work_item(p, wi);
      const int64_t row = (int64_t)(kConv == 1 ? w.tm * BM : w.tn * BN) + r;
      const float sc = row < nrows ? 1.f / __ldg(inv + row) : 1.f;  // exact: powers of two
      for (int kb = w.kb0; kb < w.kb1; ++kb) {
        if (parity == grp) {
          // raw tile -> registers -> halves; the raw slot is released as soon as
          // its values are consumed, before waiting for the h/l slot
          mbar_wait(smem_u32(&rfull_bar[rs]), rphase);
          const uint32_t raw = smem_u32(raw_ring + rs * kRawTileBytes) + r * 128;
          float4 x[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) x[j] = lds128f(raw + ((j ^ sw128) << 4));
          uint4 hw[4], lw[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) split8_f16(x[2 * j], x[2 * j + 1], sc, hw[j], lw[j]);
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&rempty_bar[rs]));
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);  // MMA done with the h/l slot
          const uint32_t hrow = smem_u32(ring + stage * S::kStageBytes) +
                                (kConv == 1 ? 0 : 2 * S::kABytes) + r * 64;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t off = (j ^ sw64) << 4;
            sts128(hrow + off, hw[j]);
            sts128(hrow + kConvBytes + off, lw[j]);
          }
          fence_proxy_async_smem();  // generic-proxy smem writes -> visible to UMMA
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&conv_bar[stage]));
        }
        parity ^= 1;
        if (++stage == kStages) { stage = 0; phase ^= 1; }
        if (++rs == kRawStages) { rs = 0; rphase ^= 1; }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ===================== epilogue: FP32 promotion + store =====================
    // The tensor core's accumulator truncates (measured bias ~ -0.5 ulp per MMA
    // accumulation), so each TMEM accumulation covers only p.chunk_kb k-blocks; the
    // chunk is then added into round-to-nearest FP32 register sums here.
    const int e = warp - kEpiWarp0;
    const int q = warp % 4;             // TMEM lane quarter this warp may access
    const int h = e / 4;                // column slice
    uint8_t* stg = epi + e * S::kStagingBytes;
    int acc = 0;
    uint32_t acc_phase = 0;
    const int nw = work_count(p);
    for (int wi = 0; wi < nw; ++wi) {
      const Work w = work_item(p, wi);
      const int tm = w.tm, tn = w.tn, split = w.split, kb1 = w.kb1;
      const int64_t row = (int64_t)tm * BM + q * 32 + lane;
      const int64_t col0 = (int64_t)tn * BN + h * kColsPerWarp;
      float sum[kColsPerWarp];
#pragma unroll
      for (int j = 0; j < kColsPerWarp; ++j) sum[j] = 0.f;
      float sa_pre = 1.f;  // (kTail >= 1: the tile's output scales, preloaded)
      ChunkScales<kColsPerWarp> csb{};
      for (int kc = w.kb0, kce; kc < kb1; kc = kce) {
        kce = min(kb1, kc + p.chunk_kb);
        // (the chunk's column scales load while the MMAs of the chunk finish)
        ChunkScales<kColsPerWarp> cs{};
        if (kChunkB) cs = load_chunk_scales<kColsPerWarp>(p.inv_scale_b, kc / kScaleKb, p.n, col0, lane);
        if (kTail >= 1 && Kind::kScaled && kce >= kb1) {
          // the output scales load while the tile's last chunk is still in the
          // tensor core (the store loop below would otherwise wait on L2 for them)
          if (row < p.m) sa_pre = __ldg(p.inv_scale_a + row);
          if (!kChunkB) csb = load_chunk_scales<kColsPerWarp>(p.inv_scale_b, 0, p.n, col0, lane);
        }
        mbar_wait(smem_u32(&tfull_bar[acc]), acc_phase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + h * kColsPerWarp;
#pragma unroll
        for (int c = 0; c < kColsPerWarp / 16; ++c) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(taddr + c * 16, r);
          tmem_ld_wait();
          if (kChunkB) {
            // MN-major F16S B: this promotion chunk's exact column scales
            add_chunk_scaled(sum + c * 16, r, cs, c);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) sum[c * 16 + j] += __uint_as_float(r[j]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[acc]));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      // KindF16S: undo the exact power-of-two operand scales while storing,
      // C = (acc * 1/s_a[row]) * 1/s_b[col] (MN-major B: applied per chunk above)
      if (e == 0 && lane == 0 && wi == nw - 1) trace_mark(p, 13);
      const float sa = kTail >= 1 ? sa_pre
                                  : (Kind::kScaled && row < p.m) ? __ldg(p.inv_scale_a + row) : 1.f;
      // Store: 32 rows x kColsPerWarp through a 32x16 staging tile (64B swizzle).
#pragma unroll
      for (int c = 0; c < kColsPerWarp / 16; ++c) {
        if (lane == 0) tma_store_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int pj = j ^ ((lane >> 1) & 3);
          float4 v = make_float4(sum[c * 16 + 4 * j], sum[c * 16 + 4 * j + 1],
                                 sum[c * 16 + 4 * j + 2], sum[c * 16 + 4 * j + 3]);
          if (Kind::kScaled && kChunkB) {
            v.x *= sa; v.y *= sa; v.z *= sa; v.w *= sa;
          } else if (kTail >= 1 && Kind::kScaled) {
            // column c*16 + 4j + t of the warp's slice: lane (that % 32) of csb
            const int cc = c * 16 + 4 * j;
            const float src = csb.v[cc / 32];
            v.x = (v.x * sa) * __shfl_sync(0xffffffffu, src, (cc + 0) % 32);
            v.y = (v.y * sa) * __shfl_sync(0xffffffffu, src, (cc + 1) % 32);
            v.z = (v.z * sa) * __shfl_sync(0xffffffffu, src, (cc + 2) % 32);
            v.w = (v.w * sa) * __shfl_sync(0xffffffffu, src, (cc + 3) % 32);
          } else if (Kind::kScaled) {
            // the scale vector has n entries (n % 4 == 0): whole float4s are in range
            const int64_t cj = col0 + c * 16 + 4 * j;
            const float4 sb = cj < p.n ? __ldg(reinterpret_cast<const float4*>(p.inv_scale_b + cj))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            v.x = (v.x * sa) * sb.x;
            v.y = (v.y * sa) * sb.y;
            v.z = (v.z * sa) * sb.z;
            v.w = (v.w * sa) * sb.w;
          }
          *reinterpret_cast<float4*>(stg + lane * 64 + pj * 16) = v;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&map_c, smem_u32(stg), tn * BN + h * kColsPerWarp + c * 16,
                       tm * BM + q * 32, split);
          tma_store_commit();
        }
        if (c == 0 && e == 0 && lane == 0 && wi == nw - 1) trace_mark(p, 14);
      }
    }
    if (e == 0 && lane == 0) trace_mark(p, 8);
    if (lane == 0) tma_store_wait_all();
    if (e == 0 && lane == 0) trace_mark(p, 9);
  }

  __syncwarp();  // reconverge the role branches: bar.sync is warp-aligned
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_mark(p, 10);
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(2 * BN));
  }
}

// 3xTF32 operand split of A and B in one launch (grid-stride over both).
// kHiCopy = true : hi = rna_tf32(x) written out, lo = x - hi (exact)
// kHiCopy = false: the GEMM reads x itself as hi (the tensor core uses only the
//                  top 19 bits of an fp32 operand, i.e. trunc_tf32(x)), so only
//                  lo = x - trunc_tf32(x) (exact, <= 13 significant bits) is written:
//                  8 bytes of traffic per element instead of 12.
template <bool kHiCopy>
__global__ void split_tf32_kernel(const float4* __restrict__ a, float4* __restrict__ a_hi,
                                  float4* __restrict__ a_lo, int64_t na4,
                                  const float4* __restrict__ b, float4* __restrict__ b_hi,
                                  float4* __restrict__ b_lo, int64_t nb4, int64_t row_len,
                                  bool mn_major, const FixList fa, const FixList fb) {
  pdl_trigger();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t total = na4 + nb4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const bool is_a = i < na4;
    const int64_t j = is_a ? i : i - na4;
    const float4 v = __ldg((is_a ? a : b) + j);
    float4 h, l;
    // residual vs what the tensor core multiplies (ftz(trunc_tf32) of hi and lo;
    // fix.h): only FP32-subnormal hi/lo parts miss it by more than 2^-20
#define MTNN_SPLIT(c, q)                                                       \
  {                                                                            \
    h.c = tf32_hi<kHiCopy>(v.c);                                               \
    l.c = v.c - h.c;                                                           \
    const float r = fabsf(v.c) < 0x1p-100f ? v.c - tf32_represented<kHiCopy>(v.c) : 0.f; \
    if (fabsf(r) > kFixRelTF32 * fabsf(v.c)) {                                 \
      const int64_t e = 4 * j + q, u = e / row_len, w = e % row_len;           \
      fix_push(is_a ? fa : fb, mn_major ? w : u, mn_major ? u : w, r);         \
    }                                                                          \
  }
    MTNN_SPLIT(x, 0) MTNN_SPLIT(y, 1) MTNN_SPLIT(z, 2) MTNN_SPLIT(w, 3)
#undef MTNN_SPLIT
    if (kHiCopy) (is_a ? a_hi : b_hi)[j] = h;
    (is_a ? a_lo : b_lo)[j] = l;
  }
}

// ------------------------------------------------------------------- host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

static int get_encode(EncodeTiledFn* out) {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (err == cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) return fail(MTNN_ECUDA, "cuTensorMapEncodeTiled unavailable (%s)", cudaGetErrorString(err));
  *out = fn;
  return MTNN_OK;
}

static thread_local CUtensorMapDataType encode_dtype = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;

static int encode(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                  const uint64_t* strides_bytes /* rank-1 */, const uint32_t* box,
                  CUtensorMapSwizzle swz) {
  EncodeTiledFn fn;
  MTNN_TRY(get_encode(&fn));
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) { d[i] = dims[i]; b[i] = box[i]; es[i] = 1; }
  for (int i = 0; i < rank - 1; ++i) st[i] = strides_bytes[i];
  CUresult r = fn(map, encode_dtype, rank, const_cast<void*>(base), d, st, b,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MTNN_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return MTNN_OK;
}

// Launches a GEMM kernel with programmatic stream serialization (see pdl_wait);
// MTNN_PDL=0 launches it fully serialised.
static bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MTNN_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class Kern, class... Args>
static int launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                      Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  MTNN_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  return MTNN_OK;
}

template <int BN, bool B_MN, class Kind, int kConv = 0>
static int launch_impl(const void* ahi, const void* alo, const void* bhi,
                       const void* blo, float* out, const Params& p, int grid,
                       cudaStream_t s) {
  constexpr bool kF16Conv = (kConv == 1 || kConv == 2) && Kind::kScaled;
  using S = Smem<BN, kF16Conv ? kF16ConvRows * 128 : 0, Roles<kF16Conv>::kEpi>;
  constexpr int kNumThreads = Roles<kF16Conv>::kThreads;
  CUtensorMap mah, mal, mbh, mbl, mc;
  const uint64_t eb = Kind::kElemBytes;
  // F16S operand converted in-kernel: its fp32 rows as [BK k][128 rows] boxes
  // of 128-byte rows (SWIZZLE_128B), into the stage's raw slot
  auto encode_raw = [&](CUtensorMap* map, const void* base, int64_t rows) {
    encode_dtype = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const uint64_t dims[2] = {(uint64_t)p.k, (uint64_t)rows};
    const uint64_t str[1] = {(uint64_t)p.k * 4};
    const uint32_t box[2] = {(uint32_t)Kind::BK, (uint32_t)kF16ConvRows};
    return encode(map, base, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
  };
  encode_dtype = Kind::kTmaType;
  if (kF16Conv && kConv == 1) {
    MTNN_TRY(encode_raw(&mah, ahi, p.m));
    mal = mah;  // never used
  } else {
    const uint64_t dims[2] = {(uint64_t)p.k, (uint64_t)p.m};
    const uint64_t str[1] = {(uint64_t)p.k * eb};
    const uint32_t box[2] = {(uint32_t)Kind::BK, BM};
    MTNN_TRY(encode(&mah, ahi, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B));
    MTNN_TRY(encode(&mal, alo ? alo : ahi, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B));
  }
  encode_dtype = Kind::kTmaType;
  if (!blo) blo = bhi;  // computed in-kernel (kConv == 2): the map is never used
  if (kF16Conv && kConv == 2) {
    MTNN_TRY(encode_raw(&mbh, bhi, p.n));
    mbl = mbh;
  } else if (!B_MN) {
    const uint64_t dims[2] = {(uint64_t)p.k, (uint64_t)p.n};
    const uint64_t str[1] = {(uint64_t)p.k * eb};
    const uint32_t box[2] = {(uint32_t)Kind::BK, BN};
    MTNN_TRY(encode(&mbh, bhi, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B));
    MTNN_TRY(encode(&mbl, blo, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B));
  } else {
    const uint64_t dims[2] = {(uint64_t)p.n, (uint64_t)p.k};
    const uint64_t str[1] = {(uint64_t)p.n * eb};
    const uint32_t box[2] = {(uint32_t)Kind::kMnBox, (uint32_t)Kind::BK};
    MTNN_TRY(encode(&mbh, bhi, 2, dims, str, box, Kind::kMnSwizzle));
    MTNN_TRY(encode(&mbl, blo, 2, dims, str, box, Kind::kMnSwizzle));
  }
  encode_dtype = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  {
    const uint64_t dims[3] = {(uint64_t)p.ldc, (uint64_t)p.m, (uint64_t)p.splits};
    const uint64_t str[2] = {(uint64_t)p.ldc * 4, (uint64_t)p.ldc * p.m * 4};
    const uint32_t box[3] = {16, 32, 1};
    MTNN_TRY(encode(&mc, out, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B));
  }
  auto kern = gemm_tc3x_kernel<BN, B_MN, Kind, kConv>;
  MTNN_TRY(set_max_dynamic_smem((const void*)kern, S::kTotal));
  {
    KernelTimer timer(Kind::kScaled ? MTNN_KCLASS_GEMM_TC_F16S : MTNN_KCLASS_GEMM_TC,
                      2.0 * (double)p.m * (double)p.n * (double)p.k, s);
    MTNN_TRY(launch_pdl(kern, dim3(grid), dim3(kNumThreads), S::kTotal, s, mah, mal, mbh, mbl, mc, p));
  }
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}


// ======================================================================
// CTA-pair variant (tcgen05 cta_group::2): a cluster of two CTAs on one TPC
// computes a 256 x 256 output tile with M = 256 MMAs issued by the leader CTA.
// Each CTA loads its own 128 rows of A and HALF (128 rows) of the tile's B, so
// per SM the smem/L2 operand traffic per flop drops by a third against the
// 128 x 256 single-CTA tile (A 128 + B 256 rows per 128 x 256 outputs -> A 128 +
// B 128), and each wave of 74 pair tiles touches half as many B panels, which
// halves the DRAM re-reads. Per CTA: 6-stage ring of 32 KiB stages (A h/l +
// half-B h/l), 2 x 256 TMEM columns (its 128 rows of the double-buffered
// accumulator), the same FP32-promotion epilogue on its own rows.
// Barriers: full[s] lives in the leader (2 arrivals: the leader's expect_tx and
// the peer's remote arrive; both CTAs' TMA bytes complete on it); the leader's
// commits multicast to empty[s] / tfull[] in both CTAs; tempty[] in the leader
// counts the epilogue warps of both CTAs.
// Fused all-gather: the epilogue also stores every C tile into up to
// kMaxPeers other C buffers (peer GPUs' memory mapped into this process over
// NVLink, CUDA IPC), so the gather overlaps the MMAs tile by tile.
constexpr int kMaxPeers = 7;
struct PeerMaps {
  CUtensorMap map[kMaxPeers];
};
constexpr int kPairStages = 6;
constexpr int kPairBN = 256;            // output tile N (both CTAs)
constexpr int kPairHalfN = kPairBN / 2;  // B rows loaded per CTA
struct PairSmem {
  static constexpr int kABytes = BM * 64;
  static constexpr int kBBytes = kPairHalfN * 64;
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;  // 32 KiB
  static constexpr int kRingBytes = kPairStages * kStageBytes;
  static constexpr int kStagingBytes = 32 * 16 * 4;
  static constexpr int kEpiBytes = kEpiWarps * kStagingBytes;
  static constexpr int kBarBytes = 256;
  static constexpr int kTotal = 1024 + kRingBytes + kEpiBytes + kBarBytes;
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
// arrive on the barrier at the same offset in cluster CTA `cta`
__device__ __forceinline__ void mbar_arrive_cta(uint32_t bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(bar),
      "r"(cta)
      : "memory");
}
// 2-SM TMA load: lands in this CTA's smem, completes on the LEADER's barrier
// (peer bit of the cluster address cleared)
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map,
                                                 uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
template <bool kF16>
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  const uint32_t z = 0;
  if constexpr (kF16) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(
            tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(z)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n\t}" ::"r"(
            tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(z)
        : "memory");
  }
}
// commit this CTA's outstanding MMAs; arrive on the barrier in both CTAs
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .b16 msk;\n\t"
      "mov.b16 msk, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], msk;\n\t}" ::"r"(bar)
      : "memory");
}

// units are (k-split, pair tile); pair tile = (pair of m-tiles, n-tile), grouped
// raster over kGroupM / 2 pairs (the same 16 m-tiles as the single-CTA order)
__device__ __forceinline__ void pair_unit_coords(int u, const Params& p, int& split, int& tmp,
                                                 int& tn) {
  const int tiles = p.tiles_mp * p.tiles_n;
  split = u / tiles;
  const int t = u - split * tiles;
  const int kGroupP = p.group_m;
  const int per_group = kGroupP * p.tiles_n;
  const int group = t / per_group;
  const int first = group * kGroupP;
  const int gm = min(kGroupP, p.tiles_mp - first);
  const int r = t - group * per_group;
  tmp = first + r % gm;
  tn = r / gm;
}

template <bool B_MN, class Kind>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
gemm_tc3x_pair_kernel(const __grid_constant__ CUtensorMap map_ahi,
                      const __grid_constant__ CUtensorMap map_alo,
                      const __grid_constant__ CUtensorMap map_bhi,
                      const __grid_constant__ CUtensorMap map_blo,
                      const __grid_constant__ CUtensorMap map_c, const Params p,
                      const __grid_constant__ PeerMaps peers) {
  using S = PairSmem;
  constexpr int BN = kPairBN;
  constexpr int kColsPerWarp = BN / 4;
  constexpr bool kChunkB = B_MN && Kind::kScaled;  // see gemm_tc3x_kernel
  constexpr int kScaleKb = kScaleChunkK / Kind::BK;
  static_assert(kColsPerWarp % 32 == 0, "chunk scales: 32-column groups per epilogue warp");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* epi = smem + S::kRingBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi + S::kEpiBytes);
  uint64_t* full_bar = bars;                          // [kPairStages] (leader's used)
  uint64_t* empty_bar = bars + kPairStages;           // [kPairStages]
  uint64_t* tfull_bar = bars + 2 * kPairStages;       // [2]
  uint64_t* tempty_bar = bars + 2 * kPairStages + 2;  // [2] (leader's used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kPairStages + 4);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x / 2;
  const int nclusters = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_c)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kPairStages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 2);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&tfull_bar[s]), 1);
      mbar_init(smem_u32(&tempty_bar[s]), 2 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();
  pdl_trigger();  // the next call's split may be scheduled (it waits for us)
  const int kb_per = p.kblocks_per_split;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cluster; u < p.units; u += nclusters) {
        int split, tmp, tn;
        pair_unit_coords(u, p, split, tmp, tn);
        const int tm = 2 * tmp + (int)rank;
        const int kb0 = split * kb_per;
        const int kb1 = min(p.total_kblocks, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
          const uint32_t fb = smem_u32(&full_bar[stage]);
          const uint32_t st = smem_u32(ring + stage * S::kStageBytes);
          const int kx = kb * Kind::BK;
          const int brow = tn * BN + (int)rank * kPairHalfN;
          tma_load_2d_pair(st, &map_ahi, fb, kx, tm * BM);
          tma_load_2d_pair(st + S::kABytes, &map_alo, fb, kx, tm * BM);
          if (!B_MN) {
            tma_load_2d_pair(st + 2 * S::kABytes, &map_bhi, fb, kx, brow);
            tma_load_2d_pair(st + 2 * S::kABytes + S::kBBytes, &map_blo, fb, kx, brow);
          } else {
            // this CTA's 128 columns of B^T: boxes of [BK k-rows][kMnBox columns],
            // one MN group of the canonical MN-major layout each, kMnLBO apart
#pragma unroll
            for (int g = 0; g < kPairHalfN / Kind::kMnBox; ++g) {
              tma_load_2d_pair(st + 2 * S::kABytes + g * Kind::kMnLBO, &map_bhi, fb,
                               brow + g * Kind::kMnBox, kx);
              tma_load_2d_pair(st + 2 * S::kABytes + S::kBBytes + g * Kind::kMnLBO, &map_blo, fb,
                               brow + g * Kind::kMnBox, kx);
            }
          }
          if (leader) mbar_expect_tx(fb, 2 * S::kStageBytes);  // both CTAs' bytes
          else mbar_arrive_cta(fb, 0);
          if (++stage == kPairStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    if (leader) {
      constexpr uint32_t idesc = (1u << 4) | (Kind::kFmt << 7) | (Kind::kFmt << 10) |
                                 ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)(256 >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cluster; u < p.units; u += nclusters) {
        const int split = u / (p.tiles_mp * p.tiles_n);
        const int kb0 = split * kb_per;
        const int kb1 = min(p.total_kblocks, kb0 + kb_per);
        for (int kc = kb0; kc < kb1; kc += p.chunk_kb) {
          const int kce = min(kb1, kc + p.chunk_kb);
          mbar_wait(smem_u32(&tempty_bar[acc]), acc_phase ^ 1);
          tc_fence_after();
          const uint32_t tmem_d = tmem_base + acc * BN;
          for (int kb = kc; kb < kce; ++kb) {
            mbar_wait(smem_u32(&full_bar[stage]), phase);
            tc_fence_after();
            if (elect_one()) {
              const uint32_t a_hi = smem_u32(ring + stage * S::kStageBytes);
              const uint32_t a_lo = a_hi + S::kABytes;
              const uint32_t b_hi = a_hi + 2 * S::kABytes;
              const uint32_t b_lo = b_hi + S::kBBytes;
#pragma unroll
              for (int ks = 0; ks < Kind::BK / Kind::UMMA_K; ++ks) {
                const uint64_t dah = make_sdesc(a_hi + ks * 32, 16, 512, kLayoutSW64);
                const uint64_t dal = make_sdesc(a_lo + ks * 32, 16, 512, kLayoutSW64);
                uint64_t dbh, dbl;
                if (!B_MN) {
                  dbh = make_sdesc(b_hi + ks * 32, 16, 512, kLayoutSW64);
                  dbl = make_sdesc(b_lo + ks * 32, 16, 512, kLayoutSW64);
                } else {
                  dbh = make_sdesc(b_hi + ks * Kind::kMnKStep, Kind::kMnLBO, Kind::kMnSBO,
                                   Kind::kMnLayout);
                  dbl = make_sdesc(b_lo + ks * Kind::kMnKStep, Kind::kMnLBO, Kind::kMnSBO,
                                   Kind::kMnLayout);
                }
                const uint32_t accum = (kb == kc && ks == 0) ? 0u : 1u;
                tc_mma_pair<Kind::kScaled>(tmem_d, dal, dbh, idesc, accum);
                tc_mma_pair<Kind::kScaled>(tmem_d, dah, dbl, idesc, 1u);
                tc_mma_pair<Kind::kScaled>(tmem_d, dah, dbh, idesc, 1u);
              }
              tc_commit_pair(smem_u32(&empty_bar[stage]));
              if (kb == kce - 1) tc_commit_pair(smem_u32(&tfull_bar[acc]));
            }
            __syncwarp();
            if (++stage == kPairStages) { stage = 0; phase ^= 1; }
          }
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ===================== epilogue (both CTAs, own 128 rows) =====================
    const int e = warp - kEpiWarp0;
    const int q = warp % 4;
    const int h = e / 4;
    uint8_t* stg = epi + e * S::kStagingBytes;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = cluster; u < p.units; u += nclusters) {
      int split, tmp, tn;
      pair_unit_coords(u, p, split, tmp, tn);
      const int tm = 2 * tmp + (int)rank;
      const int kb0 = split * kb_per;
      const int kb1 = min(p.total_kblocks, kb0 + kb_per);
      const int64_t row = (int64_t)tm * BM + q * 32 + lane;
      const int64_t col0 = (int64_t)tn * BN + h * kColsPerWarp;
      float sum[kColsPerWarp];
#pragma unroll
      for (int j = 0; j < kColsPerWarp; ++j) sum[j] = 0.f;
      float sa_pre = 1.f;  // (kTail >= 1: the tile's output scales, preloaded)
      ChunkScales<kColsPerWarp> csb{};
      for (int kc = kb0; kc < kb1; kc += p.chunk_kb) {
        // (the chunk's column scales load while the MMAs of the chunk finish)
        ChunkScales<kColsPerWarp> cs{};
        if (kChunkB) cs = load_chunk_scales<kColsPerWarp>(p.inv_scale_b, kc / kScaleKb, p.n, col0, lane);
        if (kTail >= 1 && Kind::kScaled && kc + p.chunk_kb >= kb1) {
          // the output scales load while the tile's last chunk is still in the
          // tensor core (as in gemm_tc3x_kernel)
          if (row < p.m) sa_pre = __ldg(p.inv_scale_a + row);
          if (!kChunkB) csb = load_chunk_scales<kColsPerWarp>(p.inv_scale_b, 0, p.n, col0, lane);
        }
        mbar_wait(smem_u32(&tfull_bar[acc]), acc_phase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + h * kColsPerWarp;
#pragma unroll
        for (int c = 0; c < kColsPerWarp / 16; ++c) {
          uint32_t r[16];
          tmem_ld_32x32b_x16(taddr + c * 16, r);
          tmem_ld_wait();
          if (kChunkB) {
            add_chunk_scaled(sum + c * 16, r, cs, c);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) sum[c * 16 + j] += __uint_as_float(r[j]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cta(smem_u32(&tempty_bar[acc]), 0);  // the leader's
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      const float sa = kTail >= 1 ? sa_pre : (Kind::kScaled && row < p.m) ? __ldg(p.inv_scale_a + row) : 1.f;
#pragma unroll
      for (int c = 0; c < kColsPerWarp / 16; ++c) {
        if (lane == 0) tma_store_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int pj = j ^ ((lane >> 1) & 3);
          float4 v = make_float4(sum[c * 16 + 4 * j], sum[c * 16 + 4 * j + 1],
                                 sum[c * 16 + 4 * j + 2], sum[c * 16 + 4 * j + 3]);
          if (Kind::kScaled && kChunkB) {
            v.x *= sa; v.y *= sa; v.z *= sa; v.w *= sa;
          } else if (kTail >= 1 && Kind::kScaled) {
            const int cc = c * 16 + 4 * j;
            const float src = csb.v[cc / 32];
            v.x = (v.x * sa) * __shfl_sync(0xffffffffu, src, (cc + 0) % 32);
            v.y = (v.y * sa) * __shfl_sync(0xffffffffu, src, (cc + 1) % 32);
            v.z = (v.z * sa) * __shfl_sync(0xffffffffu, src, (cc + 2) % 32);
            v.w = (v.w * sa) * __shfl_sync(0xffffffffu, src, (cc + 3) % 32);
          } else if (Kind::kScaled) {
            const int64_t cj = col0 + c * 16 + 4 * j;
            const float4 sb = cj < p.n ? __ldg(reinterpret_cast<const float4*>(p.inv_scale_b + cj))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            v.x = (v.x * sa) * sb.x;
            v.y = (v.y * sa) * sb.y;
            v.z = (v.z * sa) * sb.z;
            v.w = (v.w * sa) * sb.w;
          }
          *reinterpret_cast<float4*>(stg + lane * 64 + pj * 16) = v;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&map_c, smem_u32(stg), tn * BN + h * kColsPerWarp + c * 16,
                       tm * BM + q * 32, split);
          for (int d = 0; d < p.npeers; ++d)  // the same tile into each peer's C
            tma_store_3d(&peers.map[d], smem_u32(stg), tn * BN + h * kColsPerWarp + c * 16,
                         tm * BM + q * 32, split);
          tma_store_commit();
        }
      }
    }
    if (lane == 0) tma_store_wait_all();
  }

  tc_fence_before();
  __syncwarp();  // reconverge the role branches: the cluster barrier is warp-aligned
  cluster_sync_all();  // both CTAs done with the accumulator before it is freed
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(2 * BN));
  }
}

template <bool B_MN, class Kind>
static int launch_pair_impl(const void* ahi, const void* alo, const void* bhi, const void* blo,
                            float* out, const Params& p, int clusters, cudaStream_t s,
                            float* const* peer_out = nullptr) {
  using S = PairSmem;
  CUtensorMap mah, mal, mbh, mbl, mc;
  PeerMaps peers;
  memset(&peers, 0, sizeof(peers));
  const uint64_t eb = Kind::kElemBytes;
  encode_dtype = Kind::kTmaType;
  {
    const uint64_t dims[2] = {(uint64_t)p.k, (uint64_t)p.m};
    const uint64_t str[1] = {(uint64_t)p.k * eb};
    const uint32_t box[2] = {(uint32_t)Kind::BK, BM};
    MTNN_TRY(encode(&mah, ahi, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B));
    MTNN_TRY(encode(&mal, alo, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B));
  }
  if (!B_MN) {
    const uint64_t dims[2] = {(uint64_t)p.k, (uint64_t)p.n};
    const uint64_t str[1] = {(uint64_t)p.k * eb};
    const uint32_t box[2] = {(uint32_t)Kind::BK, (uint32_t)kPairHalfN};
    MTNN_TRY(encode(&mbh, bhi, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B));
    MTNN_TRY(encode(&mbl, blo, 2, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B));
  } else {
    const uint64_t dims[2] = {(uint64_t)p.n, (uint64_t)p.k};
    const uint64_t str[1] = {(uint64_t)p.n * eb};
    const uint32_t box[2] = {(uint32_t)Kind::kMnBox, (uint32_t)Kind::BK};
    MTNN_TRY(encode(&mbh, bhi, 2, dims, str, box, Kind::kMnSwizzle));
    MTNN_TRY(encode(&mbl, blo, 2, dims, str, box, Kind::kMnSwizzle));
  }
  encode_dtype = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  {
    const uint64_t dims[3] = {(uint64_t)p.ldc, (uint64_t)p.m, (uint64_t)p.splits};
    const uint64_t str[2] = {(uint64_t)p.ldc * 4, (uint64_t)p.ldc * p.m * 4};
    const uint32_t box[3] = {16, 32, 1};
    MTNN_TRY(encode(&mc, out, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B));
    for (int d = 0; d < p.npeers; ++d)
      MTNN_TRY(encode(&peers.map[d], peer_out[d], 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B));
  }
  auto kern = gemm_tc3x_pair_kernel<B_MN, Kind>;
  MTNN_TRY(set_max_dynamic_smem((const void*)kern, S::kTotal));
  {
    KernelTimer timer(Kind::kScaled ? MTNN_KCLASS_GEMM_TC_F16S : MTNN_KCLASS_GEMM_TC,
                      2.0 * (double)p.m * (double)p.n * (double)p.k, s);
    MTNN_TRY(launch_pdl(kern, dim3(2 * clusters), dim3(kThreads), S::kTotal, s, mah, mal, mbh, mbl,
                        mc, p, peers));
  }
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}
}  // namespace tc

// Split mode: "trunc" (default, lo only; the tensor core truncates the raw
// fp32 operand to tf32 itself) or "rna" (hi and lo materialised) via MTNN_SPLIT.
static bool split_mode_hi_copy() {
  static const bool hi = [] {
    const char* e = getenv("MTNN_SPLIT");
    return e != nullptr && e[0] == 'r';
  }();
  return hi;
}

// k-blocks per TMEM accumulation chunk (the FP32 promotion period); both kinds
// default to 48 MMA accumulations per chunk (tf32: 8 x 16 = 128 k; f16: 8 x 32 =
// 256 k). MTNN_CHUNK_KB overrides (testing).
static int chunk_kblocks(TcKind) {
  static const int v = [] {
    const char* e = getenv("MTNN_CHUNK_KB");
    const int x = e ? atoi(e) : 0;
    return x > 0 ? x : 8;
  }();
  return v;
}

// MN-major F16S B has one scale per kScaleChunkK k-rows (split_f16.cu): every
// promotion chunk and every k-split must then lie inside one scale chunk —
// chunk_kb divides the scale chunk's k-blocks and k-splits start on its
// boundaries (kblocks_per_split rounded up to a multiple of it).
static void align_scale_chunks(tc::Params& p, TcKind kind, bool b_is_nk, int splits) {
  p.kblocks_per_split = (p.total_kblocks + splits - 1) / splits;
  if (kind == TcKind::F16S && !b_is_nk) {
    constexpr int sk = kScaleChunkK / tc::KindF16S::BK;
    if (sk % p.chunk_kb != 0) p.chunk_kb = sk;
    p.kblocks_per_split = (p.kblocks_per_split + sk - 1) / sk * sk;
  }
}

// TF32 kind, opt-in (MTNN_TF32_INKERNEL=1): the kernel computes the larger
// operand's lo half itself so only the smaller one is pre-split (1 = A, 2 = B).
// Measured on the B200 it gains <= 3% on skinny shapes (which are bound by tile
// waste and split-K waves, not split traffic) and costs ~22% on compute-bound
// shapes (smem/ALU contention with the MMA), so it is off by default.
static int tf32_inkernel_operand(int64_t m, int64_t n) {
  static const bool on = [] {
    const char* e = getenv("MTNN_TF32_INKERNEL");
    return e && e[0] == '1';
  }();
  if (!on) return 0;
  return m >= n ? 1 : 2;
}

// F16S kind: skinny problems (the output's short side <= 256 by default, the
// long side >= 1024) read the long operand raw and split it in-kernel, so DRAM
// sees 4 B (row-max pass) + 4 B (GEMM) per element of it instead of the split's
// 8 B plus the GEMM's 4 B; those shapes are HBM-bound on that operand. Wide
// problems keep the pre-split operands: each operand tile there is consumed by
// many output tiles, so converting per tile would multiply the conversion work.
// MTNN_F16S_INKERNEL=0 disables; MTNN_F16S_INKERNEL_MAX overrides the threshold.
// mtnn_config_set("f16s_inkernel_max_short", v) changes it at run time.
static std::atomic<int64_t> g_f16s_inkernel_max{-1};

int64_t f16s_inkernel_max_short() {
  int64_t v = g_f16s_inkernel_max.load(std::memory_order_relaxed);
  if (v >= 0) return v;
  const char* e = getenv("MTNN_F16S_INKERNEL");
  const char* t = getenv("MTNN_F16S_INKERNEL_MAX");
  const long long x = t ? atoll(t) : 0;
  v = (e && e[0] == '0') ? 0 : (x > 0 ? x : 256);
  g_f16s_inkernel_max.store(v, std::memory_order_relaxed);
  return v;
}

void set_f16s_inkernel_max_short(int64_t v) { g_f16s_inkernel_max.store(v, std::memory_order_relaxed); }

static int f16s_inkernel_operand(int64_t m, int64_t n, bool b_is_nk) {
  const int64_t max_short = f16s_inkernel_max_short();
  const int64_t lo = std::min(m, n), hi = std::max(m, n);
  if (lo > max_short || hi < 1024) return 0;
  if (m >= n) return 1;
  return b_is_nk ? 2 : 0;  // B^T (MN-major) is always pre-split
}

int tc_inkernel_operand(int64_t m, int64_t n, bool b_is_nk, TcKind kind) {
  return kind == TcKind::TF32 ? tf32_inkernel_operand(m, n) : f16s_inkernel_operand(m, n, b_is_nk);
}

// Operands only: A and B (or B^T) can feed TMA (16-byte aligned bases and row
// strides; F16S halves need k % 8; MN-major B^T needs n % 16 column groups).
bool tc_eligible_operands(const float* A, const float* B, int64_t m, int64_t n, int64_t k,
                          bool b_is_nk, TcKind kind) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (m <= 0 || n <= 0 || k <= 0) return false;
  if (k % 4 != 0) return false;                          // 16-byte TMA row strides (fp32)
  if (kind == TcKind::F16S && k % 8 != 0) return false;  // 16-byte rows of fp16 halves
  if (!b_is_nk && n % 16 != 0) return false;             // MN-major column groups
  if (m > (1LL << 31) - 1 || n > (1LL << 31) - 1 || k > (1LL << 31) - 1) return false;
  return al16(A) && al16(B);
}

// Operands and C: C is stored by TMA too (n % 4, 16-byte aligned base).
bool tc_eligible(const float* A, const float* B, const float* C, int64_t m, int64_t n,
                 int64_t k, bool b_is_nk, TcKind kind) {
  if (!tc_eligible_operands(A, B, m, n, k, b_is_nk, kind)) return false;
  return n % 4 == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Split one operand into its hi/lo halves (+ per-row scales for F16S).
// K-major (rows x k: A, or B of NT) or MN-major (k x cols: B^T of NN).
int tc_prepare(const float* X, int64_t rows, int64_t k, bool mn_major, TcKind kind,
               bool inkernel, ScratchBuffer& ws, FixHandle* fh, TcOperand* out, cudaStream_t s) {
  const DeviceInfo* di = nullptr;
  MTNN_TRY(device_info(&di));
  const int64_t count = rows * k;  // MN-major: k x rows (rows = n)
  // residual list (fix.h), carved from the end of the workspace
  const bool track = fh != nullptr && fixup_enabled() && !(inkernel && kind == TcKind::TF32);
  const unsigned cap = track ? fix_capacity(count) : 0;
  const size_t fix_bytes = track ? fix_entry_bytes(cap) : 0;
  auto attach = [&](uint8_t* entries) -> int {
    if (!track) {
      out->fix = FixList{};
      return MTNN_OK;
    }
    MTNN_TRY(fix_attach(fh, entries, cap, 0, s));
    out->fix = fh->list;
    return MTNN_OK;
  };
  if (inkernel) {
    // split in-kernel from the raw rows (K-major only); F16S needs the row scales
    if (mn_major && kind == TcKind::F16S)
      return fail(MTNN_EINVAL, "in-kernel F16S split needs a K-major operand");
    out->hi = X;
    out->lo = nullptr;
    out->inv_scale = nullptr;
    out->fix = FixList{};
    if (kind == TcKind::F16S) {
      const size_t osc = align256((size_t)rows * sizeof(float));
      MTNN_TRY(ws.alloc(osc + fix_bytes, s));
      float* inv = static_cast<float*>(ws.ptr);
      MTNN_TRY(attach(static_cast<uint8_t*>(ws.ptr) + osc));
      MTNN_TRY(launch_rowmax_f16(X, inv, rows, k, out->fix, s));
      out->inv_scale = inv;
    }
    return MTNN_OK;
  }
  if (kind == TcKind::TF32) {
    const bool hi_copy = split_mode_hi_copy();
    const size_t olo = align256((size_t)((hi_copy ? 2 : 1) * count) * sizeof(float));
    MTNN_TRY(ws.alloc(olo + fix_bytes, s));
    float* lo = static_cast<float*>(ws.ptr);
    float* hi = hi_copy ? lo + count : nullptr;
    MTNN_TRY(attach(static_cast<uint8_t*>(ws.ptr) + olo));
    const int64_t total4 = count / 4;
    const int64_t blocks =
        std::max<int64_t>(1, std::min<int64_t>((total4 + 255) / 256, (int64_t)di->sm_count * 8));
    KernelTimer timer(MTNN_KCLASS_SPLIT, (hi_copy ? 12.0 : 8.0) * (double)count, s);
    auto x4 = reinterpret_cast<const float4*>(X);
    // entries are (operand row, k index): for MN-major B^T (k x n) element
    // p * n + j is operand row j, k index p
    const int64_t row_len = mn_major ? rows : k;
    if (hi_copy)
      tc::split_tf32_kernel<true><<<(unsigned)blocks, 256, 0, s>>>(
          x4, reinterpret_cast<float4*>(hi), reinterpret_cast<float4*>(lo), total4, nullptr,
          nullptr, nullptr, 0, row_len, mn_major, out->fix, FixList{});
    else
      tc::split_tf32_kernel<false><<<(unsigned)blocks, 256, 0, s>>>(
          x4, nullptr, reinterpret_cast<float4*>(lo), total4, nullptr, nullptr, nullptr, 0,
          row_len, mn_major, out->fix, FixList{});
    MTNN_CUDA_TRY(cudaGetLastError());
    out->hi = hi_copy ? static_cast<const void*>(hi) : X;
    out->lo = lo;
    out->inv_scale = nullptr;
    return MTNN_OK;
  }
  // F16S: [h | l | 1/s | residual entries]; MN-major: 1/s per (256-row chunk, column)
  const size_t oh = align256((size_t)count * 2);
  const int64_t scale_rows = mn_major ? (k + kScaleChunkK - 1) / kScaleChunkK : 1;
  const size_t osc = align256((size_t)(scale_rows * rows) * 4);
  MTNN_TRY(ws.alloc(2 * oh + osc + fix_bytes, s));
  uint8_t* base = static_cast<uint8_t*>(ws.ptr);
  float* inv = reinterpret_cast<float*>(base + 2 * oh);
  MTNN_TRY(attach(base + 2 * oh + osc));
  if (!mn_major) {
    MTNN_TRY(launch_split_rows_f16(X, base, base + oh, inv, rows, k, out->fix, s));
  } else {
    MTNN_TRY(launch_split_cols_f16(X, base, base + oh, inv, k, rows, out->fix, s));
  }
  out->hi = base;
  out->lo = base + oh;
  out->inv_scale = inv;
  return MTNN_OK;
}

int tc_prepare_pair(const float* A, int64_t m, const float* B, int64_t n, int64_t k,
                    bool b_mn_major, TcKind kind, int conv, ScratchBuffer& wa, ScratchBuffer& wb,
                    FixHandle* fa, FixHandle* fb, TcOperand* a, TcOperand* b, cudaStream_t s) {
  if (kind != TcKind::F16S || (b_mn_major && conv != 0)) {
    MTNN_TRY(tc_prepare(A, m, k, false, kind, conv == 1, wa, fa, a, s));
    return tc_prepare(B, n, k, b_mn_major, kind, conv == 2, wb, fb, b, s);
  }
  // F16S: [h | l | 1/s | entries] per split operand, [1/s | entries] per in-kernel
  // one; an MN-major B^T has 1/s per (256-row chunk, column)
  const bool track = fixup_enabled();
  auto layout = [&](const float* X, int64_t rows, bool ink, ScratchBuffer& ws, FixHandle* fh,
                    TcOperand* o, int64_t scale_rows = 1) {
    const size_t oh = ink ? 0 : align256((size_t)rows * k * 2);
    const size_t osc = align256((size_t)(scale_rows * rows) * 4);
    const bool t = track && fh != nullptr;
    const unsigned cap = t ? fix_capacity(rows * k) : 0;
    MTNN_TRY(ws.alloc(2 * oh + osc + (t ? fix_entry_bytes(cap) : 0), s));
    uint8_t* base = static_cast<uint8_t*>(ws.ptr);
    o->hi = ink ? static_cast<const void*>(X) : base;
    o->lo = ink ? nullptr : base + oh;
    o->inv_scale = reinterpret_cast<float*>(base + 2 * oh);
    o->fix = FixList{};
    if (t) {
      MTNN_TRY(fix_attach(fh, base + 2 * oh + osc, cap, 0, s));
      o->fix = fh->list;
    }
    return MTNN_OK;
  };
  MTNN_TRY(layout(A, m, conv == 1, wa, fa, a));
  if (b_mn_major) {
    // NN: B^T's column split and A's row split in one launch
    MTNN_TRY(layout(B, n, false, wb, fb, b, (k + kScaleChunkK - 1) / kScaleChunkK));
    return launch_split_cols_f16(B, const_cast<void*>(b->hi), const_cast<void*>(b->lo),
                                 const_cast<float*>(b->inv_scale), k, n, b->fix, s, A,
                                 const_cast<void*>(a->hi), const_cast<void*>(a->lo),
                                 const_cast<float*>(a->inv_scale), m, a->fix);
  }
  MTNN_TRY(layout(B, n, conv == 2, wb, fb, b));
  return launch_split_rows_f16_pair(
      A, conv == 1 ? nullptr : const_cast<void*>(a->hi), const_cast<void*>(a->lo),
      const_cast<float*>(a->inv_scale), m, a->fix, B, conv == 2 ? nullptr : const_cast<void*>(b->hi),
      const_cast<void*>(b->lo), const_cast<float*>(b->inv_scale), n, b->fix, k, s);
}

// Split-K factor: minimise (waves of units) x (k-blocks per unit + per-unit
// overhead) plus the partial-sum traffic a split adds (the GEMM writes `s`
// partial C's, the reduction reads them and writes C). Wave quantisation
// matters: 64 tiles x 3 splits = 192 units is two waves on 148 SMs and slower
// than 2 splits in one wave.
static int choose_splits(int tiles, int kblocks, int64_t m, int64_t n, int sms,
                         double* time_out = nullptr) {
  constexpr double kKblockSeconds = 0.5e-6;  // ~6 MMAs x 128 clk at ~1.6 GHz
  constexpr double kUnitOverheadKb = 2.0;    // prologue + epilogue drain, in k-blocks
  constexpr double kHbm = 5.0e12;
  constexpr double kReduceLaunchSeconds = 4.0e-6;
  if (tiles >= 4 * sms || kblocks < 8) {
    if (time_out) *time_out = std::ceil((double)tiles / sms) * (kblocks + kUnitOverheadKb) * kKblockSeconds;
    return 1;
  }
  const double mn = (double)m * (double)n;
  int best = 1;
  double best_t = 1e300;
  for (int s = 1; s <= 32 && s <= kblocks / 4; ++s) {
    const int per = (kblocks + s - 1) / s;
    const int real_s = (kblocks + per - 1) / per;
    if (real_s != s) continue;
    const double waves = std::ceil((double)tiles * s / sms);
    double t = waves * (per + kUnitOverheadKb) * kKblockSeconds;
    // split-K: partial write + re-read + the reduce kernel's launch and ramp
    // (~4 us measured on tiny outputs, where it used to be worth the split)
    if (s > 1) t += 4.0 * (2.0 * s + 1.0) * mn / kHbm + kReduceLaunchSeconds;
    if (t < best_t * 0.98) {  // prefer fewer splits unless clearly better
      best_t = t;
      best = s;
    }
  }
  if (time_out) *time_out = best_t;
  static const int cap = [] {  // MTNN_SPLITK_MAX: cap the factor (A/B runs)
    const char* e = getenv("MTNN_SPLITK_MAX");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  if (cap > 0 && best > cap) {
    int s = cap;
    while (s > 1 && (kblocks + (kblocks + s - 1) / s - 1) / ((kblocks + s - 1) / s) != s) --s;
    best = s;
  }
  return best;
}

// mtnn_profile_trace: phase timestamps of the single-CTA kernel's CTAs.
static std::atomic<unsigned long long*> g_trace{nullptr};
static std::atomic<int64_t> g_trace_ctas{0};
int set_gemm_trace(void* buf, int64_t ctas) {
#ifdef MTNN_TRACE
  g_trace.store(static_cast<unsigned long long*>(buf));
  g_trace_ctas.store(ctas);
  return MTNN_OK;
#else
  (void)ctas;
  if (buf == nullptr) return MTNN_OK;
  return fail(MTNN_ENOTSUP, "phase trace not compiled in (build with -DMTNN_TRACE: tools/build_variant.sh)");
#endif
}

// MN-major B^T on CTA pairs: each CTA's 128 columns are whole 64-column TMA
// boxes; n a multiple of 16 (the NN eligibility rule) keeps every box start on a
// 16-byte boundary, and boxes past n are zero-filled.
constexpr int kPairMnCols = 16;
// CTA-pair kernel switch: mtnn_config_set("tc_pair", 0/1), env MTNN_TC_PAIR=0.
static std::atomic<int> g_tc_pair{-1};
// 0 = off, 1 = on for large problems (default), 2 = whenever structurally possible (tests)
// Longest k that takes CTA pairs under tc_pair mode 1 (MTNN_PAIR_MAXK; default
// no limit).
static int64_t pair_max_k() {
  static const int64_t v = [] {
    const char* e = getenv("MTNN_PAIR_MAXK");
    const long long x = e ? atoll(e) : 0;
    return (int64_t)(x > 0 ? x : INT64_MAX);
  }();
  return v;
}

// Fewest 256 x 256 tiles that take CTA pairs under mode 1 (MTNN_PAIR_MIN_TILES).
// Per-case A/B (cases with 16-73 tiles) showed 8192 x 512 x k gaining 7-10% on
// pairs, but interleaved whole-sweep runs put 74 ahead of 32 by ~1%
// (379.7-380.5 vs 373.9-378.2 TFLOP/s), so the default stays at 74.
static int64_t pair_min_tiles() {
  static const int64_t v = [] {
    const char* e = getenv("MTNN_PAIR_MIN_TILES");
    const long long x = e ? atoll(e) : 0;
    return (int64_t)(x > 0 ? x : 74);
  }();
  return v;
}

int tc_pair_mode() {
  int v = g_tc_pair.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("MTNN_TC_PAIR");
    v = e ? std::min(2, std::max(0, atoi(e))) : 1;
    g_tc_pair.store(v, std::memory_order_relaxed);
  }
  return v;
}
void set_tc_pair_mode(int v) { g_tc_pair.store(v, std::memory_order_relaxed); }

// 256 x 256 output tiles on CTA pairs (NT, pre-split operands).
static int tc_run_pair(const TcOperand& a, const TcOperand& b, float* C, int64_t m, int64_t n,
                       int64_t k, int64_t ldc, bool b_is_nk, TcKind kind, cudaStream_t s,
                       float* const* peers = nullptr, int npeers = 0) {
  const DeviceInfo* di = nullptr;
  MTNN_TRY(device_info(&di));
  if (di->max_smem_optin < tc::PairSmem::kTotal)
    return fail(MTNN_ENOTSUP, "CTA-pair GEMM needs %d B smem, device allows %d",
                tc::PairSmem::kTotal, di->max_smem_optin);
  const int bk = kind == TcKind::F16S ? tc::KindF16S::BK : tc::KindTF32::BK;
  tc::Params p{};
  p.m = m; p.n = n; p.k = k; p.ldc = ldc;
  p.chunk_kb = chunk_kblocks(kind);
  p.inv_scale_a = a.inv_scale;
  p.inv_scale_b = b.inv_scale;
  p.tiles_m = (int)((m + tc::BM - 1) / tc::BM);
  p.tiles_mp = (p.tiles_m + 1) / 2;
  static const int group_env = [] {
    const char* e = getenv("MTNN_PAIR_GROUP");  // m-tile pairs per raster group (testing)
    return e ? atoi(e) : 0;
  }();
  p.group_m = group_env > 0 ? group_env : tc::kGroupM;  // 16 pairs = 32 m-tiles per raster group: least DRAM traffic of 2..37
  p.tiles_n = (int)((n + tc::kPairBN - 1) / tc::kPairBN);
  p.total_kblocks = (int)((k + bk - 1) / bk);
  const int pairs = di->sm_count / 2;
  const int tiles = p.tiles_mp * p.tiles_n;
  // peer stores go straight from the epilogue: no split-K partials
  int splits = npeers > 0 ? 1 : choose_splits(tiles, p.total_kblocks, m, n, pairs);
  p.npeers = npeers;
  align_scale_chunks(p, kind, b_is_nk, splits);
  splits = (p.total_kblocks + p.kblocks_per_split - 1) / p.kblocks_per_split;
  p.splits = splits;
  p.units = tiles * splits;
  const int clusters = std::min(p.units, pairs);
  float* out = C;
  ScratchBuffer part;
  if (splits > 1) {
    MTNN_TRY(part.alloc((size_t)splits * m * ldc * sizeof(float), s));
    out = static_cast<float*>(part.ptr);
  }
  int rc;
  if (kind == TcKind::F16S)
    rc = b_is_nk ? tc::launch_pair_impl<false, tc::KindF16S>(a.hi, a.lo, b.hi, b.lo, out, p, clusters, s, peers)
                 : tc::launch_pair_impl<true, tc::KindF16S>(a.hi, a.lo, b.hi, b.lo, out, p, clusters, s, peers);
  else
    rc = b_is_nk ? tc::launch_pair_impl<false, tc::KindTF32>(a.hi, a.lo, b.hi, b.lo, out, p, clusters, s, peers)
                 : tc::launch_pair_impl<true, tc::KindTF32>(a.hi, a.lo, b.hi, b.lo, out, p, clusters, s, peers);
  MTNN_TRY(rc);
  if (splits > 1) MTNN_TRY(launch_splitk_reduce(out, C, m * ldc, splits, s));
  return MTNN_OK;
}

template <int BN>
static int tc_run_bn(const TcOperand& a, const TcOperand& b, float* C, int64_t m, int64_t n,
                     int64_t k, int64_t ldc, bool b_is_nk, TcKind kind, int conv, cudaStream_t s) {
  const DeviceInfo* di = nullptr;
  MTNN_TRY(device_info(&di));
  using S = tc::Smem<BN>;
  if (di->max_smem_optin < S::kTotal)
    return fail(MTNN_ENOTSUP, "tensor-core GEMM needs %d B smem, device allows %d", S::kTotal,
                di->max_smem_optin);
  const int bk = kind == TcKind::F16S ? tc::KindF16S::BK : tc::KindTF32::BK;
  tc::Params p{};
  p.m = m; p.n = n; p.k = k; p.ldc = ldc;
  p.chunk_kb = chunk_kblocks(kind);
  p.inv_scale_a = a.inv_scale;
  p.inv_scale_b = b.inv_scale;
  p.tiles_m = (int)((m + tc::BM - 1) / tc::BM);
  p.tiles_n = (int)((n + BN - 1) / BN);
  p.total_kblocks = (int)((k + bk - 1) / bk);
  const int tiles = p.tiles_m * p.tiles_n;
  int splits = choose_splits(tiles, p.total_kblocks, m, n, di->sm_count);
  align_scale_chunks(p, kind, b_is_nk, splits);
  splits = (p.total_kblocks + p.kblocks_per_split - 1) / p.kblocks_per_split;
  p.splits = splits;
  p.units = tiles * splits;
  const int grid = std::min(p.units, di->sm_count);
  if (g_trace.load() && grid <= g_trace_ctas.load()) p.trace = g_trace.load();
  float* out = C;
  ScratchBuffer part;
  if (splits > 1) {
    MTNN_TRY(part.alloc((size_t)splits * m * ldc * sizeof(float), s));
    out = static_cast<float*>(part.ptr);
  }
  int rc;
  if (kind == TcKind::F16S && conv == 0)
    rc = b_is_nk ? tc::launch_impl<BN, false, tc::KindF16S>(a.hi, a.lo, b.hi, b.lo, out, p, grid, s)
                 : tc::launch_impl<BN, true, tc::KindF16S>(a.hi, a.lo, b.hi, b.lo, out, p, grid, s);
  else if (conv != 0 && kind == TcKind::F16S) {
    if constexpr (BN == tc::kF16ConvRows) {
      if (conv == 1)
        rc = b_is_nk ? tc::launch_impl<BN, false, tc::KindF16S, 1>(a.hi, a.lo, b.hi, b.lo, out, p, grid, s)
                     : tc::launch_impl<BN, true, tc::KindF16S, 1>(a.hi, a.lo, b.hi, b.lo, out, p, grid, s);
      else if (b_is_nk)
        rc = tc::launch_impl<BN, false, tc::KindF16S, 2>(a.hi, a.lo, b.hi, b.lo, out, p, grid, s);
      else
        rc = fail(MTNN_EINVAL, "in-kernel split of B^T (MN-major) is not supported");
    } else {
      rc = fail(MTNN_EINVAL, "in-kernel F16S split needs the 128-wide N tile");
    }
  } else if (conv == 1)
    rc = b_is_nk ? tc::launch_impl<BN, false, tc::KindTF32, 1>(a.hi, a.lo, b.hi, b.lo, out, p, grid, s)
                 : tc::launch_impl<BN, true, tc::KindTF32, 1>(a.hi, a.lo, b.hi, b.lo, out, p, grid, s);
  else if (conv == 2)
    rc = b_is_nk ? tc::launch_impl<BN, false, tc::KindTF32, 2>(a.hi, a.lo, b.hi, b.lo, out, p, grid, s)
                 : tc::launch_impl<BN, true, tc::KindTF32, 2>(a.hi, a.lo, b.hi, b.lo, out, p, grid, s);
  else
    rc = b_is_nk ? tc::launch_impl<BN, false, tc::KindTF32>(a.hi, a.lo, b.hi, b.lo, out, p, grid, s)
                 : tc::launch_impl<BN, true, tc::KindTF32>(a.hi, a.lo, b.hi, b.lo, out, p, grid, s);
  MTNN_TRY(rc);
  if (splits > 1) MTNN_TRY(launch_splitk_reduce(out, C, m * ldc, splits, s));
  return MTNN_OK;
}

// N tile: 256 (UMMA N=256, best smem-read/MMA ratio) unless n <= 128, where a
// 256-wide tile would waste half its MMAs on zero columns.
int tc_run(const TcOperand& a, const TcOperand& b, float* C, int64_t m, int64_t n, int64_t k,
           bool b_is_nk, TcKind kind, cudaStream_t s, int64_t ldc) {
  // an operand without a lo half has it computed in-kernel (TF32 only, one operand)
  const int conv = a.lo == nullptr ? 1 : b.lo == nullptr ? 2 : 0;
  if (conv && a.lo == nullptr && b.lo == nullptr)
    return fail(MTNN_EINVAL, "in-kernel operand split needs one prepared operand");
  if (conv && kind == TcKind::F16S && (conv == 1 ? a.inv_scale : b.inv_scale) == nullptr)
    return fail(MTNN_EINVAL, "in-kernel F16S split needs the operand's row scales");
  // CTA pairs for problems with enough 256 x 256 tiles to fill the chip's 74
  // TPCs at least once (split-K would otherwise be needed for occupancy).
  // Back-to-back at the power cap (tools/probe_pair_sustained.py, interleaved
  // blocks) pairs win 20% at k = 1024, 11% at 2048 and, with the current
  // kernels, 2-6% at k = 8192-16384 (65536x8192x8192: 23.7 vs 25.1 ms, 16384^3:
  // 22.7 vs 24.1 ms) although their DRAM traffic is ~1.6x the single-CTA
  // kernel's: the third of L2->SM and smem operand traffic they save is the
  // larger energy term. (An earlier build measured a 5% loss at 8192, hence
  // the MTNN_PAIR_MAXK knob.)
  const int pair = tc_pair_mode();
  if (conv == 0 && n > 128 && m > 128 && (b_is_nk || n % kPairMnCols == 0) &&
      (pair == 2 || (pair == 1 && k <= pair_max_k() && ((m + 255) / 256) * ((n + 255) / 256) >= pair_min_tiles())))
    return tc_run_pair(a, b, C, m, n, k, ldc < n ? n : ldc, b_is_nk, kind, s);
  // F16S in-kernel split: 128-wide N tile (raw slot + 4-stage ring fit the smem)
  if (n <= 128 || (conv && kind == TcKind::F16S))
    return tc_run_bn<128>(a, b, C, m, n, k, ldc < n ? n : ldc, b_is_nk, kind, conv, s);
  return tc_run_bn<256>(a, b, C, m, n, k, ldc < n ? n : ldc, b_is_nk, kind, conv, s);
}

FixRep tc_fix_rep(TcKind kind) {
  if (kind == TcKind::F16S) return FixRep::F16S;
  return split_mode_hi_copy() ? FixRep::TF32_RNA : FixRep::TF32_TRUNC;
}

// Fix-up arguments of one GEMM whose operands were prepared whole (fix.h).
static FixupArgs tc_fix_args(const float* A, const TcOperand& a, const float* B,
                             const TcOperand& b, float* const* dsts, int ndst, int64_t m, int64_t n,
                             int64_t k, int64_t ldc, bool b_is_nk, TcKind kind) {
  FixupArgs f;
  f.A = A;
  f.inv_a = a.inv_scale;
  f.inv_b = b.inv_scale;
  f.B = B;
  f.ldb = n;
  for (int d = 0; d < ndst; ++d) f.C[d] = dsts[d];
  f.ndst = ndst;
  f.ldc = ldc;
  f.m = m;
  f.n = n;
  f.k = k;
  f.b_is_nk = b_is_nk;
  f.rep = tc_fix_rep(kind);
  f.fa = a.fix;
  f.fb = b.fix;
  return f;
}

// Launches the fix-up (it resets the lists' counters on the device).
static int tc_fixup_finish(FixupArgs& f, FixHandle& fa, FixHandle& fb, cudaStream_t s) {
  if (f.fa.ctr == nullptr && f.fb.ctr == nullptr) return MTNN_OK;
  MTNN_TRY(launch_fixup(f, s));
  fa.consumed = fb.consumed = true;
  return MTNN_OK;
}

// Row block of a row-sharded NT with the all-gather fused into the epilogue:
// C_local = A_local x B^T (m_local x n, row stride n) is stored into C_local and
// into each peer pointer (the same rows of the peers' C). CTA-pair tc3xf16s
// kernel with the peer stores (the residual fix-up then adds to every copy);
// shapes it cannot take are computed locally and pushed to the peers by
// device-to-device copies on the same stream.
int gemm_nt_allgather(const float* A, const float* B, float* C_local, float* const* peers,
                      int npeers, int64_t m, int64_t n, int64_t k, cudaStream_t s) {
  if (npeers < 0 || npeers > tc::kMaxPeers)
    return fail(MTNN_EINVAL, "npeers must be in [0, %d], got %d", tc::kMaxPeers, npeers);
  if (m == 0 || n == 0) return MTNN_OK;
  const bool pair_ok = m > 128 && n > 128 && k > 0 && tc_eligible(A, B, C_local, m, n, k, true, TcKind::F16S);
  bool peers_ok = true;
  for (int d = 0; d < npeers; ++d) peers_ok = peers_ok && (reinterpret_cast<uintptr_t>(peers[d]) & 15) == 0;
  if (pair_ok && peers_ok) {
    ScratchBuffer wa, wb;
    FixHandle fa, fb;
    TcOperand a{}, b{};
    MTNN_TRY(tc_prepare_pair(A, m, B, n, k, false, TcKind::F16S, 0, wa, wb, &fa, &fb, &a, &b, s));
    MTNN_TRY(tc_run_pair(a, b, C_local, m, n, k, n, true, TcKind::F16S, s, peers, npeers));
    float* dsts[8] = {C_local};
    for (int d = 0; d < npeers; ++d) dsts[1 + d] = peers[d];
    FixupArgs f = tc_fix_args(A, a, B, b, dsts, 1 + npeers, m, n, k, n, true, TcKind::F16S);
    return tc_fixup_finish(f, fa, fb, s);
  }
  MTNN_TRY(gemm_dispatch_nt(A, B, C_local, m, n, k, s));
  for (int d = 0; d < npeers; ++d)
    MTNN_CUDA_TRY(cudaMemcpyAsync(peers[d], C_local, (size_t)(m * n) * sizeof(float),
                                  cudaMemcpyDefault, s));
  return MTNN_OK;
}

int launch_gemm_tc(const float* A, const float* B, float* C, int64_t m, int64_t n,
                   int64_t k, bool b_is_nk, TcKind kind, cudaStream_t s) {
  const char* name = kind == TcKind::F16S ? "tc3xf16s" : "tc3xtf32";
  if (!tc_eligible_operands(A, B, m, n, k, b_is_nk, kind))
    return fail(MTNN_ENOTSUP, "%s: shape/alignment not eligible (m=%lld n=%lld k=%lld)", name,
                (long long)m, (long long)n, (long long)k);
  ScratchBuffer wa, wb, wc;
  FixHandle fa, fb;
  TcOperand a{}, b{};
  const int conv = tc_inkernel_operand(m, n, b_is_nk, kind);
  MTNN_TRY(tc_prepare_pair(A, m, B, n, k, !b_is_nk, kind, conv, wa, wb, &fa, &fb, &a, &b, s));
  if (tc_eligible(A, B, C, m, n, k, b_is_nk, kind)) {
    float* dsts[1] = {C};
    FixupArgs f = tc_fix_args(A, a, B, b, dsts, 1, m, n, k, n, b_is_nk, kind);
    MTNN_TRY(tc_run(a, b, C, m, n, k, b_is_nk, kind, s));
    return tc_fixup_finish(f, fa, fb, s);
  }
  // C cannot be a TMA store target (n % 4 != 0, e.g. a 10-class output layer, or
  // an unaligned base): compute into a row-padded buffer (fixed up there) and
  // copy the n columns out (B's missing rows are TMA zero fill, so the padding
  // columns are zeros)
  const int64_t np = (n + 3) / 4 * 4;
  MTNN_TRY(wc.alloc((size_t)(m * np) * sizeof(float), s));
  float* cp = static_cast<float*>(wc.ptr);
  float* dsts[1] = {cp};
  FixupArgs f = tc_fix_args(A, a, B, b, dsts, 1, m, n, k, np, b_is_nk, kind);
  MTNN_TRY(tc_run(a, b, cp, m, n, k, b_is_nk, kind, s, np));
  MTNN_TRY(tc_fixup_finish(f, fa, fb, s));
  MTNN_CUDA_TRY(cudaMemcpy2DAsync(C, (size_t)n * 4, cp, (size_t)np * 4, (size_t)n * 4, (size_t)m,
                                  cudaMemcpyDeviceToDevice, s));
  return MTNN_OK;
}

}  // namespace mtnn
