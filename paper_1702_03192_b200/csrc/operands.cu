// Seeded synthetic operands, bit-identical to the reference harness.
//
// Reference: pkg/src/mtnn/bench.py:104-114 (make_operands): rng =
// np.random.default_rng(seed); A = rng.uniform(-1, 1, (m, k)).astype(float32)
// is drawn first, then B (n x k). numpy's default generator is PCG64 (128-bit
// LCG, XSL-RR output): state' = state * M + inc, draw = rotr64(hi ^ lo,
// state' >> 122); a double is (draw >> 11) * 2^-53 and uniform(low, high) is
// low + (high - low) * double, then rounded to float32.
//
// Generating the reference's operands on the host costs ~1 s per 2^28 draws
// and a PCIe copy; here every lane jumps to its first draw with the LCG's
// O(log n) advance and then walks the stream 32 draws at a time (one 128-bit
// multiply-add with the precomputed 32-step constants), so a warp writes 32
// consecutive floats per step. The seed's initial (state, inc) comes from
// numpy itself (bit_generator.state), so no SeedSequence restatement is needed.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.h"
#include "pdl.h"

namespace mtnn {
namespace {

using u128 = unsigned __int128;

constexpr uint64_t kMulHi = 0x2360ED051FC65DA4ull;
constexpr uint64_t kMulLo = 0x4385DF649FCCF645ull;

__host__ __device__ inline u128 pcg_mult() { return ((u128)kMulHi << 64) | kMulLo; }

// (mult, plus) of `delta` LCG steps: state_{i+delta} = mult * state_i + plus.
__host__ __device__ inline void pcg_jump(u128 inc, uint64_t delta, u128& mult, u128& plus) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  mult = acc_mult;
  plus = acc_plus;
}

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
  const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// Draw `skip + i` of the stream -> out[i], for i in [0, count).
__global__ void __launch_bounds__(256)
pcg64_uniform_kernel(float* __restrict__ out, int64_t count, uint64_t st_lo, uint64_t st_hi,
                     uint64_t inc_lo, uint64_t inc_hi, uint64_t skip, double low, double range,
                     uint64_t j32_mult_lo, uint64_t j32_mult_hi, uint64_t j32_plus_lo,
                     uint64_t j32_plus_hi, int64_t per_warp) {
  pdl_enter();
  const u128 st0 = ((u128)st_hi << 64) | st_lo;
  const u128 inc = ((u128)inc_hi << 64) | inc_lo;
  const u128 jm = ((u128)j32_mult_hi << 64) | j32_mult_lo;
  const u128 jp = ((u128)j32_plus_hi << 64) | j32_plus_lo;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t i0 = warp * per_warp;
  if (i0 >= count) return;
  const int64_t i1 = min(count, i0 + per_warp);
  // the draw for element i comes from the state after skip + i + 1 steps
  u128 m, p;
  pcg_jump(inc, skip + (uint64_t)(i0 + lane) + 1, m, p);
  u128 s = m * st0 + p;
  for (int64_t i = i0 + lane; i < i1; i += 32) {
    const double u = (double)(xsl_rr(s) >> 11) * (1.0 / 9007199254740992.0);
    out[i] = __double2float_rn(__dadd_rn(low, __dmul_rn(range, u)));
    s = jm * s + jp;
  }
}

}  // namespace

int fill_uniform_pcg64(float* out, int64_t count, const uint64_t state[4], int64_t skip,
                       double low, double high, cudaStream_t s) {
  if (count < 0 || skip < 0) return fail(MTNN_EINVAL, "count and skip must be non-negative");
  if (count == 0) return MTNN_OK;
  if (!out || !state) return fail(MTNN_EINVAL, "null pointer");
  const DeviceInfo* di = nullptr;
  MTNN_TRY(device_info(&di));
  const u128 inc = ((u128)state[3] << 64) | state[2];
  u128 jm, jp;
  pcg_jump(inc, 32, jm, jp);
  // ~8 warps of 32 x 64 draws per SM slot, at least 2048 draws per warp
  const int64_t warps_wanted = (int64_t)di->sm_count * 64;
  int64_t per_warp = std::max<int64_t>(2048, (count + warps_wanted - 1) / warps_wanted);
  per_warp = (per_warp + 31) / 32 * 32;
  const int64_t warps = (count + per_warp - 1) / per_warp;
  const int64_t blocks = (warps * 32 + 255) / 256;
  MTNN_TRY(launch_chained(pcg64_uniform_kernel, dim3((unsigned)blocks), dim3(256), 0, s, out, count,
                          state[0], state[1], state[2], state[3], (uint64_t)skip, low, high - low,
                          (uint64_t)jm, (uint64_t)(jm >> 64), (uint64_t)jp, (uint64_t)(jp >> 64),
                          per_warp));
  MTNN_CUDA_TRY(cudaGetLastError());
  return MTNN_OK;
}

}  // namespace mtnn
