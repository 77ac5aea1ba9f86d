// s2_decode.cu — the standalone K4 decode kernel and its launcher (body in s2_decode.cuh).
#include <cstdlib>

#include "s2_device.cuh"
#include "s2_decode.cuh"

namespace s2 {

// ---------------------------------------------------------------- decode (K4)

// zt/zc: the NEXT reduce's sketch table and counters, zeroed here so that the next
// compress needs no memset (plan ping-pong, s2_reduce); may be null.
// health (s2_reduce only): a set poison word (exchange timed out) replaces the whole output
// with NaN; block 0 ORs the step's status bits into the status word.
template <int R, bool BLOCKS>
__global__ void __launch_bounds__(kThreads)
k_decode(const uint32_t* __restrict__ bitmap, int64_t dim, int64_t bs,
         const float* __restrict__ table, float workers, float inv_workers, int workers_pow2,
         float* __restrict__ out, float4* __restrict__ zt, int64_t zt_n4,
         unsigned long long* __restrict__ zc, const __grid_constant__ HashParams hp,
         const __grid_constant__ DecodeHealth health) {
  zero_next(zt, zt_n4, zc);
  // in s2_reduce_many's two-stream schedule the compress that follows this decode uses the table
  // just zeroed and may start (late_wait) once every CTA has passed launch_dependents: the zeroing
  // must be visible by then.  (Elsewhere the fence costs ~1.7 µs of decode for nothing.)
  if (health.fence_zero && zt != nullptr) __threadfence();
  griddep_wait();  // bitmap + table come from the compress / exchange kernel
  griddep_launch_dependents();
  const uint32_t poisoned = health.poison != nullptr ? *reinterpret_cast<volatile const uint32_t*>(health.poison) : 0u;
  if (health.status != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    uint32_t st = poisoned ? S2_STATUS_EXCHANGE : 0u;
    if (health.counters != nullptr && health.counters[S2_CNT_NONFINITE] != 0ull) st |= S2_STATUS_NONFINITE;
    // OR into the word (decodes of one stream are ordered): a batch of reduces sharing one word
    // keeps any step's error; the caller zeroes the word before arming it
    volatile uint32_t* w = reinterpret_cast<volatile uint32_t*>(health.status);
    if (st) *w = *w | st;
  }
  if (poisoned) {  // a peer never arrived: the sums are incomplete, mark every coordinate invalid
    const float nan = __int_as_float(0x7FC00000);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x)
      out[i] = nan;
    return;
  }
  __shared__ uint16_t s_q[kWarps][kTile];
  __shared__ __align__(16) float s_v[kWarps][kTile];
  const int wib = threadIdx.x >> 5;
  const int64_t ntiles = (dim + kTile - 1) / kTile;
  if (BLOCKS) {  // block bitmaps: decode_tile_clear keeps the stage zero outside the set positions
    float4* v4 = reinterpret_cast<float4*>(s_v[wib]);
    for (int k = threadIdx.x & 31; k < kTile / 4; k += 32) v4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
  }
  DecodeCtx c{bitmap, table, out, dim, bs, workers, inv_workers, workers_pow2};
  decode_range<R, BLOCKS, BLOCKS>(c, (int64_t)blockIdx.x * kWarps + wib, (int64_t)gridDim.x * kWarps, ntiles, hp, s_q[wib],
                          s_v[wib]);
}

template <int R>
static cudaError_t launch_decode_r(const Plan& p, const uint32_t* bitmap, const float* table, int workers,
                                   float* out, float* zt, unsigned long long* zc, const DecodeHealth& health,
                                   cudaStream_t st) {
  const int64_t ntiles = (p.dim + kTile - 1) / kTile;
  // Multi-wave grid: ~3 tiles per warp (4 CTAs per SM are resident, so 8+ per SM means
  // later waves of short-lived CTAs that rebalance the tail); measured vs one resident wave:
  // ResNet-50 step 41.5 -> 40.6 µs, 4 % density 62.4 -> 60.2 µs, GPT-2-M 99 % 505 -> 471 µs
  // (cap 48 per SM: 32 -> 48 gained 1.5 % at GPT-2-M 99 % and 3 % at the LSTM row bitmap).
  // S2_DECODE_CTAS_PER_SM overrides.
  static int per_sm_env = -1;
  if (per_sm_env < 0) {
    const char* e = getenv("S2_DECODE_CTAS_PER_SM");
    per_sm_env = e && atoi(e) > 0 ? atoi(e) : 0;
  }
  int per_sm = per_sm_env;
  if (per_sm == 0) {
    const int64_t want = (ntiles + (int64_t)num_sms() * kWarps * 3 - 1) / ((int64_t)num_sms() * kWarps * 3);
    per_sm = (int)(want < 4 ? 4 : (want > 48 ? 48 : want));
  }
  const int grid = grid_for(ntiles, per_sm);
  const int pow2 = (workers & (workers - 1)) == 0;
  const float inv = 1.0f / (float)workers;
  const int64_t zn4 = zt ? ((int64_t)p.hp.rows * p.hp.cols + 3) / 4 : 0;
  float4* z4 = reinterpret_cast<float4*>(zt);
  if (p.block_size == 1)
    return launch_ex(k_decode<R, false>, grid, kThreads, 0, st, bitmap, p.dim, (int64_t)1, table, (float)workers,
                     inv, pow2, out, z4, zn4, zc, p.hp, health);
  return launch_ex(k_decode<R, true>, grid, kThreads, 0, st, bitmap, p.dim, p.block_size, table, (float)workers, inv,
                   pow2, out, z4, zn4, zc, p.hp, health);
}

cudaError_t preload_decode(const Plan& p) {
  cudaFuncAttributes fa;
  const bool blocks = p.block_size != 1;
  switch (p.hp.rows) {
#define S2_CASE(r) \
  case r: return cudaFuncGetAttributes(&fa, blocks ? k_decode<r, true> : k_decode<r, false>);
    S2_CASE(1) S2_CASE(2) S2_CASE(3) S2_CASE(4) S2_CASE(5)
#undef S2_CASE
    default: return cudaFuncGetAttributes(&fa, blocks ? k_decode<0, true> : k_decode<0, false>);
  }
}

cudaError_t launch_decode(const Plan& p, const uint32_t* bitmap, const float* table, int workers,
                          float* out, cudaStream_t st, float* zero_table, unsigned long long* zero_counters,
                          const DecodeHealth* health) {
  DecodeHealth h{};
  if (health != nullptr) h = *health;
  cudaError_t e;
  switch (p.hp.rows) {
#define S2_CASE(r) \
  case r: e = launch_decode_r<r>(p, bitmap, table, workers, out, zero_table, zero_counters, h, st); break;
    S2_CASE(1) S2_CASE(2) S2_CASE(3) S2_CASE(4) S2_CASE(5)
#undef S2_CASE
    default: e = launch_decode_r<0>(p, bitmap, table, workers, out, zero_table, zero_counters, h, st); break;
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace s2
