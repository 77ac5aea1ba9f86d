// s2_decode.cuh — the K4 decode body (sparse_decompress, sparse.py:199-214 + CountSketchTable.query,
// sketch.py:114-128), used by k_decode (s2_decode.cu) and k_query_pairs (s2_kernels.cu).
#pragma once

#include "s2_common.cuh"
#include "s2_kernels.h"

namespace s2 {

constexpr int kDecTile = 1024;  // elements per warp tile (32 bitmap words)

// lower median (element (R-1)/2 of the sorted estimates, sketch.py:127-128)
template <int R>
__device__ __forceinline__ float lower_median(float (&e)[R]) {
  if constexpr (R == 1) {
    return e[0];
  } else if constexpr (R == 2) {
    return fminf(e[0], e[1]);
  } else if constexpr (R == 3) {
    return fmaxf(fminf(e[0], e[1]), fminf(fmaxf(e[0], e[1]), e[2]));
  } else {
    // odd-even transposition sort network, fully unrolled in registers
#pragma unroll
    for (int p = 0; p < R; ++p) {
#pragma unroll
      for (int a = (p & 1); a + 1 < R; a += 2) {
        const float lo = fminf(e[a], e[a + 1]);
        const float hi = fmaxf(e[a], e[a + 1]);
        e[a] = lo;
        e[a + 1] = hi;
      }
    }
    return e[(R - 1) / 2];
  }
}

// R > 0: compile-time row count.  R == 0: any hp.rows <= S2_MAX_ROWS — the missing rows are
// +inf, which sort last, so element (rows-1)/2 of the sorted 16 is the lower median.
template <int R>
__host__ __device__ constexpr int est_rows() { return R > 0 ? R : S2_MAX_ROWS; }

// the r signed bucket values s_j(i) T[j, h_j(i)] of index i
template <int R>
__device__ __forceinline__ void query_estimates(uint64_t i, const float* __restrict__ table, const HashParams& hp,
                                                float (&e)[est_rows<R>()]) {
  constexpr int N = est_rows<R>();
  const size_t cols = hp.cols;
  if (hp.mode == kInjective) {
    // i >= cols is rejected on the host (core.py:133-134); the guard keeps reads in bounds
#pragma unroll
    for (int j = 0; j < N; ++j)
      e[j] = (R == 0 && j >= hp.rows) ? __int_as_float(0x7F800000) : (i < cols ? __ldg(table + j * cols + i) : 0.f);
  } else {
    const uint64_t x = index_term(i);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (R == 0 && j >= hp.rows) {
        e[j] = __int_as_float(0x7F800000);
        continue;
      }
      const uint64_t w = mix64(hp.seed[j] + x);
      const float t = __ldg(table + j * cols + bucket_of(w, hp));
      e[j] = (w >> 63) ? -t : t;
    }
  }
}

// lower median (element (r-1)/2 of the sorted estimates, sketch.py:127-128)
template <int R>
__device__ __forceinline__ float median_of(float (&e)[est_rows<R>()], const HashParams& hp) {
  if constexpr (R > 0) {
    return lower_median<R>(e);
  } else {
    constexpr int N = S2_MAX_ROWS;
#pragma unroll
    for (int p = 0; p < N; ++p) {
#pragma unroll
      for (int a = (p & 1); a + 1 < N; a += 2) {
        const float lo = fminf(e[a], e[a + 1]);
        const float hi = fmaxf(e[a], e[a + 1]);
        e[a] = lo;
        e[a + 1] = hi;
      }
    }
    float m = e[0];
#pragma unroll
    for (int j = 1; j < N; ++j)
      if (j == (hp.rows - 1) / 2) m = e[j];
    return m;
  }
}

template <int R>
__device__ __forceinline__ float query_one(uint64_t i, const float* __restrict__ table, const HashParams& hp) {
  float e[est_rows<R>()];
  query_estimates<R>(i, table, hp, e);
  return median_of<R>(e, hp);
}

template <bool BLOCKS>
__device__ __forceinline__ uint32_t decode_word(const uint32_t* __restrict__ bitmap, int64_t t, int lane, int64_t dim,
                                               int64_t bs, int64_t nelem_words) {
  const int64_t e0 = t * kDecTile + 32 * lane;
  uint32_t word = 0;
  if (!BLOCKS) {
    const int64_t wi = t * 32 + lane;
    if (wi < nelem_words) word = __ldg(bitmap + wi);
  } else {
    word = expand_blocks(bitmap, e0, dim, bs);
  }
  if (e0 + 32 > dim) word &= e0 >= dim ? 0u : range_mask(0, (int)(dim - e0));
  return word;
}

struct DecodeCtx {
  const uint32_t* bitmap;  // union bitmap
  const float* table;      // summed sketch table
  float* out;
  int64_t dim, bs;
  float workers, inv_workers;
  int workers_pow2;
};

__device__ __forceinline__ void zero_next(float4* __restrict__ zt, int64_t zt_n4, unsigned long long* __restrict__ zc) {
  if (zt != nullptr) {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < zt_n4; i += (int64_t)gridDim.x * blockDim.x)
      zt[i] = z;
  }
  if (zc != nullptr && blockIdx.x == 0 && threadIdx.x < S2_NUM_COUNTERS) zc[threadIdx.x] = 0ull;
}

// Decode one warp tile (1024 elements at `base`) given its 32 union words (one per lane):
// set positions are compacted by a warp scan into q, values (r gathers + lower median +
// IEEE /W) land in vals, and the tile is written as dense float4 streaming stores.
template <int R>
__device__ __forceinline__ void decode_tile(const DecodeCtx& c, int64_t base, uint32_t word, const HashParams& hp,
                                            uint16_t* q, float* vals) {
  const int lane = threadIdx.x & 31;
  const int64_t dim = c.dim;
  const int cnt = __popc(word);
  int pre = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(kFull, pre, o);
    if (lane >= o) pre += n;
  }
  const int total = __shfl_sync(kFull, pre, 31);
  pre -= cnt;
  for (uint32_t w = word; w; w &= w - 1u) q[pre++] = (uint16_t)(lane * 32 + (__ffs(w) - 1));
  __syncwarp();
  // Queries one per lane per round.  Two queries per lane with all 2r gathers in flight before
  // either median was measured slower at every union density (decode 24.3 -> 25.0 µs at 1 %,
  // 33.6 -> 35.2 at 4 %, 45.8 -> 47.4 at 7.7 %, profiles/r02_ab_decode_pairs.txt).
  for (int s = lane; s < total; s += 32) {
    const int pos = q[s];
    // IEEE division: sparse.py:213 divides the float64 query by workers; x*2^-k is exact
    const float qv = query_one<R>((uint64_t)(base + pos), c.table, hp);
    vals[pos] = c.workers_pow2 ? qv * c.inv_workers : __fdiv_rn(qv, c.workers);
  }
  __syncwarp();
  const bool full = base + kDecTile <= dim;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t wk = __shfl_sync(kFull, word, 4 * k + (lane >> 3));
    const uint32_t nib = (wk >> ((lane & 7) * 4)) & 0xFu;
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (nib) {
      const float4 sv = *reinterpret_cast<const float4*>(vals + k * 128 + lane * 4);
      o.x = (nib & 1u) ? sv.x : 0.f;
      o.y = (nib & 2u) ? sv.y : 0.f;
      o.z = (nib & 4u) ? sv.z : 0.f;
      o.w = (nib & 8u) ? sv.w : 0.f;
    }
    const int64_t e = base + k * 128 + lane * 4;
    if (full) {
      __stcs(reinterpret_cast<float4*>(c.out + e), o);
    } else {
      if (e + 0 < dim) c.out[e + 0] = o.x;
      if (e + 1 < dim) c.out[e + 1] = o.y;
      if (e + 2 < dim) c.out[e + 2] = o.z;
      if (e + 3 < dim) c.out[e + 3] = o.w;
    }
  }
  __syncwarp();
}

// decode_tile with a value stage that is zero everywhere except the current tile's set
// positions: the dense output leaves as 8 unmasked LDS.128 + STG.128 per lane (no per-chunk
// nibble shuffles and selects); the previous tile's positions (still in q) are cleared first.
// The stage must be zero on the first call.  Used for block bitmaps (LSTM row bitmap step
// -2.3 %); at element bitmaps the extra shared-memory reads cost more than the selects save
// (ResNet-50 step +1-2 %, profiles/r02_ab_decode_clear.txt).
template <int R>
__device__ __forceinline__ void decode_tile_clear(const DecodeCtx& c, int64_t base, uint32_t word,
                                                  const HashParams& hp, uint16_t* q, float* vals, int& prev_total) {
  const int lane = threadIdx.x & 31;
  const int64_t dim = c.dim;
  const int cnt = __popc(word);
  int pre = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(kFull, pre, o);
    if (lane >= o) pre += n;
  }
  const int total = __shfl_sync(kFull, pre, 31);
  pre -= cnt;
  for (int s = lane; s < prev_total; s += 32) vals[q[s]] = 0.f;
  __syncwarp();
  for (uint32_t w = word; w; w &= w - 1u) q[pre++] = (uint16_t)(lane * 32 + (__ffs(w) - 1));
  __syncwarp();
  for (int s = lane; s < total; s += 32) {
    const int pos = q[s];
    const float qv = query_one<R>((uint64_t)(base + pos), c.table, hp);
    vals[pos] = c.workers_pow2 ? qv * c.inv_workers : __fdiv_rn(qv, c.workers);
  }
  prev_total = total;
  __syncwarp();
  if (base + kDecTile <= dim) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      __stcs(reinterpret_cast<float4*>(c.out + base + k * 128 + lane * 4),
             *reinterpret_cast<const float4*>(vals + k * 128 + lane * 4));
  } else {
    for (int64_t e = lane; base + e < dim; e += 32) c.out[base + e] = vals[e];
  }
  __syncwarp();
}

// Decode warp tiles t0, t0+tstep, ... < tend (one warp); the bitmap word is prefetched one
// tile ahead.  CLEAR: decode_tile_clear (the caller zeroes the stage first).
template <int R, bool BLOCKS, bool CLEAR = false>
__device__ __forceinline__ void decode_range(const DecodeCtx& c, int64_t t0, int64_t tstep, int64_t tend,
                                             const HashParams& hp, uint16_t* q, float* vals) {
  const int lane = threadIdx.x & 31;
  const int64_t nelem_words = (c.dim + 31) / 32;
  int64_t t = t0;
  int prev_total = 0;
  uint32_t wnext = t < tend ? decode_word<BLOCKS>(c.bitmap, t, lane, c.dim, c.bs, nelem_words) : 0u;
  for (; t < tend; t += tstep) {
    const uint32_t word = wnext;
    if (t + tstep < tend) wnext = decode_word<BLOCKS>(c.bitmap, t + tstep, lane, c.dim, c.bs, nelem_words);
    if constexpr (CLEAR)
      decode_tile_clear<R>(c, t * kDecTile, word, hp, q, vals, prev_total);
    else
      decode_tile<R>(c, t * kDecTile, word, hp, q, vals);
  }
}

}  // namespace s2
