// s2_decode.cuh — the K4 decode body (sparse_decompress, sparse.py:199-214 + CountSketchTable.query,
// sketch.py:114-128), shared by the standalone decode kernel (s2_kernels.cu) and the fused
// exchange+decode kernel (s2_p2p.cu).
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

template <int R>
__device__ __forceinline__ float query_one(uint64_t i, const float* __restrict__ table,
                                           const HashParams& hp) {
  const size_t cols = hp.cols;
  float e[R];
  if (hp.mode == kInjective) {
#pragma unroll
    for (int j = 0; j < R; ++j) e[j] = __ldg(table + j * cols + i);
  } else {
    const uint64_t x = index_term(i);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const uint64_t w = mix64(hp.seed[j] + x);
      const float t = __ldg(table + j * cols + bucket_of(w, hp));
      e[j] = (w >> 63) ? -t : t;
    }
  }
  return lower_median<R>(e);
}

template <bool BLOCKS>
__device__ __forceinline__ uint32_t decode_word(const uint32_t* __restrict__ bitmap, const PeerMaps& pm, int64_t t,
                                               int lane, int64_t dim, int64_t bs, int64_t nelem_words) {
  const int64_t e0 = t * kDecTile + 32 * lane;
  uint32_t word = 0;
  if (!BLOCKS) {
    const int64_t wi = t * 32 + lane;
    if (wi < nelem_words) {
      if (pm.n == 0) {
        word = __ldg(bitmap + wi);
      } else {
        // union of the W ranks' bitmaps read straight from peer memory (NVLink) — the
        // exchange kernel then only has to move the sketch table (BlockMask.union, sparse.py:55-58)
#pragma unroll
        for (int q = 0; q < kMaxWorld; ++q)
          if (q < pm.n) word |= __ldcg(pm.p[q] + wi);
      }
    }
  } else {
    word = expand_blocks(bitmap, e0, dim, bs);
  }
  if (e0 + 32 > dim) word &= e0 >= dim ? 0u : range_mask(0, (int)(dim - e0));
  return word;
}

struct DecodeCtx {
  const uint32_t* bitmap;  // union bitmap (ignored when PeerMaps n > 0)
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

__device__ __forceinline__ float finish_value(const DecodeCtx& c, float qv) {
  // IEEE division: sparse.py:213 divides the float64 query by workers; x*2^-k is exact
  return c.workers_pow2 ? qv * c.inv_workers : __fdiv_rn(qv, c.workers);
}

// Decode warp tiles t0, t0+tstep, ... < tend (one warp).  Per tile: the bitmap word is
// prefetched one tile ahead and set positions are compacted by a warp scan into q.  A
// full tile is assembled in shared memory (zero-fill + the decoded values: r gathers,
// lower median, /W) and written to HBM by ONE TMA bulk store (cp.async.bulk
// shared->global, `UBLKCP` in SASS) — no per-lane stores, no L1 store traffic; the
// buffer is reused once the previous bulk store has finished reading it, and the
// gathers of the tile's first 32 values overlap that wait.  The ragged last tile
// uses plain stores.
template <int R, bool BLOCKS>
__device__ __forceinline__ void decode_range(const DecodeCtx& c, const PeerMaps& pm, int64_t t0, int64_t tstep,
                                             int64_t tend, const HashParams& hp, uint16_t* q, float* vals) {
  const int lane = threadIdx.x & 31;
  const int64_t nelem_words = (c.dim + 31) / 32;
  const int64_t dim = c.dim;
  int64_t t = t0;
  uint32_t wnext = t < tend ? decode_word<BLOCKS>(c.bitmap, pm, t, lane, dim, c.bs, nelem_words) : 0u;
  for (; t < tend; t += tstep) {
    const int64_t base = t * kDecTile;
    const uint32_t word = wnext;
    if (t + tstep < tend) wnext = decode_word<BLOCKS>(c.bitmap, pm, t + tstep, lane, dim, c.bs, nelem_words);
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
    // first batch of values into registers (their gathers overlap the buffer wait below)
    int pos0 = -1;
    float v0 = 0.f;
    if (lane < total) {
      pos0 = q[lane];
      v0 = finish_value(c, query_one<R>((uint64_t)(base + pos0), c.table, hp));
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // vals free again
    __syncwarp();
    const bool full = base + kDecTile <= dim;
    float4* v4 = reinterpret_cast<float4*>(vals);
    if (full) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v4[k * 32 + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncwarp();
    }
    if (pos0 >= 0) vals[pos0] = v0;
    for (int s = 32 + lane; s < total; s += 32) {
      const int pos = q[s];
      vals[pos] = finish_value(c, query_one<R>((uint64_t)(base + pos), c.table, hp));
    }
    __syncwarp();
    if (full) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
      __syncwarp();
      if (lane == 0) {
        asm volatile(
            "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
            "cp.async.bulk.commit_group;" ::"l"(c.out + base),
            "r"((uint32_t)__cvta_generic_to_shared(vals)), "r"((uint32_t)(kDecTile * 4))
            : "memory");
      }
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t wk = __shfl_sync(kFull, word, 4 * k + (lane >> 3));
        const uint32_t nib = (wk >> ((lane & 7) * 4)) & 0xFu;
        const float4 sv = v4[k * 32 + lane];
        const int64_t e = base + k * 128 + lane * 4;
        if (e + 0 < dim) c.out[e + 0] = (nib & 1u) ? sv.x : 0.f;
        if (e + 1 < dim) c.out[e + 1] = (nib & 2u) ? sv.y : 0.f;
        if (e + 2 < dim) c.out[e + 2] = (nib & 4u) ? sv.z : 0.f;
        if (e + 3 < dim) c.out[e + 3] = (nib & 8u) ? sv.w : 0.f;
      }
      __syncwarp();
    }
  }
}

// the warp's bulk stores must have completed before its results are consumed / smem is freed
__device__ __forceinline__ void decode_drain() {
  if ((threadIdx.x & 31) == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncwarp();
}

}  // namespace s2
