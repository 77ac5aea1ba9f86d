// s2_p2p.cu — sketch SUM + bitmap OR across the GPUs of one box over NVLink peer memory.
//
// Replaces the in-process sparse_merge fold (sparse.py:174-196): sketch.merge (sum,
// sketch.py:213-216) and BlockMask.union (bitwise OR, sparse.py:55-58) of W payloads.
// NCCL has no OR reduction and its small-message all-reduce/all-gather pair costs
// tens of microseconds at these sizes, so the exchange is one kernel that reads the
// peers' buffers directly (CUDA IPC mappings, NVLink loads):
//
//   barrier 1   CTA b of every rank announces it started, i.e. that rank's compress
//               finished (stream order); CTA b waits for CTA b of all ranks.
//   phase A     reduce-scatter: rank r sums (table) / ORs (bitmap) slice r, chunk b,
//               over all W ranks in fixed rank order 0..W-1, into its own buffers.
//   barrier 2   same pairing: chunk b of every slice is final.
//   phase B     all-gather: rank r copies chunk b of every other rank's slice.
//
// Per rank this moves 2 (W-1)/W of (table + bitmap) bytes over NVLink (two-shot), and
// every rank ends with bit-identical tables (one summation order) — so the replicated
// decode is identical on all ranks.  CTA b only ever waits for CTA b of the other
// ranks, so no intra-GPU grid barrier is needed; the launch is cooperative so all G
// CTAs are co-resident.  Epochs live in the arena (one counter per CTA), which keeps
// the kernel replayable inside a CUDA graph.
#include "s2_kernels.h"

namespace s2 {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int W>
__device__ __forceinline__ void cross_rank_barrier(const P2PArgs& a, int64_t off_flags, uint32_t ep) {
  __syncthreads();
  if (threadIdx.x < W) {
    const int q = threadIdx.x;
    __threadfence_system();  // this CTA's phase writes before the flag (cumulative via bar.sync)
    uint32_t* remote = reinterpret_cast<uint32_t*>(a.base[q] + off_flags) + a.rank * gridDim.x + blockIdx.x;
    st_release_sys(remote, ep);
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(a.base[a.rank] + off_flags) + q * gridDim.x + blockIdx.x;
    while ((int32_t)(ld_acquire_sys(mine) - ep) < 0) {
    }
  }
  __syncthreads();
}

// chunk [lo, hi) of n vectors for CTA b of G
__device__ __forceinline__ void chunk_of(int64_t n, int64_t& lo, int64_t& hi) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  lo = (int64_t)blockIdx.x * per;
  hi = lo + per < n ? lo + per : n;
  if (lo > n) lo = n;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

#define S2_TRACE(slot)                                                          \
  do {                                                                          \
    if (a.trace != nullptr && threadIdx.x == 0)                                 \
      a.trace[(int64_t)blockIdx.x * 8 + (slot)] = globaltimer();                \
  } while (0)

template <int W>
__global__ void __launch_bounds__(512) k_p2p_aggregate(const __grid_constant__ P2PArgs a) {
  __shared__ uint32_t s_ep;
  S2_TRACE(0);
  const int me = a.rank;
  const int cur = a.cur;
  if (threadIdx.x == 0) {
    uint32_t* e = reinterpret_cast<uint32_t*>(a.base[me] + a.off_epoch) + blockIdx.x;
    s_ep = *e + 1u;
    *e = s_ep;
  }
  __syncthreads();
  const uint32_t ep = s_ep;
  cross_rank_barrier<W>(a, a.off_flags_a, ep);
  S2_TRACE(1);

  const int64_t t4 = a.cells / 4 / W;  // float4 per slice
  const int64_t w4 = a.words / 4 / W;  // uint4 per slice
  {
    // phase A: slice `me`
    int64_t lo, hi;
    chunk_of(t4, lo, hi);
    const float4* src[W];
#pragma unroll
    for (int q = 0; q < W; ++q) src[q] = reinterpret_cast<const float4*>(a.base[q] + a.off_table[cur]) + me * t4;
    float4* dst = reinterpret_cast<float4*>(a.base[me] + a.off_table[cur]) + me * t4;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      float4 v[W];
#pragma unroll
      for (int q = 0; q < W; ++q) v[q] = __ldcg(src[q] + i);
      float4 s = v[0];
#pragma unroll
      for (int q = 1; q < W; ++q) {
        s.x += v[q].x; s.y += v[q].y; s.z += v[q].z; s.w += v[q].w;
      }
      dst[i] = s;
    }
    chunk_of(w4, lo, hi);
    const uint4* bsrc[W];
#pragma unroll
    for (int q = 0; q < W; ++q) bsrc[q] = reinterpret_cast<const uint4*>(a.base[q] + a.off_bitmap[cur]) + me * w4;
    uint4* udst = reinterpret_cast<uint4*>(a.base[me] + a.off_union[cur]) + me * w4;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      uint4 v[W];
#pragma unroll
      for (int q = 0; q < W; ++q) v[q] = __ldcg(bsrc[q] + i);
      uint4 s = v[0];
#pragma unroll
      for (int q = 1; q < W; ++q) {
        s.x |= v[q].x; s.y |= v[q].y; s.z |= v[q].z; s.w |= v[q].w;
      }
      udst[i] = s;
    }
  }
  S2_TRACE(2);
  cross_rank_barrier<W>(a, a.off_flags_b, ep);
  S2_TRACE(3);
  {
    // phase B: every other rank's slice, chunk b
    int64_t lo, hi;
    chunk_of(t4, lo, hi);
    float4* tdst = reinterpret_cast<float4*>(a.base[me] + a.off_table[cur]);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      float4 v[W];
#pragma unroll
      for (int q = 0; q < W; ++q)
        if (q != me) v[q] = __ldcg(reinterpret_cast<const float4*>(a.base[q] + a.off_table[cur]) + q * t4 + i);
#pragma unroll
      for (int q = 0; q < W; ++q)
        if (q != me) tdst[q * t4 + i] = v[q];
    }
    chunk_of(w4, lo, hi);
    uint4* udst = reinterpret_cast<uint4*>(a.base[me] + a.off_union[cur]);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      uint4 v[W];
#pragma unroll
      for (int q = 0; q < W; ++q)
        if (q != me) v[q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + a.off_union[cur]) + q * w4 + i);
#pragma unroll
      for (int q = 0; q < W; ++q)
        if (q != me) udst[q * w4 + i] = v[q];
    }
  }
  __syncthreads();
  S2_TRACE(4);
}

cudaError_t launch_p2p_aggregate(const P2PArgs& a, int grid, cudaStream_t st) {
  void* args[] = {const_cast<P2PArgs*>(&a)};
  const void* fn = nullptr;
  switch (a.world) {
    case 2: fn = (const void*)k_p2p_aggregate<2>; break;
    case 3: fn = (const void*)k_p2p_aggregate<3>; break;
    case 4: fn = (const void*)k_p2p_aggregate<4>; break;
    case 5: fn = (const void*)k_p2p_aggregate<5>; break;
    case 6: fn = (const void*)k_p2p_aggregate<6>; break;
    case 7: fn = (const void*)k_p2p_aggregate<7>; break;
    case 8: fn = (const void*)k_p2p_aggregate<8>; break;
    default: return cudaErrorInvalidValue;
  }
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(512), args, 0, st);
}

}  // namespace s2
