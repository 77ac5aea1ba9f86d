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
#include <cstdlib>

#include "s2_kernels.h"
#include "s2_decode.cuh"

namespace s2 {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer();

// CTA b of this rank <-> CTA b of every rank.  A spin that outlives 10 s records an error
// in the arena and gives up instead of hanging the GPU (a peer died or diverged).
template <int W>
__device__ __forceinline__ void cross_rank_barrier(const P2PArgs& a, int64_t off_flags, uint32_t ep) {
  __syncthreads();  // the CTA's writes happen-before thread q's release (bar.sync is cumulative)
  if (threadIdx.x < W) {
    const int q = threadIdx.x;
    uint32_t* remote = reinterpret_cast<uint32_t*>(a.base[q] + off_flags) + a.rank * gridDim.x + blockIdx.x;
    st_release_sys(remote, ep);
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(a.base[a.rank] + off_flags) + q * gridDim.x + blockIdx.x;
    uint64_t t0 = 0;
    for (int spin = 0; (int32_t)(ld_acquire_sys(mine) - ep) < 0; ++spin) {
      if ((spin & 1023) == 1023) {
        const uint64_t now = globaltimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > 10000000000ull) {
          atomicOr(reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_error), 1u);
          break;
        }
      }
    }
  }
  __syncthreads();
}

// Barrier 1 when the compress kernels signal completion themselves (a.csig): every rank's
// last compress CTA stored its compress epoch into slot [rank] of this rank's flag array;
// wait until all W slots reached the epoch our own compress wrote.
template <int W>
__device__ __forceinline__ void compress_done_barrier(const P2PArgs& a) {
  if (threadIdx.x < W) {
    const int q = threadIdx.x;
    const uint32_t ep = *reinterpret_cast<volatile const uint32_t*>(a.base[a.rank] + a.off_cepoch);
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(a.base[a.rank] + a.off_flags_c) + q;
    uint64_t t0 = 0;
    for (int spin = 0; (int32_t)(ld_acquire_sys(mine) - ep) < 0; ++spin) {
      if ((spin & 1023) == 1023) {
        uint64_t now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (t0 == 0) t0 = now;
        else if (now - t0 > 10000000000ull) {
          atomicOr(reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_error), 1u);
          break;
        }
      }
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

struct XSync {
  unsigned long long* arrive;  // local arrival counter (cumulative)
  uint32_t* release;           // CTA 0 -> local CTAs: last cross-rank epoch passed (x2 per call)
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// all CTAs of this grid arrive; returns when `target` arrivals were counted
__device__ __forceinline__ void local_arrive_wait(unsigned long long* arrive, unsigned long long target,
                                                  bool wait_all) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(arrive, 1ull);
    if (wait_all)
      while (ld_acquire_gpu64(arrive) < target) {
      }
  }
  __syncthreads();
}

// CTA 0 <-> CTA 0 of every rank (flag slot [rank] of each rank's array), then release locally
template <int W>
__device__ __forceinline__ void rank_barrier(const P2PArgs& a, int64_t off_flags, uint32_t ep, uint32_t* release,
                                             uint32_t rel_val) {
  if (blockIdx.x == 0) {
    if (threadIdx.x < W) {
      const int q = threadIdx.x;
      st_release_sys(reinterpret_cast<uint32_t*>(a.base[q] + off_flags) + a.rank, ep);
      const uint32_t* mine = reinterpret_cast<const uint32_t*>(a.base[a.rank] + off_flags) + q;
      uint64_t t0 = 0;
      for (int spin = 0; (int32_t)(ld_acquire_sys(mine) - ep) < 0; ++spin) {
        if ((spin & 1023) == 1023) {
          const uint64_t now = globaltimer();
          if (t0 == 0) t0 = now;
          else if (now - t0 > 10000000000ull) {
            atomicOr(reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_error), 1u);
            break;
          }
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) st_release_gpu(release, rel_val);
  } else if (threadIdx.x == 0) {
    uint64_t t0 = 0;
    for (int spin = 0; (int32_t)(ld_acquire_gpu(release) - rel_val) < 0; ++spin) {
      if ((spin & 1023) == 1023) {
        const uint64_t now = globaltimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > 10000000000ull) break;
      }
    }
  }
  __syncthreads();
}

constexpr int kP2PThreads = 1024;
// vectors per thread whose W loads are all in flight together (register budget: 64/thread)
template <int W>
__host__ __device__ constexpr int p2p_batch() { return W <= 4 ? 2 : 1; }

// One 16-byte vector v of the combined index space [table float4 | bitmap uint4]:
// index i < t4 is table vector i, else bitmap vector i - t4 (per-slice indexing).
template <int W>
__device__ __forceinline__ void reduce_batch(const P2PArgs& a, int64_t i0, int64_t hi, int64_t t4, int64_t w4) {
  const int me = a.rank, cur = a.cur;
  constexpr int kP2PBatch = p2p_batch<W>();
  uint4 v[kP2PBatch][W];
#pragma unroll
  for (int k = 0; k < kP2PBatch; ++k) {
    const int64_t i = i0 + (int64_t)k * kP2PThreads;
    if (i < hi) {
      const bool tab = i < t4;
      const int64_t off = tab ? a.off_table[cur] + (me * t4 + i) * 16 : a.off_bitmap[cur] + (me * w4 + i - t4) * 16;
#pragma unroll
      for (int q = 0; q < W; ++q) v[k][q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + off));
    }
  }
#pragma unroll
  for (int k = 0; k < kP2PBatch; ++k) {
    const int64_t i = i0 + (int64_t)k * kP2PThreads;
    if (i < hi) {
      uint4 s;
      if (i < t4) {  // sketch.merge: fixed rank order 0..W-1 -> identical sums on every rank
        float fx = __uint_as_float(v[k][0].x), fy = __uint_as_float(v[k][0].y);
        float fz = __uint_as_float(v[k][0].z), fw = __uint_as_float(v[k][0].w);
#pragma unroll
        for (int q = 1; q < W; ++q) {
          fx += __uint_as_float(v[k][q].x);
          fy += __uint_as_float(v[k][q].y);
          fz += __uint_as_float(v[k][q].z);
          fw += __uint_as_float(v[k][q].w);
        }
        s = make_uint4(__float_as_uint(fx), __float_as_uint(fy), __float_as_uint(fz), __float_as_uint(fw));
        *reinterpret_cast<uint4*>(a.base[me] + a.off_table[cur] + (me * t4 + i) * 16) = s;
      } else {  // BlockMask.union
        s = v[k][0];
#pragma unroll
        for (int q = 1; q < W; ++q) {
          s.x |= v[k][q].x; s.y |= v[k][q].y; s.z |= v[k][q].z; s.w |= v[k][q].w;
        }
        *reinterpret_cast<uint4*>(a.base[me] + a.off_union[cur] + (me * w4 + i - t4) * 16) = s;
      }
    }
  }
}

template <int W>
__device__ __forceinline__ void gather_batch(const P2PArgs& a, int64_t i0, int64_t hi, int64_t t4, int64_t w4) {
  const int me = a.rank, cur = a.cur;
  constexpr int kP2PBatch = p2p_batch<W>();
  uint4 v[kP2PBatch][W];
#pragma unroll
  for (int k = 0; k < kP2PBatch; ++k) {
    const int64_t i = i0 + (int64_t)k * kP2PThreads;
    if (i < hi) {
      const bool tab = i < t4;
#pragma unroll
      for (int q = 0; q < W; ++q) {
        if (q == me) continue;
        const int64_t off = tab ? a.off_table[cur] + (q * t4 + i) * 16 : a.off_union[cur] + (q * w4 + i - t4) * 16;
        v[k][q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + off));
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kP2PBatch; ++k) {
    const int64_t i = i0 + (int64_t)k * kP2PThreads;
    if (i < hi) {
      const bool tab = i < t4;
#pragma unroll
      for (int q = 0; q < W; ++q) {
        if (q == me) continue;
        const int64_t off = tab ? a.off_table[cur] + (q * t4 + i) * 16 : a.off_union[cur] + (q * w4 + i - t4) * 16;
        *reinterpret_cast<uint4*>(a.base[me] + off) = v[k][q];
      }
    }
  }
}

template <int W>
__global__ void __launch_bounds__(kP2PThreads) k_p2p_aggregate(const __grid_constant__ P2PArgs a) {
  __shared__ uint32_t s_ep;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic launch: compress must be complete
  S2_TRACE(0);
  if (threadIdx.x == 0) {
    uint32_t* e = reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_epoch) + blockIdx.x;
    s_ep = *e + 1u;
    *e = s_ep;
  }
  __syncthreads();
  const uint32_t ep = s_ep;
  const int64_t t4 = a.cells / 4 / W;  // 16-byte vectors per slice: table ...
  const int64_t w4 = a.table_only ? 0 : a.words / 4 / W;  // ... and bitmap (unless the decode ORs them)
  int64_t lo, hi;
  chunk_of(t4 + w4, lo, hi);
  unsigned long long* arrive = reinterpret_cast<unsigned long long*>(a.base[a.rank] + a.off_lsync);
  uint32_t* release = reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_lsync + 8);
  if (a.csig) compress_done_barrier<W>(a);
  else if (a.hier) rank_barrier<W>(a, a.off_flags_a, ep, release, 2u * ep - 1u);
  else cross_rank_barrier<W>(a, a.off_flags_a, ep);
  S2_TRACE(1);
  // peers are all in this reduce now: the decode may launch (its prologue zeroes the NEXT
  // ping-pong table, which no peer reads any more)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (int64_t)p2p_batch<W>() * kP2PThreads)
    reduce_batch<W>(a, i0, hi, t4, w4);  // phase A: reduce-scatter
  S2_TRACE(2);
  if (a.hier) {  // all local CTAs' slices written -> CTA 0 <-> peers -> local release
    local_arrive_wait(arrive, (unsigned long long)ep * gridDim.x, blockIdx.x == 0);
    rank_barrier<W>(a, a.off_flags_b, ep, release, 2u * ep);
  } else {
    cross_rank_barrier<W>(a, a.off_flags_b, ep);
  }
  S2_TRACE(3);
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (int64_t)p2p_batch<W>() * kP2PThreads)
    gather_batch<W>(a, i0, hi, t4, w4);  // phase B: all-gather
  __syncthreads();
  S2_TRACE(4);
}

// One-shot variant (small W): after barrier 1 every rank reduces the WHOLE table and bitmap
// from all W ranks into private buffers (sum -> tsum[cur], OR -> union[cur]); one barrier,
// (W-1) x (table + bitmap) bytes over NVLink per rank.
template <int W>
__global__ void __launch_bounds__(kP2PThreads) k_p2p_oneshot(const __grid_constant__ P2PArgs a) {
  __shared__ uint32_t s_ep;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic launch: compress must be complete
  S2_TRACE(0);
  if (threadIdx.x == 0) {
    uint32_t* e = reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_epoch) + blockIdx.x;
    s_ep = *e + 1u;
    *e = s_ep;
  }
  __syncthreads();
  const int me = a.rank, cur = a.cur;
  const int64_t t4 = a.cells / 4, w4 = a.table_only ? 0 : a.words / 4;
  int64_t lo, hi;
  chunk_of(t4 + w4, lo, hi);
  if (a.csig) compress_done_barrier<W>(a);
  else if (a.hier) rank_barrier<W>(a, a.off_flags_a, s_ep, reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_lsync + 8),
                                   2u * s_ep - 1u);
  else cross_rank_barrier<W>(a, a.off_flags_a, s_ep);
  S2_TRACE(1);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int B = p2p_batch<W>();
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (int64_t)B * kP2PThreads) {
    uint4 v[B][W];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int64_t i = i0 + (int64_t)k * kP2PThreads;
      if (i < hi) {
        if (i < t4 || !a.push) {
          const int64_t off = i < t4 ? a.off_table[cur] + i * 16 : a.off_bitmap[cur] + (i - t4) * 16;
#pragma unroll
          for (int q = 0; q < W; ++q) v[k][q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + off));
        } else {  // bitmaps pushed by the peers' compress kernels: all local
#pragma unroll
          for (int q = 0; q < W; ++q) {
            const int64_t off = q == me ? a.off_bitmap[cur] + (i - t4) * 16
                                        : a.off_inbox[cur] + (int64_t)q * a.words * 4 + (i - t4) * 16;
            v[k][q] = __ldcg(reinterpret_cast<const uint4*>(a.base[me] + off));
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int64_t i = i0 + (int64_t)k * kP2PThreads;
      if (i >= hi) continue;
      if (i < t4) {
        float fx = __uint_as_float(v[k][0].x), fy = __uint_as_float(v[k][0].y);
        float fz = __uint_as_float(v[k][0].z), fw = __uint_as_float(v[k][0].w);
#pragma unroll
        for (int q = 1; q < W; ++q) {
          fx += __uint_as_float(v[k][q].x);
          fy += __uint_as_float(v[k][q].y);
          fz += __uint_as_float(v[k][q].z);
          fw += __uint_as_float(v[k][q].w);
        }
        *reinterpret_cast<uint4*>(a.base[me] + a.off_tsum[cur] + i * 16) =
            make_uint4(__float_as_uint(fx), __float_as_uint(fy), __float_as_uint(fz), __float_as_uint(fw));
      } else {
        uint4 o = v[k][0];
#pragma unroll
        for (int q = 1; q < W; ++q) {
          o.x |= v[k][q].x; o.y |= v[k][q].y; o.z |= v[k][q].z; o.w |= v[k][q].w;
        }
        *reinterpret_cast<uint4*>(a.base[me] + a.off_union[cur] + (i - t4) * 16) = o;
      }
    }
  }
  __syncthreads();
  S2_TRACE(4);
}

// ============================================================ pipelined two-shot
//
// Same data movement as k_p2p_aggregate, but every CTA waits for ONE peer at a time:
// phase A accumulates slice `me` peer by peer (rotation order me+1, me+2, ...) as soon as
// that peer's CTA b has arrived, phase B copies each peer's reduced slice as soon as that
// peer's CTA b has finished its phase A — so transfers from early peers overlap the wait
// for late ones instead of queueing behind two all-peer barriers.  The owner of a slice
// sums it once and broadcasts it, so every rank still ends with identical tables.
// Thread 0 spins until at least one peer in `pending` (bit q) has reached `ep` in flag
// array off_flags, then returns (to the whole CTA) the set of peers ready now.
template <int W>
__device__ __forceinline__ uint32_t wait_any(const P2PArgs& a, int64_t off_flags, uint32_t pending, uint32_t ep,
                                             uint32_t* s_mask) {
  if (threadIdx.x == 0) {
    uint32_t ready = 0;
    uint64_t t0 = 0;
    for (int spin = 0;; ++spin) {
#pragma unroll
      for (int q = 0; q < W; ++q) {
        if (!((pending >> q) & 1u)) continue;
        const uint32_t* f = reinterpret_cast<const uint32_t*>(a.base[a.rank] + off_flags) + q * gridDim.x + blockIdx.x;
        if ((int32_t)(ld_acquire_sys(f) - ep) >= 0) ready |= 1u << q;
      }
      if (ready) break;
      if ((spin & 1023) == 1023) {
        const uint64_t now = globaltimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > 10000000000ull) {
          atomicOr(reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_error), 1u);
          ready = pending;  // give up waiting; results are flagged as invalid
          break;
        }
      }
    }
    *s_mask = ready;
  }
  __syncthreads();
  const uint32_t r = *s_mask;
  __syncthreads();
  return r;
}

template <int W>
__device__ __forceinline__ void signal_flags(const P2PArgs& a, int64_t off_flags, uint32_t ep) {
  __syncthreads();  // this CTA's writes happen-before thread q's release (bar.sync is cumulative)
  if (threadIdx.x < W)
    st_release_sys(reinterpret_cast<uint32_t*>(a.base[threadIdx.x] + off_flags) + a.rank * gridDim.x + blockIdx.x, ep);
}

// Same data movement as k_p2p_aggregate, but a CTA never waits for all peers at once:
// phase A accumulates slice `me` from whichever peers have arrived (all ready peers'
// loads in flight together), phase B copies each peer's reduced slice chunk as soon as
// that peer's CTA b has finished its phase A.  The owner of a slice sums it once and
// broadcasts it, so every rank still ends with identical tables.
template <int W>
__global__ void __launch_bounds__(kP2PThreads) k_p2p_pipe(const __grid_constant__ P2PArgs a) {
  __shared__ uint32_t s_ep, s_mask;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic launch: compress must be complete
  S2_TRACE(0);
  if (threadIdx.x == 0) {
    uint32_t* e = reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_epoch) + blockIdx.x;
    s_ep = *e + 1u;
    *e = s_ep;
  }
  __syncthreads();
  const uint32_t ep = s_ep;
  const int me = a.rank, cur = a.cur;
  const int64_t t4 = a.cells / 4 / W;  // 16-byte vectors per slice: table ...
  const int64_t w4 = a.words / 4 / W;  // ... and bitmap
  int64_t lo, hi;
  chunk_of(t4 + w4, lo, hi);
  signal_flags<W>(a, a.off_flags_a, ep);  // my compress is complete
  const uint32_t others = ((1u << W) - 1u) & ~(1u << me);
  constexpr int B = W <= 2 ? 2 : 1;  // register budget (64/thread at 1024 threads)
  // each thread owns at most B vectors of the chunk per round (rounds only when the chunk is large)
  for (int64_t r0 = lo; r0 < hi; r0 += (int64_t)B * kP2PThreads) {
    uint4 acc[B];
    int64_t off[B];
    bool tab[B], ok[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int64_t i = r0 + threadIdx.x + (int64_t)k * kP2PThreads;
      ok[k] = i < hi;
      tab[k] = i < t4;
      off[k] = tab[k] ? a.off_table[cur] + (me * t4 + i) * 16 : a.off_bitmap[cur] + (me * w4 + i - t4) * 16;
      if (ok[k]) acc[k] = *reinterpret_cast<const uint4*>(a.base[me] + off[k]);
    }
    uint32_t pending = others;
    while (pending) {
      const uint32_t ready = wait_any<W>(a, a.off_flags_a, pending, ep, &s_mask);
      pending &= ~ready;
      uint4 v[W][B];
#pragma unroll
      for (int q = 0; q < W; ++q) {
        if (!((ready >> q) & 1u)) continue;
#pragma unroll
        for (int k = 0; k < B; ++k)
          if (ok[k]) v[q][k] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + off[k]));
      }
#pragma unroll
      for (int q = 0; q < W; ++q) {
        if (!((ready >> q) & 1u)) continue;
#pragma unroll
        for (int k = 0; k < B; ++k) {
          if (!ok[k]) continue;
          if (tab[k]) {
            acc[k].x = __float_as_uint(__uint_as_float(acc[k].x) + __uint_as_float(v[q][k].x));
            acc[k].y = __float_as_uint(__uint_as_float(acc[k].y) + __uint_as_float(v[q][k].y));
            acc[k].z = __float_as_uint(__uint_as_float(acc[k].z) + __uint_as_float(v[q][k].z));
            acc[k].w = __float_as_uint(__uint_as_float(acc[k].w) + __uint_as_float(v[q][k].w));
          } else {
            acc[k].x |= v[q][k].x; acc[k].y |= v[q][k].y; acc[k].z |= v[q][k].z; acc[k].w |= v[q][k].w;
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      if (!ok[k]) continue;
      const int64_t i = r0 + threadIdx.x + (int64_t)k * kP2PThreads;
      const int64_t dst = tab[k] ? off[k] : a.off_union[cur] + (me * w4 + i - t4) * 16;
      *reinterpret_cast<uint4*>(a.base[me] + dst) = acc[k];
    }
  }
  S2_TRACE(1);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // every peer has arrived
  signal_flags<W>(a, a.off_flags_b, ep);  // my reduced slice chunk is final
  S2_TRACE(2);
  uint32_t pending = others;
  while (pending) {
    const uint32_t ready = wait_any<W>(a, a.off_flags_b, pending, ep, &s_mask);
    pending &= ~ready;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kP2PThreads) {
      uint4 v[W];
#pragma unroll
      for (int q = 0; q < W; ++q) {
        if (!((ready >> q) & 1u)) continue;
        const int64_t o = i < t4 ? a.off_table[cur] + (q * t4 + i) * 16 : a.off_union[cur] + (q * w4 + i - t4) * 16;
        v[q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + o));
      }
#pragma unroll
      for (int q = 0; q < W; ++q) {
        if (!((ready >> q) & 1u)) continue;
        const int64_t o = i < t4 ? a.off_table[cur] + (q * t4 + i) * 16 : a.off_union[cur] + (q * w4 + i - t4) * 16;
        *reinterpret_cast<uint4*>(a.base[me] + o) = v[q];
      }
    }
  }
  __syncthreads();
  S2_TRACE(4);
}

// ============================================================ NVLS (in-switch) exchange
//
// With torch symmetric memory the arena also has a multicast address: a load-reduce on it
// returns the SUM (float) or OR (bits) of all W ranks' copies, computed inside the
// NVSwitch, and a multicast store writes all W copies.  Rank r reduces slice r of the
// table and the bitmap and broadcasts the result into every rank's table[cur] (in place)
// and union[cur]: per rank (table + bitmap)/W bytes in and out over NVLink, instead of
// 2(W-1)/W (two-shot) — and no peer ever reads another's partially written slice.
__device__ __forceinline__ float4 mc_ld_add_v4f32(const void* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void mc_st_v4f32(void* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ uint64_t mc_ld_or_b64(const void* p) {
  uint64_t v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.or.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mc_st_b64(void* p, uint64_t v) {
  asm volatile("multimem.st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int W>
__global__ void __launch_bounds__(kP2PThreads) k_nvls_exchange(const __grid_constant__ P2PArgs a) {
  __shared__ uint32_t s_ep;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic launch: compress must be complete
  S2_TRACE(0);
  if (threadIdx.x == 0) {
    uint32_t* e = reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_epoch) + blockIdx.x;
    s_ep = *e + 1u;
    *e = s_ep;
  }
  __syncthreads();
  const uint32_t ep = s_ep;
  const int me = a.rank, cur = a.cur;
  const int64_t t4 = a.cells / 4 / W;  // float4 per slice
  const int64_t w8 = a.words / 2 / W;  // uint64 per slice
  cross_rank_barrier<W>(a, a.off_flags_a, ep);  // every rank's compress is complete
  S2_TRACE(1);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  {
    int64_t lo, hi;
    chunk_of(t4 + w8, lo, hi);
    char* tab = a.mc + a.off_table[cur] + me * t4 * 16;
    const char* bm = a.mc + a.off_bitmap[cur] + me * w8 * 8;
    char* un = a.mc + a.off_union[cur] + me * w8 * 8;
    constexpr int B = 4;  // independent load-reduces in flight per thread
    for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (int64_t)B * kP2PThreads) {
      float4 tv[B];
      uint64_t bv[B];
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const int64_t i = i0 + (int64_t)k * kP2PThreads;
        if (i < hi) {
          if (i < t4) tv[k] = mc_ld_add_v4f32(tab + i * 16);
          else bv[k] = mc_ld_or_b64(bm + (i - t4) * 8);
        }
      }
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const int64_t i = i0 + (int64_t)k * kP2PThreads;
        if (i < hi) {
          if (i < t4) mc_st_v4f32(tab + i * 16, tv[k]);
          else mc_st_b64(un + (i - t4) * 8, bv[k]);
        }
      }
    }
  }
  asm volatile("fence.proxy.alias;" ::: "memory");  // multicast-alias stores before the unicast flag
  S2_TRACE(2);
  __syncthreads();
  if (threadIdx.x < W) __threadfence_system();
  cross_rank_barrier<W>(a, a.off_flags_b, ep);  // every slice of every rank is broadcast
  S2_TRACE(3);
}

// ============================================================ fused exchange + decode
//
// k_xdecode replaces k_p2p_* + k_decode for W > 1: one cooperative launch per reduce
// after the compress.  Cross-rank synchronisation is hierarchical — CTA 0 exchanges one
// flag per rank pair over NVLink and releases the local CTAs through a gpu-scope word —
// and the local grid barrier before the decode is a 64-bit arrival counter.  CTA b
// computes the union bitmap words of ITS OWN decode tile range (OR of the W ranks'
// bitmaps, peer loads batched with the table loads), so only the table needs the grid
// barrier.  Table: one-shot (W <= 2 by default) or two-shot (reduce-scatter, barrier,
// all-gather).
template <int R, int W, bool ONESHOT>
__global__ void __launch_bounds__(256, 4)
k_xdecode(const __grid_constant__ P2PArgs a, const __grid_constant__ DecodeCtx dc, const __grid_constant__ HashParams hp,
          float4* __restrict__ zt, int64_t zt_n4, unsigned long long* __restrict__ zc) {
  extern __shared__ __align__(16) unsigned char x_smem[];  // vals [8][1024] f32 | queue [8][1024] u16
  float (*s_v)[kDecTile] = reinterpret_cast<float (*)[kDecTile]>(x_smem);
  uint16_t (*s_q)[kDecTile] = reinterpret_cast<uint16_t (*)[kDecTile]>(x_smem + 8 * kDecTile * 4);
  __shared__ uint32_t s_ep;
  __shared__ int s_next;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  S2_TRACE(0);
  const int me = a.rank, cur = a.cur, G = gridDim.x;
  if (threadIdx.x == 0) {
    uint32_t* e = reinterpret_cast<uint32_t*>(a.base[me] + a.off_epoch) + blockIdx.x;
    s_ep = *e + 1u;
    *e = s_ep;
    s_next = 0;
  }
  __syncthreads();
  const uint32_t ep = s_ep;
  unsigned long long* arrive = reinterpret_cast<unsigned long long*>(a.base[me] + a.off_lsync);
  uint32_t* release = reinterpret_cast<uint32_t*>(a.base[me] + a.off_lsync + 8);
  constexpr int K = ONESHOT ? 1 : 2;  // local arrivals per call

  // barrier 1: every rank's compress is complete
  rank_barrier<W>(a, a.off_flags_a, ep, release, 2u * ep - 1u);
  S2_TRACE(1);
  // the NEXT ping-pong table held the previous reduce, which peers read before reaching
  // barrier 1 of this one — only now may it be zeroed for the next compress
  zero_next(zt, zt_n4, zc);

  // this CTA's decode tiles and their union words
  const int64_t ntiles = (dc.dim + kDecTile - 1) / kDecTile;
  const int64_t per = (ntiles + G - 1) / G;
  const int64_t tb = (int64_t)blockIdx.x * per < ntiles ? (int64_t)blockIdx.x * per : ntiles;
  const int64_t te = tb + per < ntiles ? tb + per : ntiles;
  uint32_t* un = reinterpret_cast<uint32_t*>(a.base[me] + a.off_union[cur]);
  {
    // union words of [tb, te) tiles: 32 words per tile -> 8 uint4 per tile, W loads each (batched)
    const int64_t v0 = tb * 8;
    const int64_t v1 = te * 8 < (a.words / 4) ? te * 8 : (a.words / 4);
    constexpr int B = p2p_batch<W>();
    for (int64_t i0 = v0 + threadIdx.x; i0 < v1; i0 += B * blockDim.x) {
      uint4 v[B][W];
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const int64_t i = i0 + k * blockDim.x;
        if (i < v1)
#pragma unroll
          for (int q = 0; q < W; ++q) v[k][q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + a.off_bitmap[cur]) + i);
      }
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const int64_t i = i0 + k * blockDim.x;
        if (i < v1) {
          uint4 o = v[k][0];
#pragma unroll
          for (int q = 1; q < W; ++q) {
            o.x |= v[k][q].x; o.y |= v[k][q].y; o.z |= v[k][q].z; o.w |= v[k][q].w;
          }
          reinterpret_cast<uint4*>(un)[i] = o;
        }
      }
    }
  }
  // table
  if (ONESHOT) {
    const int64_t t4 = a.cells / 4;
    int64_t lo, hi;
    chunk_of(t4, lo, hi);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      uint4 v[W];
#pragma unroll
      for (int q = 0; q < W; ++q) v[q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + a.off_table[cur]) + i);
      float fx = __uint_as_float(v[0].x), fy = __uint_as_float(v[0].y);
      float fz = __uint_as_float(v[0].z), fw = __uint_as_float(v[0].w);
#pragma unroll
      for (int q = 1; q < W; ++q) {
        fx += __uint_as_float(v[q].x); fy += __uint_as_float(v[q].y);
        fz += __uint_as_float(v[q].z); fw += __uint_as_float(v[q].w);
      }
      reinterpret_cast<float4*>(a.base[me] + a.off_tsum[cur])[i] = make_float4(fx, fy, fz, fw);
    }
  } else {
    const int64_t t4 = a.cells / 4 / W;  // per slice
    int64_t lo, hi;
    chunk_of(t4, lo, hi);
    float4* dst = reinterpret_cast<float4*>(a.base[me] + a.off_table[cur]) + me * t4;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      uint4 v[W];
#pragma unroll
      for (int q = 0; q < W; ++q)
        v[q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + a.off_table[cur]) + me * t4 + i);
      float fx = __uint_as_float(v[0].x), fy = __uint_as_float(v[0].y);
      float fz = __uint_as_float(v[0].z), fw = __uint_as_float(v[0].w);
#pragma unroll
      for (int q = 1; q < W; ++q) {
        fx += __uint_as_float(v[q].x); fy += __uint_as_float(v[q].y);
        fz += __uint_as_float(v[q].z); fw += __uint_as_float(v[q].w);
      }
      dst[i] = make_float4(fx, fy, fz, fw);
    }
    // barrier 2: every rank's reduced slice is final
    local_arrive_wait(arrive, ((unsigned long long)(ep - 1) * K + 1) * G, blockIdx.x == 0);
    rank_barrier<W>(a, a.off_flags_b, ep, release, 2u * ep);
    float4* tab = reinterpret_cast<float4*>(a.base[me] + a.off_table[cur]);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
      uint4 v[W];
#pragma unroll
      for (int q = 0; q < W; ++q)
        if (q != me) v[q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + a.off_table[cur]) + q * t4 + i);
#pragma unroll
      for (int q = 0; q < W; ++q)
        if (q != me) tab[q * t4 + i] = *reinterpret_cast<float4*>(&v[q]);
    }
  }
  S2_TRACE(2);
  // local grid barrier: the whole summed table is in place
  local_arrive_wait(arrive, ((unsigned long long)(ep - 1) * K + K) * G, true);
  S2_TRACE(3);
  // decode this CTA's tile range; warps take tiles dynamically (shared counter)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  PeerMaps none{};
  DecodeCtx c = dc;
  c.bitmap = un;
  c.table = ONESHOT ? reinterpret_cast<const float*>(a.base[me] + a.off_tsum[cur])
                    : reinterpret_cast<const float*>(a.base[me] + a.off_table[cur]);
  for (;;) {
    int k = 0;
    if (lane == 0) k = atomicAdd(&s_next, 1);
    k = __shfl_sync(kFull, k, 0);
    const int64_t t = tb + k;
    if (t >= te) break;
    decode_range<R, false>(c, none, t, 1, t + 1, hp, s_q[wib], s_v[wib]);
  }
  S2_TRACE(4);
}

static const void* xdecode_fn(int rows, int world, int oneshot) {
  const void* fn = nullptr;
#define S2_X(R, W)                                                                    \
  if (rows == R && world == W)                                                        \
    fn = oneshot ? (const void*)k_xdecode<R, W, true> : (const void*)k_xdecode<R, W, false>;
  S2_X(3, 2) S2_X(3, 3) S2_X(3, 4) S2_X(3, 5) S2_X(3, 6) S2_X(3, 7) S2_X(3, 8)
  S2_X(5, 2) S2_X(5, 3) S2_X(5, 4) S2_X(5, 5) S2_X(5, 6) S2_X(5, 7) S2_X(5, 8)
  S2_X(1, 2) S2_X(1, 4) S2_X(1, 8)
#undef S2_X
  return fn;
}

constexpr int kXSmem = 8 * kDecTile * (4 + 2);

cudaError_t xdecode_grid(const HashParams& hp, int world, int oneshot, int* grid) {
  const void* fn = xdecode_fn(hp.rows, world, oneshot);
  *grid = 0;
  if (fn == nullptr) return cudaErrorNotSupported;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kXSmem);
  if (e != cudaSuccess) return e;
  int per_sm = 0, dev = 0, sms = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, kXSmem);
  if (e != cudaSuccess) return e;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (per_sm > 4) per_sm = 4;
  *grid = per_sm * sms;
  return cudaSuccess;
}

cudaError_t launch_xdecode(const P2PArgs& a, const DecodeCtx& dc, const HashParams& hp, int grid, float* zt,
                           int64_t zt_n4, unsigned long long* zc, cudaStream_t st) {
  const void* fn = xdecode_fn(hp.rows, a.world, a.oneshot);
  if (fn == nullptr) return cudaErrorNotSupported;
  constexpr int kSmem = kXSmem;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  float4* z4 = reinterpret_cast<float4*>(zt);
  void* args[] = {const_cast<P2PArgs*>(&a), const_cast<DecodeCtx*>(&dc), const_cast<HashParams*>(&hp), &z4,
                  &zt_n4, &zc};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// Exchange kernels only wait on the SAME CTA index of the other ranks, so one CTA per SM
// needs no cooperative launch (measured 1.7 µs per step faster at W = 2 and 4 without it);
// hierarchical barriers (a.hier) make CTAs wait on CTA 0 of their own grid and do need it.
// S2_P2P_COOP=1 forces the cooperative launch.
static cudaError_t launch_coop(const void* fn, const P2PArgs& a, int grid, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kP2PThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;  // all G CTAs co-resident
  attr[1].val.cooperative = 1;
  static int force = -1;
  if (force < 0) {
    const char* e = getenv("S2_P2P_COOP");
    force = e ? atoi(e) : 0;
  }
  cfg.attrs = attr;
  cfg.numAttrs = (a.hier || force) ? 2 : 1;
  void* args[] = {const_cast<P2PArgs*>(&a)};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_p2p_aggregate(const P2PArgs& a, int grid, cudaStream_t st) {
  const void* fn = nullptr;
  if (a.nvls) {
    switch (a.world) {
      case 2: fn = (const void*)k_nvls_exchange<2>; break;
      case 3: fn = (const void*)k_nvls_exchange<3>; break;
      case 4: fn = (const void*)k_nvls_exchange<4>; break;
      case 5: fn = (const void*)k_nvls_exchange<5>; break;
      case 6: fn = (const void*)k_nvls_exchange<6>; break;
      case 7: fn = (const void*)k_nvls_exchange<7>; break;
      case 8: fn = (const void*)k_nvls_exchange<8>; break;
      default: return cudaErrorInvalidValue;
    }
  } else if (a.pipe && !a.oneshot) {
    switch (a.world) {
      case 2: fn = (const void*)k_p2p_pipe<2>; break;
      case 3: fn = (const void*)k_p2p_pipe<3>; break;
      case 4: fn = (const void*)k_p2p_pipe<4>; break;
      case 5: fn = (const void*)k_p2p_pipe<5>; break;
      case 6: fn = (const void*)k_p2p_pipe<6>; break;
      case 7: fn = (const void*)k_p2p_pipe<7>; break;
      case 8: fn = (const void*)k_p2p_pipe<8>; break;
      default: return cudaErrorInvalidValue;
    }
  } else if (a.oneshot) {
    switch (a.world) {
      case 2: fn = (const void*)k_p2p_oneshot<2>; break;
      case 3: fn = (const void*)k_p2p_oneshot<3>; break;
      case 4: fn = (const void*)k_p2p_oneshot<4>; break;
      default: return cudaErrorInvalidValue;
    }
  } else {
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
  }
  return launch_coop(fn, a, grid, st);
}

}  // namespace s2
