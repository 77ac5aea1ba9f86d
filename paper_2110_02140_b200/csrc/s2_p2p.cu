// s2_p2p.cu — K3: sketch SUM + bitmap OR across the GPUs of one box over NVLink peer memory.
//
// Replaces the in-process sparse_merge fold (sparse.py:174-196): sketch.merge (sum,
// sketch.py:213-216) and BlockMask.union (bitwise OR, sparse.py:55-58) of W payloads.
// NCCL has no OR reduction and its small-message all-reduce/all-gather pair costs
// tens of microseconds at these sizes, so the exchange is one kernel that reads the
// peers' buffers directly (CUDA-IPC mappings or caller-provided symmetric memory):
//
// two-shot (k_p2p_aggregate, default W > 2)
//   barrier 1   CTA b of every rank announces it started, i.e. that rank's compress
//               finished (stream order); CTA b waits for CTA b of all ranks.
//   phase A     reduce-scatter: rank r sums (table) / ORs (bitmap) slice r, chunk b,
//               over all W ranks in fixed rank order 0..W-1, into its own buffers.
//   barrier 2   same pairing: chunk b of every slice is final.
//   phase B     all-gather: rank r copies chunk b of every other rank's slice.
//   Per rank 2 (W-1)/W of (table + bitmap) bytes cross NVLink.
// one-shot (k_p2p_oneshot, default W <= 2)
//   barrier 1, then every rank sums / ORs the WHOLE table and bitmap of all W ranks into
//   private buffers: (W-1) x (table + bitmap) bytes in per rank, one barrier.
//
// Every rank sums in rank order 0..W-1, so all ranks end with bit-identical tables and the
// replicated decode is identical on every rank.  CTA b only ever waits for CTA b of the
// other ranks, so no grid-wide barrier is needed and the launch is a plain (programmatic)
// launch: a CTA that waits is one whose peers' CTA b has not started yet, which needs only
// that the W grids together fit on the GPUs they run on (always true for one grid per GPU;
// the single-GPU harness sizes the grids so W x G CTAs are co-resident).  Epochs live in the
// arena (one counter per CTA), which keeps the kernel replayable inside a CUDA graph.
//
// A barrier that spins longer than a.timeout_ns (S2_P2P_TIMEOUT_S, default 300 s, NCCL-
// watchdog-like) sets the arena's sticky error word and stops waiting; later exchanges skip
// their waits.  The decode then writes NaN over the whole output and reports
// S2_STATUS_EXCHANGE (s2_decode.cu), so a lost rank never produces a silently wrong average.
#include <cstdlib>

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

// CTA b announces epoch `ep` to CTA b of every rank (flag slot [rank * G + b] of each rank's
// array): every write of this CTA — local, or remote stores into a peer's inbox — happens-
// before the release (bar.sync is cumulative), so a peer that acquires the flag sees them.
template <int W>
__device__ __forceinline__ void signal_ranks(const P2PArgs& a, int64_t off_flags, uint32_t ep) {
  __syncthreads();
  if (threadIdx.x < W)
    st_release_sys(reinterpret_cast<uint32_t*>(a.base[threadIdx.x] + off_flags) + a.rank * gridDim.x + blockIdx.x, ep);
}

// CTA b waits until CTA b of every rank has announced `ep` in this rank's flag array.
template <int W>
__device__ __forceinline__ void wait_ranks(const P2PArgs& a, int64_t off_flags, uint32_t ep) {
  if (threadIdx.x < W) {
    const int q = threadIdx.x;
    uint32_t* err = reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_error);
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(a.base[a.rank] + off_flags) + q * gridDim.x + blockIdx.x;
    if (*reinterpret_cast<volatile uint32_t*>(err) == 0u) {  // after a timeout the epochs no longer pair up
      uint64_t t0 = 0;
      for (int spin = 0; (int32_t)(ld_acquire_sys(mine) - ep) < 0; ++spin) {
        if ((spin & 1023) == 1023) {
          const uint64_t now = globaltimer();
          if (t0 == 0) {
            t0 = now;
          } else if (now - t0 > a.timeout_ns || *reinterpret_cast<volatile uint32_t*>(err) != 0u) {
            atomicOr(err, 1u);  // sticky: this and every later output of the plan is NaN
            break;
          }
        }
      }
    }
  }
  __syncthreads();
}

// CTA b of this rank <-> CTA b of every rank
template <int W>
__device__ __forceinline__ void cross_rank_barrier(const P2PArgs& a, int64_t off_flags, uint32_t ep) {
  signal_ranks<W>(a, off_flags, ep);
  wait_ranks<W>(a, off_flags, ep);
}

// chunk [lo, hi) of n vectors for CTA b of G
__device__ __forceinline__ void chunk_of(int64_t n, int64_t& lo, int64_t& hi) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  lo = (int64_t)blockIdx.x * per;
  hi = lo + per < n ? lo + per : n;
  if (lo > n) lo = n;
}

__device__ __forceinline__ uint32_t next_epoch(const P2PArgs& a, uint32_t* s_ep) {
  if (threadIdx.x == 0) {
    uint32_t* e = reinterpret_cast<uint32_t*>(a.base[a.rank] + a.off_epoch) + blockIdx.x;
    *s_ep = *e + 1u;
    *e = *s_ep;
  }
  __syncthreads();
  return *s_ep;
}

constexpr int kP2PThreads = 1024;
// vectors per thread whose W loads are all in flight together (register budget: 64/thread)
template <int W>
__host__ __device__ constexpr int p2p_batch() { return W <= 4 ? 2 : 1; }

__device__ __forceinline__ uint4 add4(uint4 s, uint4 v) {
  return make_uint4(__float_as_uint(__uint_as_float(s.x) + __uint_as_float(v.x)),
                    __float_as_uint(__uint_as_float(s.y) + __uint_as_float(v.y)),
                    __float_as_uint(__uint_as_float(s.z) + __uint_as_float(v.z)),
                    __float_as_uint(__uint_as_float(s.w) + __uint_as_float(v.w)));
}
__device__ __forceinline__ uint4 or4(uint4 s, uint4 v) { return make_uint4(s.x | v.x, s.y | v.y, s.z | v.z, s.w | v.w); }

// One 16-byte vector v of the combined index space [table float4 | bitmap uint4]:
// index i < t4 is table vector i, else bitmap vector i - t4 (per-slice indexing).
template <int W>
__device__ __forceinline__ void reduce_batch(const P2PArgs& a, int64_t i0, int64_t hi, int64_t t4, int64_t w4) {
  const int me = a.rank, cur = a.cur, tc = a.tcur;
  constexpr int B = p2p_batch<W>();
  uint4 v[B][W];
#pragma unroll
  for (int k = 0; k < B; ++k) {
    const int64_t i = i0 + (int64_t)k * kP2PThreads;
    if (i < hi) {
      const int64_t off = i < t4 ? a.off_table[tc] + (me * t4 + i) * 16 : a.off_bitmap[tc] + (me * w4 + i - t4) * 16;
#pragma unroll
      for (int q = 0; q < W; ++q) v[k][q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + off));
    }
  }
#pragma unroll
  for (int k = 0; k < B; ++k) {
    const int64_t i = i0 + (int64_t)k * kP2PThreads;
    if (i >= hi) continue;
    uint4 s = v[k][0];
    if (i < t4) {  // sketch.merge: fixed rank order 0..W-1 -> identical sums on every rank
#pragma unroll
      for (int q = 1; q < W; ++q) s = add4(s, v[k][q]);
      *reinterpret_cast<uint4*>(a.base[me] + a.off_table[tc] + (me * t4 + i) * 16) = s;
    } else {  // BlockMask.union
#pragma unroll
      for (int q = 1; q < W; ++q) s = or4(s, v[k][q]);
      *reinterpret_cast<uint4*>(a.base[me] + a.off_union[cur] + (me * w4 + i - t4) * 16) = s;
    }
  }
}

template <int W>
__device__ __forceinline__ void gather_batch(const P2PArgs& a, int64_t i0, int64_t hi, int64_t t4, int64_t w4) {
  const int me = a.rank, cur = a.cur, tc = a.tcur;
  constexpr int B = p2p_batch<W>();
  uint4 v[B][W];
#pragma unroll
  for (int k = 0; k < B; ++k) {
    const int64_t i = i0 + (int64_t)k * kP2PThreads;
    if (i < hi) {
#pragma unroll
      for (int q = 0; q < W; ++q) {
        if (q == me) continue;
        const int64_t off = i < t4 ? a.off_table[tc] + (q * t4 + i) * 16 : a.off_union[cur] + (q * w4 + i - t4) * 16;
        v[k][q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + off));
      }
    }
  }
#pragma unroll
  for (int k = 0; k < B; ++k) {
    const int64_t i = i0 + (int64_t)k * kP2PThreads;
    if (i >= hi) continue;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      if (q == me) continue;
      const int64_t off = i < t4 ? a.off_table[tc] + (q * t4 + i) * 16 : a.off_union[cur] + (q * w4 + i - t4) * 16;
      *reinterpret_cast<uint4*>(a.base[me] + off) = v[k][q];
    }
  }
}

template <int W>
__global__ void __launch_bounds__(kP2PThreads) k_p2p_aggregate(const __grid_constant__ P2PArgs a) {
  __shared__ uint32_t s_ep;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic launch: compress must be complete
  S2_TRACE(0);
  const uint32_t ep = next_epoch(a, &s_ep);
  const int64_t t4 = a.cells / 4 / W;  // 16-byte vectors per slice: table ...
  const int64_t w4 = a.words / 4 / W;  // ... and bitmap
  int64_t lo, hi;
  chunk_of(t4 + w4, lo, hi);
  cross_rank_barrier<W>(a, a.off_flags_a, ep);
  S2_TRACE(1);
  // peers are all in this reduce now: the decode may launch (its prologue zeroes the NEXT
  // ping-pong table, which no peer reads any more)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (int64_t)p2p_batch<W>() * kP2PThreads)
    reduce_batch<W>(a, i0, hi, t4, w4);  // phase A: reduce-scatter
  S2_TRACE(2);
  cross_rank_barrier<W>(a, a.off_flags_b, ep);
  S2_TRACE(3);
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (int64_t)p2p_batch<W>() * kP2PThreads)
    gather_batch<W>(a, i0, hi, t4, w4);  // phase B: all-gather
  __syncthreads();
  S2_TRACE(4);
}

template <int W>
__global__ void __launch_bounds__(kP2PThreads) k_p2p_oneshot(const __grid_constant__ P2PArgs a) {
  __shared__ uint32_t s_ep;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic launch: compress must be complete
  S2_TRACE(0);
  const uint32_t ep = next_epoch(a, &s_ep);
  const int me = a.rank, cur = a.cur, tc = a.tcur;
  const int64_t t4 = a.cells / 4, w4 = a.words / 4;
  int64_t lo, hi;
  chunk_of(t4 + w4, lo, hi);
  cross_rank_barrier<W>(a, a.off_flags_a, ep);
  S2_TRACE(1);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int B = p2p_batch<W>();
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (int64_t)B * kP2PThreads) {
    uint4 v[B][W];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int64_t i = i0 + (int64_t)k * kP2PThreads;
      if (i < hi) {
        const int64_t off = i < t4 ? a.off_table[tc] + i * 16 : a.off_bitmap[tc] + (i - t4) * 16;
#pragma unroll
        for (int q = 0; q < W; ++q) v[k][q] = __ldcg(reinterpret_cast<const uint4*>(a.base[q] + off));
      }
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int64_t i = i0 + (int64_t)k * kP2PThreads;
      if (i >= hi) continue;
      uint4 s = v[k][0];
      if (i < t4) {
#pragma unroll
        for (int q = 1; q < W; ++q) s = add4(s, v[k][q]);
        *reinterpret_cast<uint4*>(a.base[me] + a.off_tsum[cur] + i * 16) = s;
      } else {
#pragma unroll
        for (int q = 1; q < W; ++q) s = or4(s, v[k][q]);
        *reinterpret_cast<uint4*>(a.base[me] + a.off_union[cur] + (i - t4) * 16) = s;
      }
    }
  }
  __syncthreads();
  S2_TRACE(4);
}

// ============================================================ push exchange (S2_P2P_PUSH=1)
//
// The same sums and ORs, but every rank STORES its data into the peers' inboxes (remote NVLink
// writes) before announcing it, instead of announcing first and letting the peers pull: a rank
// that finishes its compress early moves its data while the late ranks are still compressing,
// and each flag wait is followed by local reads only.
//   one-shot: push my whole table+bitmap chunk into inbox slot [me] of every peer, signal, wait,
//             then sum / OR the W copies (own buffers + W-1 inbox slots, all local) in rank order.
//   two-shot: push slice q of my chunk into inbox slot [me] of rank q, signal, wait; reduce my
//             slice from the W copies in rank order (in place); push the reduced slice into every
//             peer's table / union, signal, wait.
template <int W>
__global__ void __launch_bounds__(kP2PThreads) k_p2p_push_oneshot(const __grid_constant__ P2PArgs a) {
  __shared__ uint32_t s_ep;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic launch: compress must be complete
  S2_TRACE(0);
  const uint32_t ep = next_epoch(a, &s_ep);
  const int me = a.rank, cur = a.cur, tc = a.tcur;
  const int64_t t4 = a.cells / 4, w4 = a.words / 4, slot = (t4 + w4) * 16;
  int64_t lo, hi;
  chunk_of(t4 + w4, lo, hi);
  const int64_t in_me = a.off_inbox[cur] + me * slot;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kP2PThreads) {
    const int64_t off = i < t4 ? a.off_table[tc] + i * 16 : a.off_bitmap[tc] + (i - t4) * 16;
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(a.base[me] + off));
#pragma unroll
    for (int q = 0; q < W; ++q)
      if (q != me) __stcg(reinterpret_cast<uint4*>(a.base[q] + in_me + i * 16), v);
  }
  S2_TRACE(1);
  signal_ranks<W>(a, a.off_flags_a, ep);
  wait_ranks<W>(a, a.off_flags_a, ep);
  S2_TRACE(2);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int B = p2p_batch<W>();
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (int64_t)B * kP2PThreads) {
    uint4 v[B][W];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int64_t i = i0 + (int64_t)k * kP2PThreads;
      if (i < hi) {
        const int64_t own = i < t4 ? a.off_table[tc] + i * 16 : a.off_bitmap[tc] + (i - t4) * 16;
#pragma unroll
        for (int q = 0; q < W; ++q)
          v[k][q] = __ldcg(reinterpret_cast<const uint4*>(
              a.base[me] + (q == me ? own : a.off_inbox[cur] + q * slot + i * 16)));
      }
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int64_t i = i0 + (int64_t)k * kP2PThreads;
      if (i >= hi) continue;
      uint4 s = v[k][0];
      if (i < t4) {
#pragma unroll
        for (int q = 1; q < W; ++q) s = add4(s, v[k][q]);
        *reinterpret_cast<uint4*>(a.base[me] + a.off_tsum[cur] + i * 16) = s;
      } else {
#pragma unroll
        for (int q = 1; q < W; ++q) s = or4(s, v[k][q]);
        *reinterpret_cast<uint4*>(a.base[me] + a.off_union[cur] + (i - t4) * 16) = s;
      }
    }
  }
  __syncthreads();
  S2_TRACE(4);
}

template <int W>
__global__ void __launch_bounds__(kP2PThreads) k_p2p_push_twoshot(const __grid_constant__ P2PArgs a) {
  __shared__ uint32_t s_ep;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic launch: compress must be complete
  S2_TRACE(0);
  const uint32_t ep = next_epoch(a, &s_ep);
  const int me = a.rank, cur = a.cur, tc = a.tcur;
  const int64_t t4 = a.cells / 4 / W, w4 = a.words / 4 / W, slot = (t4 + w4) * 16;  // per slice
  int64_t lo, hi;
  chunk_of(t4 + w4, lo, hi);
  // vector i of slice s in this rank's table / bitmap (local) and union
  auto src = [&](int sl, int64_t i) { return i < t4 ? a.off_table[tc] + (sl * t4 + i) * 16
                                                    : a.off_bitmap[tc] + (sl * w4 + i - t4) * 16; };
  auto dst = [&](int sl, int64_t i) { return i < t4 ? a.off_table[tc] + (sl * t4 + i) * 16
                                                    : a.off_union[cur] + (sl * w4 + i - t4) * 16; };
  // reduce-scatter, push: slice q of my chunk -> inbox slot [me] of rank q
  for (int64_t i = lo + threadIdx.x; i < hi; i += kP2PThreads) {
    uint4 v[W];
#pragma unroll
    for (int q = 0; q < W; ++q)
      if (q != me) v[q] = __ldcg(reinterpret_cast<const uint4*>(a.base[me] + src(q, i)));
#pragma unroll
    for (int q = 0; q < W; ++q)
      if (q != me) __stcg(reinterpret_cast<uint4*>(a.base[q] + a.off_inbox[cur] + me * slot + i * 16), v[q]);
  }
  S2_TRACE(1);
  signal_ranks<W>(a, a.off_flags_a, ep);
  wait_ranks<W>(a, a.off_flags_a, ep);
  S2_TRACE(2);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // reduce my slice in rank order (own copy + W-1 inbox slots, all local), then all-gather, push
  for (int64_t i = lo + threadIdx.x; i < hi; i += kP2PThreads) {
    uint4 v[W];
#pragma unroll
    for (int q = 0; q < W; ++q)
      v[q] = __ldcg(reinterpret_cast<const uint4*>(
          a.base[me] + (q == me ? src(me, i) : a.off_inbox[cur] + q * slot + i * 16)));
    uint4 s = v[0];
    if (i < t4) {
#pragma unroll
      for (int q = 1; q < W; ++q) s = add4(s, v[q]);
    } else {
#pragma unroll
      for (int q = 1; q < W; ++q) s = or4(s, v[q]);
    }
    const int64_t o = dst(me, i);
#pragma unroll
    for (int q = 0; q < W; ++q) {
      if (q == me) *reinterpret_cast<uint4*>(a.base[me] + o) = s;
      else __stcg(reinterpret_cast<uint4*>(a.base[q] + o), s);
    }
  }
  S2_TRACE(3);
  signal_ranks<W>(a, a.off_flags_b, ep);
  wait_ranks<W>(a, a.off_flags_b, ep);
  S2_TRACE(4);
}

static const void* p2p_kernel(const P2PArgs& a);

cudaError_t preload_p2p(const P2PArgs& a) {
  const void* fn = p2p_kernel(a);
  if (fn == nullptr) return cudaErrorInvalidValue;
  cudaFuncAttributes fa;
  return cudaFuncGetAttributes(&fa, fn);
}

cudaError_t launch_p2p_aggregate(const P2PArgs& a, int grid, cudaStream_t st) {
  const void* fn = p2p_kernel(a);
  if (fn == nullptr) return cudaErrorInvalidValue;
  // Plain programmatic launch: CTAs only wait on the same CTA index of the other ranks
  // (measured 1.7 µs per step faster at W = 2 and 4 than a cooperative launch).
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kP2PThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {const_cast<P2PArgs*>(&a)};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

static const void* p2p_kernel(const P2PArgs& a) {
  const void* fn = nullptr;
  if (a.push) {
    switch (a.world * 2 + a.oneshot) {
      case 5: fn = (const void*)k_p2p_push_oneshot<2>; break;
      case 7: fn = (const void*)k_p2p_push_oneshot<3>; break;
      case 9: fn = (const void*)k_p2p_push_oneshot<4>; break;
      case 4: fn = (const void*)k_p2p_push_twoshot<2>; break;
      case 6: fn = (const void*)k_p2p_push_twoshot<3>; break;
      case 8: fn = (const void*)k_p2p_push_twoshot<4>; break;
      case 10: fn = (const void*)k_p2p_push_twoshot<5>; break;
      case 12: fn = (const void*)k_p2p_push_twoshot<6>; break;
      case 14: fn = (const void*)k_p2p_push_twoshot<7>; break;
      case 16: fn = (const void*)k_p2p_push_twoshot<8>; break;
      default: return nullptr;
    }
  } else if (a.oneshot) {
    switch (a.world) {
      case 2: fn = (const void*)k_p2p_oneshot<2>; break;
      case 3: fn = (const void*)k_p2p_oneshot<3>; break;
      case 4: fn = (const void*)k_p2p_oneshot<4>; break;
      default: return nullptr;
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
      default: return nullptr;
    }
  }
  return fn;
}

}  // namespace s2
