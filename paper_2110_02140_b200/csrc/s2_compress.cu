// s2_kernels.cu — sm_100a kernels of the S2 sparse-sketch reduce.
//
//   K1+K2  k_compress_elem / k_compress_blocks
//          read g once (128-bit streaming loads), __ballot_sync bitmap words,
//          warp-level prefix compaction of the non-zeros into a per-warp shared
//          queue, and count-sketch insertion (r hashes, red.global.add.f32 into
//          the L2-resident table) once 32 entries are queued, so every lane of
//          the hashing warp is busy.  Replaces sparse_compress (sparse.py:151-171)
//          + CountSketchTable.insert (sketch.py:102-112).
//   K3b    k_bitmap_or — BlockMask.union over W gathered bitmaps (sparse.py:55-58)
//   K4     k_decode — walk the union bitmap, compact set positions per warp tile,
//          r gathers + lower-median network, ÷W (IEEE), dense float4 streaming
//          stores incl. zeros.  Replaces sparse_decompress (sparse.py:199-214)
//          + CountSketchTable.query (sketch.py:114-128).
//   aux    k_compact_* (ordered (idx,val) compaction = selected_indices,
//          sparse.py:44-49 / :164-168), k_selected_count (sparse.py:51-53),
//          k_table_sum (sketch.py:213-216).
//
// Data layout: g float32[dim]; bitmap uint32[ceil(num_blocks/32)] LE bit order;
// table float32[rows][cols] row-major.  A warp tile is 1024 elements = 32
// bitmap words = 8 float4 per lane.
#include "s2_device.cuh"

namespace s2 {

// ------------------------------------------------------- compress (K1+K2)
//
// MODE 0: element bitmap (block size 1), mask = g != 0, bitmap written directly.
// MODE 1: block bitmap built from g != 0 (block size > 1), atomicOr into a zeroed bitmap.
// MODE 2: given block bitmap (any block size): insert non-zeros of set blocks only.
//
// Per warp tile (1024 elements): lane l holds float4 chunks k = 0..7 at elements
// base + 128k + 4l (coalesced 512 B per load instruction).  Its 32 non-zero flags
// form one register m (bit 4k+c <-> element base+128k+4l+c).  The bitmap word of
// lane L (elements base+32L..+31) is the transpose of m across the 8-lane group
// (8 shuffles).  Non-zeros are appended to a per-warp shared queue at positions
// from one warp scan of popc(m); every full batch of 32 is hashed and inserted by
// the 32 lanes together.  NaN/Inf are non-zeros, so finiteness is tested on the
// queue only (MODE 2 tests every element: unselected non-zeros never reach the queue).
constexpr int kQFast = 128;  // tile non-zeros appended in one go when they fit

template <int R>
__device__ __forceinline__ void flush_full(uint32_t* qi, float* qv, int& qn, int lane, float* __restrict__ table,
                                           const HashParams& hp, uint32_t& bad) {
  __syncwarp();
  while (qn >= 32) {
    qn -= 32;
    const float v = qv[qn + lane];
    bad |= nonfinite(v);
    insert_one<R>(qi[qn + lane], v, table, hp);
  }
  __syncwarp();
}

__device__ __forceinline__ void load_tile(float4 (&v)[8], const float* __restrict__ g, int64_t t, int64_t dim,
                                          int lane) {
  const int64_t base = t * kTile;
  if (base + kTile <= dim) {
    const float4* g4 = reinterpret_cast<const float4*>(g) + (base >> 2) + lane;
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcs(g4 + k * 32);
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t e = base + k * 128 + lane * 4;
      v[k].x = e + 0 < dim ? g[e + 0] : 0.f;
      v[k].y = e + 1 < dim ? g[e + 1] : 0.f;
      v[k].z = e + 2 < dim ? g[e + 2] : 0.f;
      v[k].w = e + 3 < dim ? g[e + 3] : 0.f;
    }
  }
}

// ---- "this rank's compress is complete" signal (W > 1, peer-memory exchange) -------------
// The last CTA to finish (threadFenceReduction pattern) bumps the compress epoch and stores
// it with release semantics at system scope into slot [rank] of every rank's flag array, so
// the exchange kernel's first barrier is a local poll instead of a round of NVLink flag
// traffic issued only once its own CTAs have launched.
__device__ __forceinline__ void signal_done(const DoneSignal& sig) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(sig.done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence();
      const unsigned ep = *sig.epoch + 1u;
      *sig.epoch = ep;
      *sig.done = 0u;
      __threadfence_system();
      for (int q = 0; q < sig.world; ++q)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sig.peer_flags[q] + sig.rank), "r"(ep) : "memory");
    }
  }
}

// ---- TMA (cp.async.bulk) + mbarrier helpers -------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// order this thread's prior generic-proxy shared accesses before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// one elected lane: arm the barrier with the byte count and start a 1D bulk copy global -> smem
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint64_t pol) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "S2_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra S2_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// LOAD 0: the next tile's 8 float4 per lane are loaded into registers before the current
//         tile is processed (needs ~127 registers -> 2 CTAs/SM).
// LOAD 1: the next tile (4 KB) is prefetched into a per-warp shared buffer by one TMA bulk
//         copy (cp.async.bulk + mbarrier) right after the current tile has been moved to
//         registers, so prefetch costs no registers and 4 CTAs (32 warps) fit per SM.
// PUSH (MODE 0): every bitmap word is also stored into the peers' inbox slots (BitmapPush),
//         so the exchange kernel only has to move the sketch table.
template <int R, int MODE, int LOAD, bool SIG = false, bool PUSH = false>
__global__ void __launch_bounds__(kThreads, LOAD == 0 ? 2 : 4)
k_compress(const float* __restrict__ g, int64_t dim, int64_t bs, uint32_t* __restrict__ bitmap,
           float* __restrict__ table, unsigned long long* __restrict__ counters,
           const __grid_constant__ HashParams hp, const __grid_constant__ DoneSignal sig,
           const __grid_constant__ BitmapPush push) {
  constexpr int kCap = 32 + kQFast;
  __shared__ uint32_t s_qi[kWarps][kCap];
  __shared__ float s_qv[kWarps][kCap];
  __shared__ __align__(128) float4 s_tile[kWarps][kTile / 4];  // LOAD 1: TMA target; LOAD 0: value stage
  __shared__ __align__(8) uint64_t s_bar[kWarps];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  uint32_t* qi = s_qi[wib];
  float* qv = s_qv[wib];
  const int64_t ntiles = (dim + kTile - 1) / kTile;
  const int64_t nfull = dim / kTile;  // tiles that TMA can move whole
  const int64_t nelem_words = (dim + 31) / 32;
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  const int src_grp = 8 * (lane & 3);  // transpose: word L gathers lanes 8(L&3)..+7
  const int src_sh = 4 * (lane >> 2);  //            at nibble k = L>>2

  int qn = 0;                  // warp-uniform queue depth
  unsigned long long nnz = 0;  // warp-uniform
  unsigned long long sel = 0;  // per-lane selected coordinates (MODE 2)
  uint32_t bad = 0;
  float fin = 0.f;  // MODE 2: sum of 0*x, NaN iff a non-finite element was seen

  griddep_wait();  // g may be written by the caller's previous kernel
  griddep_launch_dependents();
  int64_t t = (int64_t)blockIdx.x * kWarps + wib;
  float4 vn[LOAD == 0 ? 8 : 1];
  uint32_t parity = 0;
  uint64_t pol = 0;
  if (LOAD == 0) {
    if (t < ntiles) load_tile(*reinterpret_cast<float4(*)[8]>(vn), g, t, dim, lane);
  } else if (LOAD == 1) {
    if (lane == 0) {
      mbar_init(&s_bar[wib], 1);
      fence_barrier_init();
    }
    __syncwarp();
    pol = policy_evict_first();
    if (lane == 0 && t < nfull) tma_load_1d(s_tile[wib], g + t * kTile, kTile * 4, &s_bar[wib], pol);
  }
#pragma unroll 1
  for (; t < ntiles; t += nw) {
    const int64_t base = t * kTile;
    float4 v[8];
    if (LOAD == 0) {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = vn[k < (LOAD == 0 ? 8 : 1) ? k : 0];
      if (t + nw < ntiles) load_tile(*reinterpret_cast<float4(*)[8]>(vn), g, t + nw, dim, lane);
    } else if (LOAD == 3) {
      load_tile(v, g, t, dim, lane);  // no prefetch: 64 registers, 4 CTAs (32 warps) per SM
    } else {
      if (t < nfull) {
        mbar_wait(&s_bar[wib], parity);
        parity ^= 1u;
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = s_tile[wib][k * 32 + lane];
      } else {
        load_tile(v, g, t, dim, lane);  // ragged last tile
      }
    }
    // non-zero flags (-0.0 == 0 is not a non-zero, sparse.py:167)
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      m |= ((uint32_t)(v[k].x != 0.f) << (4 * k)) | ((uint32_t)(v[k].y != 0.f) << (4 * k + 1)) |
           ((uint32_t)(v[k].z != 0.f) << (4 * k + 2)) | ((uint32_t)(v[k].w != 0.f) << (4 * k + 3));
    }
    if (LOAD == 1) {
      // every lane has consumed its shared-tile reads (m depends on all of v): release the
      // buffer to the async proxy and prefetch the next tile while this one is processed
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && t + nw < nfull) tma_load_1d(s_tile[wib], g + (t + nw) * kTile, kTile * 4, &s_bar[wib], pol);
    }
    if (MODE == 2) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        fin += 0.f * v[k].x + 0.f * v[k].y + 0.f * v[k].z + 0.f * v[k].w;
      // selection word of elements base+32L..+31, then the inverse transpose into m's layout
      uint32_t mword = bs == 1 ? ((t * 32 + lane) < nelem_words ? __ldg(bitmap + t * 32 + lane) : 0u)
                               : expand_blocks(bitmap, base + 32 * lane, dim, bs);
      const int64_t e0 = base + 32 * lane;
      if (e0 + 32 > dim) mword &= e0 >= dim ? 0u : range_mask(0, (int)(dim - e0));
      sel += __popc(mword);
      uint32_t msel = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t mk = __shfl_sync(kFull, mword, 4 * k + (lane >> 3));
        msel |= ((mk >> ((lane & 7) * 4)) & 0xFu) << (4 * k);
      }
      m &= msel;
    }
    const int cnt = __popc(m);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += n;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    uint32_t word = 0;  // MODE 0/1: non-zero word of elements base+32*lane..+31
    if (total) {
      if (MODE != 2) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t mq = __shfl_sync(kFull, m, src_grp + q);
          word |= ((mq >> src_sh) & 0xFu) << (4 * q);
        }
      }
      nnz += (unsigned)total;
      if (qn + total <= kCap) {
        int pos = qn + incl - cnt;
        if (LOAD == 0 || LOAD == 3) {
          // stage the tile (8 STS.128 per lane) so the append loop can index values dynamically:
          // ~popc(m) iterations instead of 32 per-element predicated appends
          float4* st = s_tile[wib];
#pragma unroll
          for (int k = 0; k < 8; ++k) st[k * 32 + lane] = v[k];
          __syncwarp();
          const float* sf = reinterpret_cast<const float*>(st);
          for (uint32_t mm = m; mm; mm &= mm - 1u) {
            const int b = __ffs(mm) - 1;  // bit 4k+c <-> tile offset 128k + 4*lane + c
            const uint32_t off = 128u * (uint32_t)(b >> 2) + 4u * lane + (uint32_t)(b & 3);
            qi[pos] = (uint32_t)base + off;
            qv[pos] = sf[off];
            ++pos;
          }
          __syncwarp();
        } else {
          const uint32_t e0 = (uint32_t)(base + lane * 4);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t nib = (m >> (4 * k)) & 0xFu;
            if (nib) {
              const uint32_t e = e0 + 128u * k;
              if (nib & 1u) { qi[pos] = e + 0; qv[pos] = v[k].x; ++pos; }
              if (nib & 2u) { qi[pos] = e + 1; qv[pos] = v[k].y; ++pos; }
              if (nib & 4u) { qi[pos] = e + 2; qv[pos] = v[k].z; ++pos; }
              if (nib & 8u) { qi[pos] = e + 3; qv[pos] = v[k].w; ++pos; }
            }
          }
        }
        qn += total;
        flush_full<R>(qi, qv, qn, lane, table, hp, bad);
      } else {
        // dense tile: append chunk by chunk (<= 128 per chunk), flushing in between
        const uint32_t lt = lanemask_lt();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t nib = (m >> (4 * k)) & 0xFu;
          const uint32_t b0 = __ballot_sync(kFull, nib & 1u);
          const uint32_t b1 = __ballot_sync(kFull, nib & 2u);
          const uint32_t b2 = __ballot_sync(kFull, nib & 4u);
          const uint32_t b3 = __ballot_sync(kFull, nib & 8u);
          int pos = qn + __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
          const int tot = __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
          const uint32_t e = (uint32_t)(base + k * 128 + lane * 4);
          if (nib & 1u) { qi[pos] = e + 0; qv[pos] = v[k].x; ++pos; }
          if (nib & 2u) { qi[pos] = e + 1; qv[pos] = v[k].y; ++pos; }
          if (nib & 4u) { qi[pos] = e + 2; qv[pos] = v[k].z; ++pos; }
          if (nib & 8u) { qi[pos] = e + 3; qv[pos] = v[k].w; ++pos; }
          qn += tot;
          flush_full<R>(qi, qv, qn, lane, table, hp, bad);
        }
      }
    }
    if (MODE == 0) {
      const int64_t wi = t * 32 + lane;
      if (wi < nelem_words) {
        bitmap[wi] = word;
        if constexpr (PUSH) {
#pragma unroll
          for (int q = 0; q < kMaxWorld; ++q)
            if (q < push.n) push.dst[q][wi] = word;
        }
      }
    } else if (MODE == 1) {
      if (word) {  // OR the flags of every block this 32-element span touches
        const int64_t e0 = base + 32 * lane;
        const int64_t e_end = e0 + 32 < dim ? e0 + 32 : dim;
        int64_t b = e0 / bs, s = e0;
        while (s < e_end) {
          int64_t be = (b + 1) * bs;
          if (be > e_end) be = e_end;
          if (word & range_mask((int)(s - e0), (int)(be - e0)))
            atomicOr(bitmap + (b >> 5), 1u << (b & 31));
          s = be;
          ++b;
        }
      }
    }
  }
  __syncwarp();
  if (lane < qn) {
    const float v = qv[lane];
    bad |= nonfinite(v);
    insert_one<R>(qi[lane], v, table, hp);
  }
  if (MODE == 2) bad |= (fin != 0.f);  // NaN != 0
  bad = __any_sync(kFull, bad);
  if (MODE == 2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sel += __shfl_xor_sync(kFull, sel, o);
  }
  if (lane == 0) {
    if (nnz) atomicAdd(counters + S2_CNT_NNZ, nnz);
    if (MODE == 0 && nnz) atomicAdd(counters + S2_CNT_SELECTED, nnz);
    if (MODE == 2 && sel) atomicAdd(counters + S2_CNT_SELECTED, sel);
    if (bad) atomicOr(counters + S2_CNT_NONFINITE, 1ull);
  }
  if constexpr (PUSH) {  // pushed words performed at system scope before the kernel ends
    if (push.fence == 1) {
      __threadfence_system();
    } else if (push.fence == 2) {
      __syncwarp();
      if (lane == 0) __threadfence_system();
    }
  }
  if constexpr (SIG) signal_done(sig);  // separate instantiation: no CTA barrier in the default kernel
}

// ------------------------------------------- compress, TMA-staged variant (default)
//
// Each warp owns a 2-stage ring of 4 KB shared tiles filled by cp.async.bulk (one
// elected lane, completion on a per-stage mbarrier), so a warp has up to two tiles
// (8 KB) in flight with no register cost.  Lane L reads ITS OWN 32 consecutive
// elements (base+32L..+31) from the staged tile — 8 LDS.128 with an XOR swizzle
// (chunk (k+L)&7 at step k) so the 8 lanes of each shared-memory phase hit 8
// different 16-byte bank groups — which makes its non-zero word m exactly bitmap
// word t*32+L: no transpose.  Non-zeros are appended to the per-warp queue by a
// loop over the set bits of m, reading values straight from the staged tile
// (~2 iterations per tile at 1% density instead of 32 per-element predicates).
constexpr int kTWarps = 4;             // warps per CTA
constexpr int kTStages = 2;            // tiles in flight per warp
constexpr int kTCap = 32 + 256;        // queue entries per warp
constexpr int kTSmemWarp = kTStages * kTile * 4 + kTCap * 8;
constexpr int kTSmemBytes = kTWarps * kTSmemWarp + kTWarps * kTStages * 8;

template <int R, int MODE>
__global__ void __launch_bounds__(kTWarps * 32, 5)
k_compress_tma(const float* __restrict__ g, int64_t dim, int64_t bs, uint32_t* __restrict__ bitmap,
               float* __restrict__ table, unsigned long long* __restrict__ counters,
               const __grid_constant__ HashParams hp) {
  extern __shared__ __align__(128) unsigned char s_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  float* tiles = reinterpret_cast<float*>(s_raw + wib * kTSmemWarp);  // [kTStages][kTile]
  uint32_t* qi = reinterpret_cast<uint32_t*>(s_raw + wib * kTSmemWarp + kTStages * kTile * 4);
  float* qv = reinterpret_cast<float*>(qi + kTCap);
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_raw + kTWarps * kTSmemWarp) + wib * kTStages;

  const int64_t ntiles = (dim + kTile - 1) / kTile;
  const int64_t nfull = dim / kTile;
  const int64_t nelem_words = (dim + 31) / 32;
  const int64_t nw = (int64_t)gridDim.x * kTWarps;
  const uint64_t pol = policy_evict_first();
  griddep_wait();
  griddep_launch_dependents();

  if (lane == 0) {
    for (int s = 0; s < kTStages; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
  }
  __syncwarp();
  int64_t t = (int64_t)blockIdx.x * kTWarps + wib;
  if (lane == 0) {
    for (int s = 0; s < kTStages; ++s) {
      const int64_t ts = t + s * nw;
      if (ts < nfull) tma_load_1d(tiles + s * kTile, g + ts * kTile, kTile * 4, &bars[s], pol);
    }
  }

  int qn = 0;
  unsigned long long nnz = 0;
  unsigned long long sel = 0;
  uint32_t bad = 0;
  float fin = 0.f;
  uint32_t parity = 0;  // bit s: phase of stage s
  int stage = 0;

#pragma unroll 1
  for (; t < ntiles; t += nw) {
    const int64_t base = t * kTile;
    float* tile = tiles + stage * kTile;
    if (t < nfull) {
      mbar_wait(&bars[stage], (parity >> stage) & 1u);
      parity ^= 1u << stage;
    } else {
      // ragged last tile: zero-filled copy through the generic proxy (no TMA in flight here)
      for (int e = lane; e < kTile; e += 32) tile[e] = base + e < dim ? g[base + e] : 0.f;
      __syncwarp();
    }
    // lane L: elements 32L..32L+31 of the tile, chunk c = (k + L) & 7 at step k
    uint32_t m = 0;
    const float4* row = reinterpret_cast<const float4*>(tile + 32 * lane);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = (k + lane) & 7;
      const float4 x = row[c];
      const uint32_t nib = (uint32_t)(x.x != 0.f) | ((uint32_t)(x.y != 0.f) << 1) |
                           ((uint32_t)(x.z != 0.f) << 2) | ((uint32_t)(x.w != 0.f) << 3);
      m |= nib << (4 * c);
      if (MODE == 2) fin += 0.f * x.x + 0.f * x.y + 0.f * x.z + 0.f * x.w;
    }
    const int64_t e0 = base + 32 * lane;
    if (MODE == 2) {
      uint32_t mword = bs == 1 ? ((t * 32 + lane) < nelem_words ? __ldg(bitmap + t * 32 + lane) : 0u)
                               : expand_blocks(bitmap, e0, dim, bs);
      if (e0 + 32 > dim) mword &= e0 >= dim ? 0u : range_mask(0, (int)(dim - e0));
      sel += __popc(mword);
      m &= mword;
    }
    const uint32_t word = m;  // MODE 0/1: the bitmap word of elements e0..e0+31
    const int cnt = __popc(m);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += n;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    nnz += (unsigned)total;
    if (qn + total <= kTCap) {
      int pos = qn + incl - cnt;
      for (uint32_t mm = m; mm; mm &= mm - 1u) {
        const int b = __ffs(mm) - 1;
        qi[pos] = (uint32_t)(e0 + b);
        qv[pos] = tile[32 * lane + b];
        ++pos;
      }
      qn += total;
    } else {
      // very dense tile: drain in rounds of at most kTCap - 32 entries
      int done = 0;  // entries of this tile already queued (warp-uniform)
      uint32_t mm = m;
      int mine = incl - cnt;  // my first rank within the tile
      while (done < total) {
        const int room = kTCap - qn;
        // queue my entries whose tile rank falls in [done, done + room)
        while (mm && mine < done + room) {
          const int b = __ffs(mm) - 1;
          const int pos = qn + (mine - done);
          qi[pos] = (uint32_t)(e0 + b);
          qv[pos] = tile[32 * lane + b];
          mm &= mm - 1u;
          ++mine;
        }
        const int take = total - done < room ? total - done : room;
        qn += take;
        done += take;
        flush_full<R>(qi, qv, qn, lane, table, hp, bad);
      }
    }
    // this tile's shared reads are done: hand the buffer back to the async proxy and
    // refill it with the tile kTStages rounds ahead
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      const int64_t tn = t + kTStages * nw;
      if (tn < nfull) tma_load_1d(tile, g + tn * kTile, kTile * 4, &bars[stage], pol);
    }
    stage = stage + 1 == kTStages ? 0 : stage + 1;
    if (MODE == 0) {
      if (t * 32 + lane < nelem_words) bitmap[t * 32 + lane] = word;
    } else if (MODE == 1) {
      if (word) {
        const int64_t e_end = e0 + 32 < dim ? e0 + 32 : dim;
        int64_t b = e0 / bs, s = e0;
        while (s < e_end) {
          int64_t be = (b + 1) * bs;
          if (be > e_end) be = e_end;
          if (word & range_mask((int)(s - e0), (int)(be - e0))) atomicOr(bitmap + (b >> 5), 1u << (b & 31));
          s = be;
          ++b;
        }
      }
    }
    flush_full<R>(qi, qv, qn, lane, table, hp, bad);
  }
  __syncwarp();
  if (lane < qn) {
    const float v = qv[lane];
    bad |= nonfinite(v);
    insert_one<R>(qi[lane], v, table, hp);
  }
  if (MODE == 2) bad |= (fin != 0.f);
  bad = __any_sync(kFull, bad);
  if (MODE == 2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sel += __shfl_xor_sync(kFull, sel, o);
  }
  if (lane == 0) {
    if (nnz) atomicAdd(counters + S2_CNT_NNZ, nnz);
    if (MODE == 0 && nnz) atomicAdd(counters + S2_CNT_SELECTED, nnz);
    if (MODE == 2 && sel) atomicAdd(counters + S2_CNT_SELECTED, sel);
    if (bad) atomicOr(counters + S2_CNT_NONFINITE, 1ull);
  }
}

// ---------------------------------------- compress, split variant: K1 (scan) + K2 (insert)
//
// K1 k_scan_compact: one warp per 1024-element tile (non-persistent grid, so the block
// scheduler balances the tail): coalesced float4 loads, non-zero word by shuffle
// transpose, bitmap store, then the tile's non-zeros are compacted (warp scan + one
// atomicAdd per tile for the list offset) into a global (index, value) list.  No hashing
// here, so the kernel is a lean streaming pass.
// K2 k_insert_list: every thread takes list entries and does the r hashes + r
// red.global.add.f32 — all 32 lanes busy, no per-warp queue.
__global__ void __launch_bounds__(kThreads)
k_scan_compact(const float* __restrict__ g, int64_t dim, uint32_t* __restrict__ bitmap, uint2* __restrict__ list,
               unsigned long long* __restrict__ counters) {
  __shared__ __align__(16) float4 s_tile[kWarps][kTile / 4];
  __shared__ int s_tot[kWarps];
  __shared__ unsigned long long s_base;
  griddep_wait();
  griddep_launch_dependents();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * kWarps + wib;
  const int64_t ntiles = (dim + kTile - 1) / kTile;
  const int64_t base = t * kTile;
  const int64_t nelem_words = (dim + 31) / 32;
  float4 v[8];
  uint32_t m = 0;
  if (t < ntiles) {
    load_tile(v, g, t, dim, lane);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      m |= ((uint32_t)(v[k].x != 0.f) << (4 * k)) | ((uint32_t)(v[k].y != 0.f) << (4 * k + 1)) |
           ((uint32_t)(v[k].z != 0.f) << (4 * k + 2)) | ((uint32_t)(v[k].w != 0.f) << (4 * k + 3));
    }
  }
  const int cnt = __popc(m);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += n;
  }
  const int total = __shfl_sync(kFull, incl, 31);
  if (lane == 0) s_tot[wib] = total;
  __syncthreads();
  // one list reservation per CTA (not per tile): the counter sees gridDim.x atomics
  if (threadIdx.x == 0) {
    int sum = 0;
    for (int w = 0; w < kWarps; ++w) {
      const int c = s_tot[w];
      s_tot[w] = sum;
      sum += c;
    }
    s_base = sum ? atomicAdd(counters + S2_CNT_NNZ, (unsigned long long)sum) : 0ull;
  }
  __syncthreads();
  if (t >= ntiles) return;
  uint32_t word = 0;
  if (total) {
    const int src_grp = 8 * (lane & 3), src_sh = 4 * (lane >> 2);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t mq = __shfl_sync(kFull, m, src_grp + q);
      word |= ((mq >> src_sh) & 0xFu) << (4 * q);
    }
    float4* st = s_tile[wib];
#pragma unroll
    for (int k = 0; k < 8; ++k) st[k * 32 + lane] = v[k];
    __syncwarp();
    const float* sf = reinterpret_cast<const float*>(st);
    unsigned long long pos = s_base + (unsigned long long)(s_tot[wib] + incl - cnt);
    for (uint32_t mm = m; mm; mm &= mm - 1u) {
      const int b = __ffs(mm) - 1;
      const uint32_t o = 128u * (uint32_t)(b >> 2) + 4u * lane + (uint32_t)(b & 3);
      list[pos++] = make_uint2((uint32_t)base + o, __float_as_uint(sf[o]));
    }
  }
  if (t * 32 + lane < nelem_words) bitmap[t * 32 + lane] = word;
}

template <int R>
__global__ void __launch_bounds__(256)
k_insert_list(const uint2* __restrict__ list, float* __restrict__ table, unsigned long long* __restrict__ counters,
              const __grid_constant__ HashParams hp) {
  griddep_wait();  // the list and its length come from k_scan_compact
  griddep_launch_dependents();
  const unsigned long long n = counters[S2_CNT_NNZ];
  uint32_t bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)n; i += stride) {
    const uint2 e = __ldcs(list + i);
    const float v = __uint_as_float(e.y);
    bad |= nonfinite(v);
    insert_one<R>(e.x, v, table, hp);
  }
  if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(counters + S2_CNT_NONFINITE, 1ull);
  if (blockIdx.x == 0 && threadIdx.x == 0) counters[S2_CNT_SELECTED] = n;
}

// =================================================================== launchers

// ------------------------------------- compress, warp-specialised variant (S2_COMPRESS_LOAD=5)
//
// One producer warp streams the CTA's tiles (t = blockIdx.x + j * gridDim.x) with cp.async.bulk
// (one elected lane, completion on a per-stage "full" mbarrier) into kWsDepth 4 KB stages per
// consumer warp; consumer warp c takes jobs j = c, c + C, ... (its own sub-ring, so a stage's
// phases are always waited in order by one warp), reads its 8 float4 per lane from the stage,
// runs the same scan / bitmap / queue / hash body as k_compress and releases the stage on its
// "empty" mbarrier once the values are queued.  Up to C x kWsDepth tiles per CTA in flight, no
// prefetch registers.
constexpr int kWsConsumers = 8;
constexpr int kWsDepth = 2;
constexpr int kWsStages = kWsConsumers * kWsDepth;
constexpr int kWsThreads = (kWsConsumers + 1) * 32;
constexpr int kWsSmem = kWsStages * kTile * 4 + kWsConsumers * (32 + kQFast) * 8 + 2 * kWsStages * 8;

template <int R>
__global__ void __launch_bounds__(kWsThreads, 2)
k_compress_ws(const float* __restrict__ g, int64_t dim, uint32_t* __restrict__ bitmap, float* __restrict__ table,
              unsigned long long* __restrict__ counters, const __grid_constant__ HashParams hp) {
  constexpr int kCap = 32 + kQFast;
  extern __shared__ __align__(128) unsigned char ws_smem[];
  float4* stages = reinterpret_cast<float4*>(ws_smem);                                     // [S][256]
  uint32_t* s_qi = reinterpret_cast<uint32_t*>(ws_smem + kWsStages * kTile * 4);          // [C][kCap]
  float* s_qv = reinterpret_cast<float*>(s_qi + kWsConsumers * kCap);                      // [C][kCap]
  uint64_t* full = reinterpret_cast<uint64_t*>(s_qv + kWsConsumers * kCap);                // [S]
  uint64_t* empty = full + kWsStages;                                                      // [S]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t ntiles = (dim + kTile - 1) / kTile;
  const int64_t nfull = dim / kTile;
  const int64_t nelem_words = (dim + 31) / 32;
  // tiles of this CTA: t_j = blockIdx.x + j * gridDim.x, j < njobs
  const int64_t njobs = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWsStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  griddep_wait();  // g may be written by the caller's previous kernel
  griddep_launch_dependents();

  if (warp == kWsConsumers) {  // producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int64_t j = 0; j < njobs; ++j) {
        const int64_t t = blockIdx.x + j * gridDim.x;
        if (t >= nfull) break;  // the ragged last tile is loaded by its consumer
        const int64_t k = j / kWsConsumers;  // the consumer's k-th job
        const int s = (int)(j % kWsConsumers) * kWsDepth + (int)(k % kWsDepth);
        if (k >= kWsDepth) mbar_wait(&empty[s], (uint32_t)(((k / kWsDepth) - 1) & 1));
        tma_load_1d(stages + s * (kTile / 4), g + t * kTile, kTile * 4, &full[s], pol);
      }
    }
    return;
  }

  // consumers
  uint32_t* qi = s_qi + warp * kCap;
  float* qv = s_qv + warp * kCap;
  const int src_grp = 8 * (lane & 3);
  const int src_sh = 4 * (lane >> 2);
  int qn = 0;
  unsigned long long nnz = 0;
  uint32_t bad = 0;
  for (int64_t j = warp; j < njobs; j += kWsConsumers) {
    const int64_t t = blockIdx.x + j * gridDim.x;
    const int64_t base = t * kTile;
    const int64_t kj = j / kWsConsumers;
    const int s = warp * kWsDepth + (int)(kj % kWsDepth);
    const bool staged = t < nfull;
    float4 v[8];
    const float4* st = stages + s * (kTile / 4);
    if (staged) {
      mbar_wait(&full[s], (uint32_t)((kj / kWsDepth) & 1));
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = st[k * 32 + lane];
    } else {
      load_tile(v, g, t, dim, lane);
    }
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      m |= ((uint32_t)(v[k].x != 0.f) << (4 * k)) | ((uint32_t)(v[k].y != 0.f) << (4 * k + 1)) |
           ((uint32_t)(v[k].z != 0.f) << (4 * k + 2)) | ((uint32_t)(v[k].w != 0.f) << (4 * k + 3));
    }
    const int cnt = __popc(m);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += n;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    uint32_t word = 0;
    if (total) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t mq = __shfl_sync(kFull, m, src_grp + q);
        word |= ((mq >> src_sh) & 0xFu) << (4 * q);
      }
      nnz += (unsigned)total;
      if (staged && qn + total <= kCap) {
        // walk the set bits, values straight from the stage (bit 4k+c <-> offset 128k + 4*lane + c)
        const float* sf = reinterpret_cast<const float*>(st);
        int pos = qn + incl - cnt;
        for (uint32_t mm = m; mm; mm &= mm - 1u) {
          const int b = __ffs(mm) - 1;
          const uint32_t off = 128u * (uint32_t)(b >> 2) + 4u * lane + (uint32_t)(b & 3);
          qi[pos] = (uint32_t)base + off;
          qv[pos] = sf[off];
          ++pos;
        }
        qn += total;
        flush_full<R>(qi, qv, qn, lane, table, hp, bad);
      } else {
      const uint32_t lt = lanemask_lt();
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // chunk by chunk (<= 128 per chunk), flushing full batches
        const uint32_t nib = (m >> (4 * k)) & 0xFu;
        const uint32_t b0 = __ballot_sync(kFull, nib & 1u);
        const uint32_t b1 = __ballot_sync(kFull, nib & 2u);
        const uint32_t b2 = __ballot_sync(kFull, nib & 4u);
        const uint32_t b3 = __ballot_sync(kFull, nib & 8u);
        const int tot = __popc(b0) + __popc(b1) + __popc(b2) + __popc(b3);
        if (tot == 0) continue;
        int pos = qn + __popc(b0 & lt) + __popc(b1 & lt) + __popc(b2 & lt) + __popc(b3 & lt);
        const uint32_t e = (uint32_t)(base + k * 128 + lane * 4);
        if (nib & 1u) { qi[pos] = e + 0; qv[pos] = v[k].x; ++pos; }
        if (nib & 2u) { qi[pos] = e + 1; qv[pos] = v[k].y; ++pos; }
        if (nib & 4u) { qi[pos] = e + 2; qv[pos] = v[k].z; ++pos; }
        if (nib & 8u) { qi[pos] = e + 3; qv[pos] = v[k].w; ++pos; }
        qn += tot;
        if (qn >= 32) flush_full<R>(qi, qv, qn, lane, table, hp, bad);
      }
      }
    }
    __syncwarp();
    if (staged && lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    const int64_t wi = t * 32 + lane;
    if (wi < nelem_words) bitmap[wi] = word;
  }
  __syncwarp();
  if (lane < qn) {
    const float v = qv[lane];
    bad |= nonfinite(v);
    insert_one<R>(qi[lane], v, table, hp);
  }
  bad = __any_sync(kFull, bad);
  if (lane == 0) {
    if (nnz) {
      atomicAdd(counters + S2_CNT_NNZ, nnz);
      atomicAdd(counters + S2_CNT_SELECTED, nnz);
    }
    if (bad) atomicOr(counters + S2_CNT_NONFINITE, 1ull);
  }
}

template <int R>
static void launch_compress_ws(const Plan& p, const float* g, uint32_t* bitmap, float* table,
                               unsigned long long* counters, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_compress_ws<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, kWsSmem);
    attr = true;
  }
  const int64_t ntiles = (p.dim + kTile - 1) / kTile;
  int64_t grid = (int64_t)num_sms() * 2;
  if (grid > ntiles) grid = ntiles;
  launch_ex(k_compress_ws<R>, (int)(grid < 1 ? 1 : grid), kWsThreads, kWsSmem, st, g, p.dim, bitmap, table, counters,
            p.hp);
}

// S2_COMPRESS_LOAD: 0 register prefetch (default: fastest measured, profiles/r01_*) |
//                   1 TMA prefetch, coalesced layout | 2 TMA-staged 2-stage ring, swizzled
static int compress_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("S2_COMPRESS_LOAD");
    v = e ? atoi(e) : 0;
    if (v < 0 || v > 5 || v == 4) v = 0;
  }
  return v;
}

template <int R, int LOAD>
static void launch_compress_rm(const Plan& p, const float* g, uint32_t* bitmap, float* table,
                               unsigned long long* counters, int mode, cudaStream_t st, const DoneSignal& sig,
                               const BitmapPush& push) {
  const int64_t ntiles = (p.dim + kTile - 1) / kTile;
  static int waves = -1;  // S2_COMPRESS_CTAS_PER_SM: grid = SMs x this (>= resident -> extra waves)
  if (waves < 0) {
    const char* e = getenv("S2_COMPRESS_CTAS_PER_SM");
    waves = e ? atoi(e) : 0;
  }
  const int grid = grid_for(ntiles, waves > 0 ? waves : (LOAD == 0 ? 2 : 4));
  if (mode == S2_MASK_GIVEN) {
    if (sig.done != nullptr)
      launch_ex(k_compress<R, 2, LOAD, true>, grid, kThreads, 0, st, g, p.dim, p.block_size, bitmap, table,
                counters, p.hp, sig, push);
    else
      launch_ex(k_compress<R, 2, LOAD>, grid, kThreads, 0, st, g, p.dim, p.block_size, bitmap, table, counters,
                p.hp, sig, push);
  } else if (p.block_size == 1) {
    if (push.n > 0)
      launch_ex(k_compress<R, 0, LOAD, false, true>, grid, kThreads, 0, st, g, p.dim, p.block_size, bitmap, table,
                counters, p.hp, sig, push);
    else if (sig.done != nullptr)
      launch_ex(k_compress<R, 0, LOAD, true>, grid, kThreads, 0, st, g, p.dim, p.block_size, bitmap, table,
                counters, p.hp, sig, push);
    else
      launch_ex(k_compress<R, 0, LOAD>, grid, kThreads, 0, st, g, p.dim, p.block_size, bitmap, table, counters,
                p.hp, sig, push);
  } else {
    if (sig.done != nullptr)
      launch_ex(k_compress<R, 1, LOAD, true>, grid, kThreads, 0, st, g, p.dim, p.block_size, bitmap, table,
                counters, p.hp, sig, push);
    else
      launch_ex(k_compress<R, 1, LOAD>, grid, kThreads, 0, st, g, p.dim, p.block_size, bitmap, table, counters,
                p.hp, sig, push);
  }
}

template <int R, int MODE>
static void launch_compress_tma(const Plan& p, const float* g, uint32_t* bitmap, float* table,
                                unsigned long long* counters, cudaStream_t st) {
  static bool attr = false;  // per instantiation
  if (!attr) {
    cudaFuncSetAttribute(k_compress_tma<R, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTSmemBytes);
    attr = true;
  }
  const int64_t ntiles = (p.dim + kTile - 1) / kTile;
  int64_t grid = (ntiles + kTWarps - 1) / kTWarps;
  const int64_t cap = (int64_t)num_sms() * 5;
  if (grid > cap) grid = cap;
  launch_ex(k_compress_tma<R, MODE>, (int)grid, kTWarps * 32, kTSmemBytes, st, g, p.dim, p.block_size, bitmap,
            table, counters, p.hp);
}

template <int R>
static void launch_compress_r(const Plan& p, const float* g, uint32_t* bitmap, float* table,
                              unsigned long long* counters, int mode, cudaStream_t st, const DoneSignal& sig,
                              const BitmapPush& push) {
  // the experimental load variants are instantiated for the default row count only
  const int v = (sig.done != nullptr || push.n > 0 || R != 3) ? 0 : compress_variant();
  if constexpr (R == 3) {
    if (v == 3) return launch_compress_rm<R, 3>(p, g, bitmap, table, counters, mode, st, sig, push);
    if (v == 1) return launch_compress_rm<R, 1>(p, g, bitmap, table, counters, mode, st, sig, push);
    if (v == 5 && mode != S2_MASK_GIVEN && p.block_size == 1)
      return launch_compress_ws<R>(p, g, bitmap, table, counters, st);
    if (v == 2) {
      if (mode == S2_MASK_GIVEN) return launch_compress_tma<R, 2>(p, g, bitmap, table, counters, st);
      if (p.block_size == 1) return launch_compress_tma<R, 0>(p, g, bitmap, table, counters, st);
      return launch_compress_tma<R, 1>(p, g, bitmap, table, counters, st);
    }
  }
  launch_compress_rm<R, 0>(p, g, bitmap, table, counters, mode, st, sig, push);
}

cudaError_t launch_compress(const Plan& p, const float* g, uint32_t* bitmap, float* table,
                            unsigned long long* counters, int mode, cudaStream_t st, bool prezeroed, void* list,
                            const DoneSignal* signal, const BitmapPush* bpush) {
  l2_window() = L2Window{table, sizeof(float) * (size_t)p.hp.rows * p.hp.cols};
  struct Reset {
    ~Reset() { l2_window() = L2Window{}; }
  } reset_window;
  DoneSignal sig{};
  if (signal != nullptr) sig = *signal;
  BitmapPush push{};
  if (bpush != nullptr && mode == S2_MASK_NONZERO && p.block_size == 1) push = *bpush;
  cudaError_t e = cudaSuccess;
  if (!prezeroed) {
    e = cudaMemsetAsync(table, 0, sizeof(float) * (size_t)p.hp.rows * p.hp.cols, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * S2_NUM_COUNTERS, st);
    if (e != cudaSuccess) return e;
  }
  if (mode == S2_MASK_NONZERO && p.block_size > 1) {
    e = cudaMemsetAsync(bitmap, 0, sizeof(uint32_t) * (size_t)p.words, st);
    if (e != cudaSuccess) return e;
  }
  if (list != nullptr && mode == S2_MASK_NONZERO && p.block_size == 1 && sig.done == nullptr && push.n == 0) {
    const int64_t ntiles = (p.dim + kTile - 1) / kTile;
    e = launch_ex(k_scan_compact, (int)((ntiles + kWarps - 1) / kWarps), kThreads, 0, st, g, p.dim, bitmap,
                  reinterpret_cast<uint2*>(list), counters);
    if (e != cudaSuccess) return e;
    const int grid = num_sms() * 8;
    switch (p.hp.rows) {
#define S2_CASE(r) \
  case r: e = launch_ex(k_insert_list<r>, grid, 256, 0, st, reinterpret_cast<const uint2*>(list), table, counters, p.hp); break;
      S2_CASE(1) S2_CASE(2) S2_CASE(3) S2_CASE(4) S2_CASE(5) S2_CASE(6) S2_CASE(7) S2_CASE(8)
#undef S2_CASE
      default: e = launch_ex(k_insert_list<0>, grid, 256, 0, st, reinterpret_cast<const uint2*>(list), table, counters, p.hp);
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  switch (p.hp.rows) {
    case 1: launch_compress_r<1>(p, g, bitmap, table, counters, mode, st, sig, push); break;
    case 3: launch_compress_r<3>(p, g, bitmap, table, counters, mode, st, sig, push); break;
    case 5: launch_compress_r<5>(p, g, bitmap, table, counters, mode, st, sig, push); break;
    default: launch_compress_r<0>(p, g, bitmap, table, counters, mode, st, sig, push); break;
  }
  if (mode == S2_MASK_NONZERO && p.block_size > 1) {
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_selected_count(p, bitmap, counters, st);
  }
  return cudaGetLastError();
}

}  // namespace s2
