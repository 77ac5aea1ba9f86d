// s2_compress.cu — K1+K2: the fused compress kernel of the S2 sparse-sketch reduce.
//
// Replaces sparse_compress (sparse.py:151-171) + CountSketchTable.insert (sketch.py:102-112)
// + the non-zero mask rule (BlockMask(part, g != 0)): read g once with
// 128-bit streaming loads, build the bitmap words from the non-zero flags, compact the
// non-zeros into a per-warp shared queue by one warp scan, and insert every full batch of
// 32 queued values into the L2-resident sketch (r hashes + r fp32 adds per value).
//
// MODE 0: element bitmap (block size 1), mask = g != 0, bitmap words stored directly.
// MODE 1: block bitmap built from g != 0 (block size > 1), atomicOr into a zeroed bitmap.
// MODE 2: given block bitmap (any block size): insert the non-zeros of set blocks only.
//
// Per warp tile (1024 elements): lane l holds float4 chunks k = 0..7 at elements
// base + 128k + 4l (coalesced 512 B per load instruction).  Its 32 non-zero flags form
// one register m (bit 4k+c <-> element base+128k+4l+c).  The bitmap word of lane L
// (elements base+32L..+31) is the transpose of m across the 8-lane group (8 shuffles).
// The next tile's 8 float4 per lane are loaded into registers before the current tile is
// processed (127 registers, 2 CTAs = 16 warps per SM); every alternative that puts more
// bytes in flight (TMA rings, warp-specialised producer, bulk L2 prefetch, extra waves)
// measured slower (code at commit 17ff0c0, the last round-1 commit).
// NaN/Inf are non-zeros, so finiteness is tested on the queue only (MODE 2 tests every
// element: unselected non-zeros never reach the queue).
#include "s2_device.cuh"

namespace s2 {

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

template <int KF>
__device__ __forceinline__ void load_tile(float4 (&v)[KF], const float* __restrict__ g, int64_t t, int64_t dim,
                                          int lane) {
  constexpr int kT = 128 * KF;
  const int64_t base = t * kT;
  if (base + kT <= dim) {
    const float4* g4 = reinterpret_cast<const float4*>(g) + (base >> 2) + lane;
#pragma unroll
    for (int k = 0; k < KF; ++k) v[k] = __ldcs(g4 + k * 32);
  } else {
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      const int64_t e = base + k * 128 + lane * 4;
      v[k].x = e + 0 < dim ? g[e + 0] : 0.f;
      v[k].y = e + 1 < dim ? g[e + 1] : 0.f;
      v[k].z = e + 2 < dim ? g[e + 2] : 0.f;
      v[k].w = e + 3 < dim ? g[e + 3] : 0.f;
    }
  }
}

// KF = float4 chunks per lane per warp tile (kCompressKF = 8: 1024 elements, 127 registers,
// 2 CTAs per SM).
template <int R, int MODE, int KF>
__global__ void __launch_bounds__(kThreads, 2)
k_compress(const float* __restrict__ g, int64_t dim, int64_t bs, uint32_t* __restrict__ bitmap,
           float* __restrict__ table, unsigned long long* __restrict__ counters,
           const __grid_constant__ HashParams hp, int late_wait) {
  constexpr int kT = 128 * KF;  // elements per warp tile
  constexpr int kW = 4 * KF;    // bitmap words per warp tile
  constexpr int kCap = 32 + kQFast;
  __shared__ uint32_t s_qi[kWarps][kCap];
  __shared__ float s_qv[kWarps][kCap];
  __shared__ __align__(16) float4 s_tile[kWarps][kT / 4];  // value stage of the current tile
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  uint32_t* qi = s_qi[wib];
  float* qv = s_qv[wib];
  const int64_t ntiles = (dim + kT - 1) / kT;
  const int64_t nelem_words = (dim + 31) / 32;
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  const int src_grp = 8 * (lane & 3);  // transpose: word L gathers lanes 8(L&3)..+7
  const int src_sh = 4 * (lane >> 2);  //            at nibble k = L>>2

  int qn = 0;                  // warp-uniform queue depth
  unsigned long long nnz = 0;  // warp-uniform
  unsigned long long sel = 0;  // per-lane selected coordinates (MODE 2)
  uint32_t bad = 0;
  float fin = 0.f;  // MODE 2: sum of 0*x, NaN iff a non-finite element was seen

  if (!late_wait) griddep_wait();  // g may be written by the caller's previous kernel
  griddep_launch_dependents();
  int64_t t = (int64_t)blockIdx.x * kWarps + wib;
  float4 vn[KF];
  if (t < ntiles) load_tile<KF>(vn, g, t, dim, lane);
#pragma unroll 1
  for (; t < ntiles; t += nw) {
    const int64_t base = t * kT;
    float4 v[KF];
#pragma unroll
    for (int k = 0; k < KF; ++k) v[k] = vn[k];
    if (t + nw < ntiles) load_tile<KF>(vn, g, t + nw, dim, lane);  // prefetch the next tile
    // non-zero flags (-0.0 == 0 is not a non-zero, sparse.py:167)
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      m |= ((uint32_t)(v[k].x != 0.f) << (4 * k)) | ((uint32_t)(v[k].y != 0.f) << (4 * k + 1)) |
           ((uint32_t)(v[k].z != 0.f) << (4 * k + 2)) | ((uint32_t)(v[k].w != 0.f) << (4 * k + 3));
    }
    if (MODE == 2) {
#pragma unroll
      for (int k = 0; k < KF; ++k) fin += 0.f * v[k].x + 0.f * v[k].y + 0.f * v[k].z + 0.f * v[k].w;
      // selection word of elements base+32L..+31 (lanes L < kW), then the inverse transpose into m's layout
      uint32_t mword = 0;
      if (lane < kW) {
        mword = bs == 1 ? ((t * kW + lane) < nelem_words ? __ldg(bitmap + t * kW + lane) : 0u)
                        : expand_blocks(bitmap, base + 32 * lane, dim, bs);
        const int64_t e0 = base + 32 * lane;
        if (e0 + 32 > dim) mword &= e0 >= dim ? 0u : range_mask(0, (int)(dim - e0));
      }
      sel += __popc(mword);
      uint32_t msel = 0;
#pragma unroll
      for (int k = 0; k < KF; ++k) {
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
        // stage the tile (8 STS.128 per lane) so the append loop can index values dynamically:
        // ~popc(m) iterations instead of 32 per-element predicated appends
        int pos = qn + incl - cnt;
        float4* st = s_tile[wib];
#pragma unroll
        for (int k = 0; k < KF; ++k) st[k * 32 + lane] = v[k];
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
        qn += total;
        flush_full<R>(qi, qv, qn, lane, table, hp, bad);
      } else {
        // dense tile: append chunk by chunk (<= 128 per chunk), flushing in between
        const uint32_t lt = lanemask_lt();
#pragma unroll
        for (int k = 0; k < KF; ++k) {
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
      const int64_t wi = t * kW + lane;
      if (lane < kW && wi < nelem_words) bitmap[wi] = word;
    } else if (MODE == 1) {
      if (lane < kW && word) {  // OR the flags of every block this 32-element span touches
        const int64_t e0 = base + 32 * lane;
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
  if (late_wait) griddep_wait();  // complete only after the stream predecessor (see launch_compress)
}

// =================================================================== launchers

// float4 per lane per warp tile.  KF = 4 (512-element tiles, 64 registers, 32 warps per SM)
// measured slower than KF = 8: compress alone 30.8 vs 24.8 µs at the ResNet-50 config, the
// ResNet step 46.9 vs 42.0 µs (profiles/r02_ab_kf.txt): the per-tile fixed work (scan,
// transpose, queue bookkeeping) doubles per byte while the bytes in flight stay the same.
// KF = 8 squeezed to 80 registers for 3 CTAs (24 warps) per SM spills and is slower still:
// compress 26.2 -> 37.0 µs at ResNet-50, 237 -> 370 µs at GPT-2-M 99 % (profiles/r02_ab_occ.txt).
constexpr int kCompressKF = 8;

template <int R, int KF>
static cudaError_t launch_compress_rk(const Plan& p, const float* g, uint32_t* bitmap, float* table,
                                      unsigned long long* counters, int mode, cudaStream_t st, int late) {
  const int64_t ntiles = (p.dim + 128 * KF - 1) / (128 * KF);
  static int per_sm = -1;  // S2_COMPRESS_CTAS_PER_SM: grid = SMs x this (> resident -> extra waves)
  if (per_sm < 0) {
    const char* e = getenv("S2_COMPRESS_CTAS_PER_SM");
    per_sm = e && atoi(e) > 0 ? atoi(e) : 0;
  }
  const int grid = grid_for(ntiles, per_sm > 0 ? per_sm : 2);
  if (mode == S2_MASK_GIVEN)
    return launch_ex(k_compress<R, 2, KF>, grid, kThreads, 0, st, g, p.dim, p.block_size, bitmap, table, counters,
                     p.hp, late);
  if (p.block_size == 1)
    return launch_ex(k_compress<R, 0, KF>, grid, kThreads, 0, st, g, p.dim, p.block_size, bitmap, table, counters,
                     p.hp, late);
  return launch_ex(k_compress<R, 1, KF>, grid, kThreads, 0, st, g, p.dim, p.block_size, bitmap, table, counters,
                   p.hp, late);
}

template <int R>
static cudaError_t launch_compress_r(const Plan& p, const float* g, uint32_t* bitmap, float* table,
                                     unsigned long long* counters, int mode, cudaStream_t st, int late) {
  return launch_compress_rk<R, kCompressKF>(p, g, bitmap, table, counters, mode, st, late);
}

cudaError_t preload_compress(const Plan& p) {
  cudaFuncAttributes fa;
  switch (p.hp.rows) {
    case 1: return cudaFuncGetAttributes(&fa, k_compress<1, 0, kCompressKF>);
    case 3: return cudaFuncGetAttributes(&fa, k_compress<3, 0, kCompressKF>);
    case 5: return cudaFuncGetAttributes(&fa, k_compress<5, 0, kCompressKF>);
    default: return cudaFuncGetAttributes(&fa, k_compress<0, 0, kCompressKF>);
  }
}

cudaError_t launch_compress(const Plan& p, const float* g, uint32_t* bitmap, float* table,
                            unsigned long long* counters, int mode, cudaStream_t st, bool prezeroed, bool late_wait) {
  const int late = late_wait && prezeroed ? 1 : 0;  // memsets in between break the programmatic edge anyway
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
  switch (p.hp.rows) {
    case 1: e = launch_compress_r<1>(p, g, bitmap, table, counters, mode, st, late); break;
    case 3: e = launch_compress_r<3>(p, g, bitmap, table, counters, mode, st, late); break;
    case 5: e = launch_compress_r<5>(p, g, bitmap, table, counters, mode, st, late); break;
    default: e = launch_compress_r<0>(p, g, bitmap, table, counters, mode, st, late); break;
  }
  if (e != cudaSuccess) return e;
  if (mode == S2_MASK_NONZERO && p.block_size > 1) return launch_selected_count(p, bitmap, counters, st);
  return cudaGetLastError();
}

}  // namespace s2
