// s2_kernels.cu — the functional-API kernels of the S2 path (the reduce's K1+K2 live in
// s2_compress.cu, K4 in s2_decode.cu, K3 in s2_p2p.cu).
//
//   K3b    k_bitmap_or — BlockMask.union over W gathered bitmaps (sparse.py:55-58)
//   pairs  k_insert_pairs / k_query_pairs — CountSketchTable.insert / .query on index
//          lists (sketch.py:102-128)
//   aux    k_compact_* (ordered (idx,val) compaction = selected_indices,
//          sparse.py:44-49 / :164-168), k_selected_count (sparse.py:51-53),
//          k_table_sum (sketch.py:213-216).
//
// Data layout: g float32[dim]; bitmap uint32[ceil(num_blocks/32)] LE bit order;
// table float32[rows][cols] row-major.  A warp tile is 1024 elements = 32
// bitmap words = 8 float4 per lane.
#include "s2_device.cuh"
#include "s2_decode.cuh"

namespace s2 {

// ----------------------------------------------------------- bitmap OR (K3b)

__global__ void k_bitmap_or(const uint32_t* __restrict__ stacked, int64_t words, int nmasks,
                            uint32_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((words & 3) == 0 && (((uintptr_t)stacked | (uintptr_t)out) & 15) == 0) {
    const int64_t w4 = words >> 2;
    const uint4* s4 = reinterpret_cast<const uint4*>(stacked);
    for (int64_t i = i0; i < w4; i += stride) {
      uint4 a = __ldcs(s4 + i);
      for (int m = 1; m < nmasks; ++m) {
        const uint4 b = __ldcs(s4 + (int64_t)m * w4 + i);
        a.x |= b.x; a.y |= b.y; a.z |= b.z; a.w |= b.w;
      }
      reinterpret_cast<uint4*>(out)[i] = a;
    }
  } else {
    for (int64_t i = i0; i < words; i += stride) {
      uint32_t a = stacked[i];
      for (int m = 1; m < nmasks; ++m) a |= stacked[(int64_t)m * words + i];
      out[i] = a;
    }
  }
}

// -------------------------------------------------------- table sum (merge)

__global__ void k_table_sum(const float* __restrict__ stacked, int64_t cells, int ntables,
                            float* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cells; i += stride) {
    float a = stacked[i];
    for (int m = 1; m < ntables; ++m) a += stacked[(int64_t)m * cells + i];  // left fold
    out[i] = a;
  }
}

// ----------------------------------------- selected coordinates (alpha * dim)

__global__ void k_selected_count(const uint32_t* __restrict__ bitmap, int64_t num_blocks,
                                 int64_t dim, int64_t bs, unsigned long long* __restrict__ counters) {
  const int64_t words = (num_blocks + 31) / 32;
  unsigned long long acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += stride) {
    uint32_t bits = bitmap[w];
    const int64_t b0 = w * 32;
    if (b0 + 32 > num_blocks) bits &= range_mask(0, (int)(num_blocks - b0));
    if ((b0 + 32) * bs <= dim) {
      acc += (unsigned long long)__popc(bits) * (unsigned long long)bs;
    } else {
      for (; bits; bits &= bits - 1u) {  // ragged / empty tail blocks (core.py:202-206)
        const int64_t b = b0 + __ffs(bits) - 1;
        int64_t st = b * bs, en = st + bs;
        if (st > dim) st = dim;
        if (en > dim) en = dim;
        acc += (unsigned long long)(en - st);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(counters + S2_CNT_SELECTED, acc);
}

// ------------------------------------------------- ordered compaction (aux)
//
// Three passes over 1024-element tiles: count, exclusive scan, write.  The
// element word of lane L covers elements base+32L..+31; with g != NULL it is
// ANDed with the non-zero bits of g (sparse.py:164-168).

__device__ __forceinline__ uint32_t compact_word(const uint32_t* __restrict__ bitmap,
                                                 const float* __restrict__ g, int64_t dim,
                                                 int64_t bs, int64_t e0, float (&vals)[32]) {
  uint32_t word;
  if (bs == 1) {
    word = e0 < dim ? __ldg(bitmap + (e0 >> 5)) : 0u;
  } else {
    word = expand_blocks(bitmap, e0, dim, bs);
  }
  if (e0 + 32 > dim) word &= e0 >= dim ? 0u : range_mask(0, (int)(dim - e0));
  if (g != nullptr && word) {
    uint32_t nzw = 0;
    if (e0 + 32 <= dim) {
      const float4* p = reinterpret_cast<const float4*>(g + e0);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float4 x = __ldg(p + k);
        vals[4 * k + 0] = x.x; vals[4 * k + 1] = x.y; vals[4 * k + 2] = x.z; vals[4 * k + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 32; ++k) vals[k] = e0 + k < dim ? g[e0 + k] : 0.f;
    }
#pragma unroll
    for (int k = 0; k < 32; ++k) nzw |= (uint32_t)(vals[k] != 0.f) << k;
    word &= nzw;
  }
  return word;
}

__global__ void __launch_bounds__(kThreads)
k_compact_count(const uint32_t* __restrict__ bitmap, const float* __restrict__ g, int64_t dim,
                int64_t bs, int64_t* __restrict__ tile_counts) {
  const int lane = threadIdx.x & 31;
  const int64_t ntiles = (dim + kTile - 1) / kTile;
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  for (int64_t t = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); t < ntiles; t += nw) {
    float vals[32];
    const uint32_t word = compact_word(bitmap, g, dim, bs, t * kTile + 32 * lane, vals);
    int c = __popc(word);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if (lane == 0) tile_counts[t] = c;
  }
}

// single-CTA exclusive scan of n int64 counts (in place); total into *total
__global__ void __launch_bounds__(1024) k_scan(int64_t* __restrict__ a, int64_t n,
                                               int64_t* __restrict__ total) {
  __shared__ int64_t s_warp[32];
  const int tid = threadIdx.x;
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t lo = tid * per;
  const int64_t hi = lo + per < n ? lo + per : n;
  int64_t sum = 0;
  for (int64_t i = lo; i < hi; ++i) sum += a[i];
  // block exclusive scan of sum
  const int lane = tid & 31, wid = tid >> 5;
  int64_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t v = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int64_t ws = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
    int64_t wi = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t v = __shfl_up_sync(kFull, wi, o);
      if (lane >= o) wi += v;
    }
    s_warp[lane] = wi - ws;
    if (lane == 31) *total = wi;
  }
  __syncthreads();
  int64_t run = s_warp[wid] + inc - sum;
  for (int64_t i = lo; i < hi; ++i) {
    const int64_t c = a[i];
    a[i] = run;
    run += c;
  }
}

__global__ void __launch_bounds__(kThreads)
k_compact_write(const uint32_t* __restrict__ bitmap, const float* __restrict__ g, int64_t dim,
                int64_t bs, const int64_t* __restrict__ tile_offsets, int64_t* __restrict__ idx_out,
                float* __restrict__ val_out) {
  const int lane = threadIdx.x & 31;
  const int64_t ntiles = (dim + kTile - 1) / kTile;
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  for (int64_t t = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); t < ntiles; t += nw) {
    float vals[32];
    const int64_t e0 = t * kTile + 32 * lane;
    uint32_t word = compact_word(bitmap, g, dim, bs, e0, vals);
    const int cnt = __popc(word);
    int pre = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(kFull, pre, o);
      if (lane >= o) pre += n;
    }
    int64_t pos = tile_offsets[t] + pre - cnt;
    for (; word; word &= word - 1u) {
      const int b = __ffs(word) - 1;
      idx_out[pos] = e0 + b;
      if (val_out != nullptr) {
#pragma unroll
        for (int k = 0; k < 32; ++k)
          if (k == b) val_out[pos] = vals[k];
      }
      ++pos;
    }
  }
}

// ------------------------------------- CountSketchTable.insert / .query (pairs)

template <int R>
__global__ void k_insert_pairs(const int64_t* __restrict__ idx, const float* __restrict__ vals, int64_t n,
                               float* __restrict__ table, const __grid_constant__ HashParams hp) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
    const float v = vals[k];
    if (v != 0.f) insert_one<R>((uint64_t)idx[k], v, table, hp);  // zero values are no-ops (sketch.py:103)
  }
}

template <int R>
__global__ void k_query_pairs(const int64_t* __restrict__ idx, int64_t n, const float* __restrict__ table,
                              float* __restrict__ out, const __grid_constant__ HashParams hp) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride)
    out[k] = query_one<R>((uint64_t)idx[k], table, hp);
}

// =================================================================== launchers

cudaError_t launch_bitmap_or(int64_t words, const uint32_t* stacked, int nmasks, uint32_t* out,
                             cudaStream_t st) {
  if (words <= 0) return cudaSuccess;
  const int64_t n = (words & 3) == 0 ? words / 4 : words;
  int64_t grid = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  k_bitmap_or<<<(int)grid, 256, 0, st>>>(stacked, words, nmasks, out);
  return cudaGetLastError();
}

cudaError_t launch_table_sum(int64_t cells, const float* stacked, int ntables, float* out,
                             cudaStream_t st) {
  if (cells <= 0) return cudaSuccess;
  int64_t grid = (cells + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  k_table_sum<<<(int)grid, 256, 0, st>>>(stacked, cells, ntables, out);
  return cudaGetLastError();
}

cudaError_t launch_selected_count(const Plan& p, const uint32_t* bitmap,
                                  unsigned long long* counters, cudaStream_t st) {
  int64_t grid = (p.words + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  k_selected_count<<<(int)grid, 256, 0, st>>>(bitmap, p.num_blocks, p.dim, p.block_size, counters);
  return cudaGetLastError();
}

cudaError_t launch_exclusive_scan(int64_t* a, int64_t n, int64_t* total, cudaStream_t st) {
  k_scan<<<1, 1024, 0, st>>>(a, n, total);
  return cudaGetLastError();
}

int64_t compact_scratch_bytes(const Plan& p) {
  const int64_t ntiles = (p.dim + kTile - 1) / kTile;
  return (ntiles + 1) * (int64_t)sizeof(int64_t);
}

cudaError_t launch_compact(const Plan& p, const uint32_t* bitmap, const float* g, int64_t* idx_out,
                           float* val_out, int64_t* count, void* scratch, cudaStream_t st) {
  const int64_t ntiles = (p.dim + kTile - 1) / kTile;
  int64_t* tiles = reinterpret_cast<int64_t*>(scratch);
  const int grid = grid_for(ntiles, 4);
  k_compact_count<<<grid, kThreads, 0, st>>>(bitmap, g, p.dim, p.block_size, tiles);
  k_scan<<<1, 1024, 0, st>>>(tiles, ntiles, count);
  if (idx_out != nullptr)  // idx_out == NULL: count only (size the output first)
    k_compact_write<<<grid, kThreads, 0, st>>>(bitmap, g, p.dim, p.block_size, tiles, idx_out, val_out);
  return cudaGetLastError();
}

template <int R>
static void launch_pairs_r(const Plan& p, const int64_t* idx, const float* vals, int64_t n, float* table,
                           float* out, cudaStream_t st) {
  int64_t grid = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (grid > cap) grid = cap;
  if (vals) k_insert_pairs<R><<<(int)grid, 256, 0, st>>>(idx, vals, n, table, p.hp);
  else k_query_pairs<R><<<(int)grid, 256, 0, st>>>(idx, n, table, out, p.hp);
}

cudaError_t launch_pairs(const Plan& p, const int64_t* idx, const float* vals, int64_t n, const float* table_in,
                         float* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  float* table = const_cast<float*>(table_in);
  if (p.hp.rows < 1 || p.hp.rows > S2_MAX_ROWS) return cudaErrorInvalidValue;
  if (p.hp.rows == 3) launch_pairs_r<3>(p, idx, vals, n, table, out, st);  // the default sketch
  else launch_pairs_r<0>(p, idx, vals, n, table, out, st);                 // any rows <= 16
  return cudaGetLastError();
}

}  // namespace s2
