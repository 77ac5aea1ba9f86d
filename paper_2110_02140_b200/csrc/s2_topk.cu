// s2_topk.cu — block Top-K mask on the GPU: block_topk (sparse.py:70-80).
//
//   norms[b] = ||g[block b]||_2 in float64 (as np.linalg.norm on the float64 upcast)
//   order    = argsort(-norms, kind="stable")  -> ties go to the LOWER block index
//   flags    = the first k blocks of that order
//
// Selection is a radix select on the norm's float64 bit pattern (non-negative doubles
// order like their uint64 bits): 8 passes of 8-bit digits, each a shared-memory
// histogram of the candidates that still match the selected prefix, then a one-CTA
// step that picks the digit holding the k-th largest key.  The final pass sets every
// block above the threshold and the first `need` blocks equal to it in index order
// (word counts + exclusive scan), which reproduces the stable tie-break exactly.
#include <cstdint>

#include "s2_kernels.h"

namespace s2 {

struct TopkState {
  unsigned long long prefix;  // selected high digits of the threshold key
  unsigned long long mask;    // which bits of prefix are decided
  long long remaining;        // how many keys >= current prefix range are still needed
  long long gt;               // keys strictly above the final threshold
};

__global__ void k_block_norms_warp(const float* __restrict__ g, int64_t dim, int64_t nb, int64_t bs,
                                   unsigned long long* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = w; b < nb; b += nw) {
    int64_t s = b * bs, e = s + bs;
    if (s > dim) s = dim;
    if (e > dim) e = dim;
    double acc = 0.0;
    for (int64_t i = s + lane; i < e; i += 32) {
      const double x = (double)__ldg(g + i);
      acc = fma(x, x, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if (lane == 0) keys[b] = (unsigned long long)__double_as_longlong(sqrt(acc));
  }
}

__global__ void __launch_bounds__(256) k_block_norms_cta(const float* __restrict__ g, int64_t dim, int64_t nb,
                                                         int64_t bs, unsigned long long* __restrict__ keys) {
  __shared__ double s_part[8];
  for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
    int64_t s = b * bs, e = s + bs;
    if (s > dim) s = dim;
    if (e > dim) e = dim;
    double acc = 0.0;
    for (int64_t i = s + threadIdx.x; i < e; i += blockDim.x) {
      const double x = (double)__ldg(g + i);
      acc = fma(x, x, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int k = 0; k < 8; ++k) t += s_part[k];
      keys[b] = (unsigned long long)__double_as_longlong(sqrt(t));
    }
    __syncthreads();
  }
}

__global__ void k_topk_init(TopkState* st, int64_t k, unsigned int* hist) {
  st->prefix = 0;
  st->mask = 0;
  st->remaining = k;
  st->gt = 0;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
}

__global__ void __launch_bounds__(256) k_topk_hist(const unsigned long long* __restrict__ keys, int64_t nb,
                                                   const TopkState* __restrict__ st, int shift,
                                                   unsigned int* __restrict__ hist) {
  __shared__ unsigned int s_h[256];
  s_h[threadIdx.x] = 0;
  __syncthreads();
  const unsigned long long prefix = st->prefix, mask = st->mask;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = keys[i];
    if ((key & mask) == prefix) atomicAdd(&s_h[(key >> shift) & 0xFFu], 1u);
  }
  __syncthreads();
  if (s_h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], s_h[threadIdx.x]);
}

// one thread: walk digits from the top, find where the running count reaches `remaining`
__global__ void k_topk_pick(TopkState* st, int shift, unsigned int* hist) {
  long long run = 0;
  int d = 255;
  for (; d > 0; --d) {
    if (run + (long long)hist[d] >= st->remaining) break;
    run += hist[d];
  }
  st->gt += run;
  st->remaining -= run;
  st->prefix |= (unsigned long long)d << shift;
  st->mask |= 0xFFull << shift;
  for (int i = 0; i < 256; ++i) hist[i] = 0;
}

// per 32-block word: count of keys equal to the threshold
__global__ void k_topk_eqcount(const unsigned long long* __restrict__ keys, int64_t nb,
                               const TopkState* __restrict__ st, int64_t* __restrict__ cnt) {
  const int64_t words = (nb + 31) / 32;
  const unsigned long long thr = st->prefix;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    for (int k = 0; k < 32; ++k) {
      const int64_t i = w * 32 + k;
      if (i < nb && keys[i] == thr) ++c;
    }
    cnt[w] = c;
  }
}

__global__ void k_topk_flags(const unsigned long long* __restrict__ keys, int64_t nb, const TopkState* __restrict__ st,
                             const int64_t* __restrict__ eq_before, uint32_t* __restrict__ bitmap) {
  const int64_t words = (nb + 31) / 32;
  const unsigned long long thr = st->prefix;
  const long long need = st->remaining;  // equal keys to take, lowest index first
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bits = 0;
    long long rank = eq_before[w];
    for (int k = 0; k < 32; ++k) {
      const int64_t i = w * 32 + k;
      if (i >= nb) break;
      const unsigned long long key = keys[i];
      if (key > thr) {
        bits |= 1u << k;
      } else if (key == thr) {
        if (rank < need) bits |= 1u << k;
        ++rank;
      }
    }
    bitmap[w] = bits;
  }
}

int64_t topk_scratch_bytes(const Plan& p) {
  const int64_t nb = p.num_blocks, words = (nb + 31) / 32;
  return nb * 8 + (words + 1) * 8 + 256 * 4 + 64 + 256;
}

cudaError_t launch_block_topk(const Plan& p, const float* g, int64_t k, uint32_t* bitmap, void* scratch,
                              cudaStream_t st) {
  const int64_t nb = p.num_blocks, words = (nb + 31) / 32;
  char* s = static_cast<char*>(scratch);
  auto* keys = reinterpret_cast<unsigned long long*>(s);
  auto* eq = reinterpret_cast<int64_t*>(s + nb * 8);
  auto* hist = reinterpret_cast<unsigned int*>(s + nb * 8 + (words + 1) * 8);
  auto* state = reinterpret_cast<TopkState*>(s + nb * 8 + (words + 1) * 8 + 256 * 4);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (nb >= 4096) {
    int64_t grid = (nb * 32 + 255) / 256;
    if (grid > (int64_t)sms * 16) grid = (int64_t)sms * 16;
    k_block_norms_warp<<<(int)grid, 256, 0, st>>>(g, p.dim, nb, p.block_size, keys);
  } else {
    k_block_norms_cta<<<(int)nb, 256, 0, st>>>(g, p.dim, nb, p.block_size, keys);
  }
  k_topk_init<<<1, 256, 0, st>>>(state, k, hist);
  int64_t grid = (nb + 255) / 256;
  if (grid > (int64_t)sms * 8) grid = (int64_t)sms * 8;
  for (int shift = 56; shift >= 0; shift -= 8) {
    k_topk_hist<<<(int)grid, 256, 0, st>>>(keys, nb, state, shift, hist);
    k_topk_pick<<<1, 1, 0, st>>>(state, shift, hist);
  }
  int64_t gw = (words + 255) / 256;
  if (gw > (int64_t)sms * 8) gw = (int64_t)sms * 8;
  k_topk_eqcount<<<(int)gw, 256, 0, st>>>(keys, nb, state, eq);
  cudaError_t e = launch_exclusive_scan(eq, words, eq + words, st);
  if (e != cudaSuccess) return e;
  k_topk_flags<<<(int)gw, 256, 0, st>>>(keys, nb, state, eq, bitmap);
  return cudaGetLastError();
}

}  // namespace s2
