// s2_common.cuh — hash family and shared device helpers for the S2 sparse-sketch path.
//
// Bit-exact restatement of the reference hash contract
// (/root/reference/pkg/src/sketchgrad/core.py):
//   mix64          core.py:27-38   splitmix64 finalizer, wraps mod 2^64
//   derive_seed    core.py:44-54   acc = mix64(acc + part*G) from 0x243F6A8885A308D3
//   _hash_words    core.py:70-75   w = mix64(seed_j + (i+1)*G)
//   hash_buckets   core.py:89-100  (w & (2^63-1)) % cols
//   hash_signs     core.py:103-106 1 - 2*(w >> 63)
// Bucket and sign come from the SAME 64-bit word.
//
// `% cols` for a non-power-of-two `cols` is replaced by a multiply-high with a
// precomputed magic (Granlund–Montgomery round-up method for 63-bit dividends):
//   l = ceil(log2 cols), m = ceil(2^(63+l) / cols) < 2^64,
//   q = umulhi(x, m) >> (l-1) == floor(x / cols) for every x < 2^63,
// because e = m*cols - 2^(63+l) lies in (0, cols) and cols <= 2^l.
// The 64-bit `%` would otherwise compile to a CALL to the remainder routine.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "s2.h"

namespace s2 {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;   // core.py:18
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;     // core.py:19
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;     // core.py:20
constexpr uint64_t kMask63 = 0x7FFFFFFFFFFFFFFFull;   // core.py:17
constexpr uint64_t kDeriveInit = 0x243F6A8885A308D3ull;  // core.py:41

enum BucketMode : uint32_t {
  kPow2 = 0,       // cols is a power of two: mask
  kMagic = 1,      // multiply-high division
  kInjective = 2,  // HashMapping(injective=True): bucket(i) = i, sign = +1 (core.py:130-141)
};

// Everything a kernel needs to evaluate h_j(i) and s_j(i); passed by value
// (__grid_constant__) so row seeds live in the constant bank.
struct HashParams {
  uint64_t seed[S2_MAX_ROWS];  // derive_seed(seed, j) (sketch.py:96-99)
  uint64_t magic;
  uint32_t shift;  // l - 1
  uint32_t cols;   // < 2^32
  uint32_t mode;   // BucketMode
  int32_t rows;
};

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t umulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// bucket of a raw hash word (core.py:99-100); not used for kInjective
__host__ __device__ __forceinline__ uint32_t bucket_of(uint64_t w, const HashParams& hp) {
  const uint64_t x = w & kMask63;
  if (hp.mode == kPow2) return (uint32_t)x & (hp.cols - 1u);
  const uint64_t q = umulhi64(x, hp.magic) >> hp.shift;
  return (uint32_t)x - (uint32_t)q * hp.cols;  // remainder < cols < 2^32
}

// (i+1)*G, shared by every row of index i (core.py:75)
__host__ __device__ __forceinline__ uint64_t index_term(uint64_t i) { return (i + 1ull) * kGolden; }

#ifdef __CUDACC__
constexpr unsigned kFull = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// non-finite test on the raw bits (exponent all ones) — as_gradient's isfinite (core.py:157)
__device__ __forceinline__ uint32_t nonfinite(float v) {
  return (__float_as_uint(v) & 0x7F800000u) == 0x7F800000u;
}

__device__ __forceinline__ uint32_t range_mask(int lo, int hi) {  // bits [lo, hi)
  const int n = hi - lo;
  return n >= 32 ? 0xFFFFFFFFu : (((1u << n) - 1u) << lo);
}

// Element-level selection word for elements [e0, e0+32) under a block bitmap with
// block size bs (BlockPartition core.py:172-211: block b covers [b*bs, min((b+1)*bs, dim))).
__device__ __forceinline__ uint32_t expand_blocks(const uint32_t* __restrict__ flags, int64_t e0,
                                                  int64_t dim, int64_t bs) {
  if (e0 >= dim) return 0u;
  const int64_t e_end = e0 + 32 < dim ? e0 + 32 : dim;
  uint32_t word = 0;
  int64_t b = e0 / bs;
  int64_t s = e0;
  while (s < e_end) {
    int64_t be = (b + 1) * bs;
    if (be > e_end) be = e_end;
    if ((__ldg(flags + (b >> 5)) >> (b & 31)) & 1u) word |= range_mask((int)(s - e0), (int)(be - e0));
    s = be;
    ++b;
  }
  return word;
}
#endif

}  // namespace s2
