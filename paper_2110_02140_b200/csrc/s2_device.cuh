// s2_device.cuh — shared device helpers and launch utilities of the S2 kernels
// (split across s2_compress.cu / s2_decode.cu / s2_kernels.cu so they compile in parallel).
#pragma once

#include <cstdio>
#include <cstdlib>
#include <utility>

#include "s2_common.cuh"
#include "s2_kernels.h"

namespace s2 {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kTile = 1024;

inline int num_sms() {
  static int g_num_sms = 0;
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// --------------------------------------------------- programmatic dependent launch
// k_compress / k_decode are launched with programmatic stream serialization: their CTAs
// become resident while the previous kernel drains, and griddepcontrol.wait holds them
// until that kernel's memory is visible.  Work that touches nothing the predecessor
// writes (the decode's zeroing of the NEXT ping-pong table) runs before the wait.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("S2_PDL");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ insert

// fp32 add into global memory that keeps subnormals.  red.global.add.f32 flushes subnormal
// inputs and results to zero (REDG.E.ADD.F32.FTZ.RN in SASS), while the reference adds in
// float64 (np.add.at, sketch.py:111).  Every fp32 value with |v| >= 2^-100 is a multiple of
// 2^-123, so any sum of such values is 0 or at least 2^-123 — a normal number — and the RED
// rounds exactly like an IEEE add.  Smaller values (never seen in real gradients) go through
// a CAS loop whose add is the IEEE, non-FTZ FADD (nvcc's default -ftz=false).  When tiny and
// normal contributions meet in one cell, a RED can still flush a subnormal intermediate:
// that error is < 2^-126, far below the 1e-5 * M tolerance of a cell holding a value >= 2^-100.
__device__ __forceinline__ void add_f32(float* p, float v) {
  if (!(fabsf(v) < 0x1p-100f)) {  // also NaN/Inf: one RED
    atomicAdd(p, v);               // RED.E.ADD.F32 (result unused)
    return;
  }
  unsigned int* a = reinterpret_cast<unsigned int*>(p);
  unsigned int old = *reinterpret_cast<volatile unsigned int*>(a), assumed;
  do {
    assumed = old;
    old = atomicCAS(a, assumed, __float_as_uint(__fadd_rn(__uint_as_float(assumed), v)));
  } while (old != assumed);
}

template <int R>
__device__ __forceinline__ void insert_one(uint64_t i, float v, float* __restrict__ table,
                                           const HashParams& hp) {
  const size_t cols = hp.cols;
  if (hp.mode == kInjective) {
    // injective mapping: bucket(i) = i, sign = +1 (core.py:131-141).  The host raises the
    // reference's ValueError for i >= cols (core.py:133-134); the guard keeps a direct C-ABI
    // caller from writing past the table.
    if (i >= cols) return;
#pragma unroll
    for (int j = 0; j < (R > 0 ? R : S2_MAX_ROWS); ++j) {
      if (R == 0 && j >= hp.rows) break;
      add_f32(table + j * cols + i, v);
    }
    return;
  }
  const uint64_t x = index_term(i);
#pragma unroll
  for (int j = 0; j < (R > 0 ? R : S2_MAX_ROWS); ++j) {
    if (R == 0 && j >= hp.rows) break;
    const uint64_t w = mix64(hp.seed[j] + x);
    const uint32_t b = bucket_of(w, hp);
    add_f32(table + j * cols + b, (w >> 63) ? -v : v);
  }
}

inline int grid_for(int64_t ntiles, int ctas_per_sm) {
  const int64_t want = (ntiles + kWarps - 1) / kWarps;
  const int64_t cap = (int64_t)num_sms() * ctas_per_sm;
  int64_t gr = want < cap ? want : cap;
  return gr < 1 ? 1 : (int)gr;
}

}  // namespace s2
