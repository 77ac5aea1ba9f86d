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

// Optional L2 persistence for the sketch table (S2_L2_PERSIST=1): the table is the only
// data with reuse (r atomics / gathers per value against a 3-50 MB table) while the
// gradient and the output stream through once; an access-policy window marks it
// persisting so the streams cannot evict it.
struct L2Window {
  const void* base = nullptr;
  size_t bytes = 0;
};
inline L2Window& l2_window() {
  static thread_local L2Window w;
  return w;
}
inline bool l2_persist_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("S2_L2_PERSIST");
    v = e ? atoi(e) : 0;
    if (v) {
      int dev = 0, maxp = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
      if (maxp <= 0 || cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp) != cudaSuccess) {
        cudaGetLastError();
        v = 0;
      }
    }
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
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const L2Window& w = l2_window();
  if (w.base != nullptr && l2_persist_enabled()) {
    attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[1].val.accessPolicyWindow.base_ptr = const_cast<void*>(w.base);
    attr[1].val.accessPolicyWindow.num_bytes = w.bytes;
    attr[1].val.accessPolicyWindow.hitRatio = 1.0f;
    attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.numAttrs = 2;
  }
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ insert

template <int R>
__device__ __forceinline__ void insert_one(uint64_t i, float v, float* __restrict__ table,
                                           const HashParams& hp) {
  const size_t cols = hp.cols;
  if (hp.mode == kInjective) {
    // injective mapping: bucket(i) = i, sign = +1 (core.py:131-141)
#pragma unroll
    for (int j = 0; j < (R > 0 ? R : S2_MAX_ROWS); ++j) {
      if (R == 0 && j >= hp.rows) break;
      atomicAdd(table + j * cols + i, v);
    }
    return;
  }
  const uint64_t x = index_term(i);
#pragma unroll
  for (int j = 0; j < (R > 0 ? R : S2_MAX_ROWS); ++j) {
    if (R == 0 && j >= hp.rows) break;
    const uint64_t w = mix64(hp.seed[j] + x);
    const uint32_t b = bucket_of(w, hp);
    atomicAdd(table + j * cols + b, (w >> 63) ? -v : v);  // RED.E.ADD.F32 (result unused)
  }
}

inline int grid_for(int64_t ntiles, int ctas_per_sm) {
  const int64_t want = (ntiles + kWarps - 1) / kWarps;
  const int64_t cap = (int64_t)num_sms() * ctas_per_sm;
  int64_t gr = want < cap ? want : cap;
  return gr < 1 ? 1 : (int)gr;
}

}  // namespace s2
