// kbench.cu — micro-kernels that isolate the memory patterns of the S2 kernels
// (experiments only; not part of libs2.so).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC tools/kbench.cu -o tools/libkbench.so
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kTile = 1024;

template <int MODE>
__device__ __forceinline__ float4 ld(const float4* p) {
  if (MODE == 0) return __ldcs(p);
  if (MODE == 1) return __ldg(p);
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// read pattern of k_compress: warp tile of 1024 floats, 8 float4 per lane, optional prefetch
template <int MODE, bool PREFETCH, int UNROLL>
__global__ void __launch_bounds__(256) k_read(const float* __restrict__ g, int64_t n, uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t ntiles = n / kTile;
  const int64_t nw = (int64_t)gridDim.x * 8;
  int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  uint32_t acc = 0;
  float4 vn[UNROLL];
  if (PREFETCH && t < ntiles)
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) vn[k] = ld<MODE>(g4 + t * (kTile / 4) + k * 32 + lane);
  for (; t < ntiles; t += nw) {
    float4 v[UNROLL];
    if (PREFETCH) {
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) v[k] = vn[k];
      if (t + nw < ntiles)
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) vn[k] = ld<MODE>(g4 + (t + nw) * (kTile / 4) + k * 32 + lane);
    } else {
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) v[k] = ld<MODE>(g4 + t * (kTile / 4) + k * 32 + lane);
    }
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < UNROLL; ++k)
      m |= ((uint32_t)(v[k].x != 0.f) << (4 * k)) | ((uint32_t)(v[k].y != 0.f) << (4 * k + 1)) |
           ((uint32_t)(v[k].z != 0.f) << (4 * k + 2)) | ((uint32_t)(v[k].w != 0.f) << (4 * k + 3));
    acc ^= m;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// store pattern of k_decode: 8 float4 streaming stores per lane per tile
template <bool STREAM>
__global__ void __launch_bounds__(256) k_write(float* __restrict__ o, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t ntiles = n / kTile;
  const int64_t nw = (int64_t)gridDim.x * 8;
  float4* o4 = reinterpret_cast<float4*>(o);
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); t < ntiles; t += nw) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (STREAM) __stcs(o4 + t * (kTile / 4) + k * 32 + lane, z);
      else o4[t * (kTile / 4) + k * 32 + lane] = z;
    }
  }
}

extern "C" int kb_read(const float* g, int64_t n, uint32_t* out, int mode, int prefetch, int grid, void* st) {
  cudaStream_t s = (cudaStream_t)st;
#define L(M, P) k_read<M, P, 8><<<grid, 256, 0, s>>>(g, n, out)
  if (mode == 0) { if (prefetch) L(0, true); else L(0, false); }
  else if (mode == 1) { if (prefetch) L(1, true); else L(1, false); }
  else { if (prefetch) L(2, true); else L(2, false); }
#undef L
  return (int)cudaGetLastError();
}

extern "C" int kb_write(float* o, int64_t n, int stream_hint, int grid, void* st) {
  cudaStream_t s = (cudaStream_t)st;
  if (stream_hint) k_write<true><<<grid, 256, 0, s>>>(o, n);
  else k_write<false><<<grid, 256, 0, s>>>(o, n);
  return (int)cudaGetLastError();
}
