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

// ---- TMA streaming read: per-warp ring of STAGES x TILE-byte bulk copies ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                   "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::
                   "r"(smem_u32(bar)), "r"(parity) : "memory");
}

template <int STAGES, int TILEB>
__global__ void k_tma_read(const float* __restrict__ g, int64_t n, uint32_t* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  unsigned char* ring = s_raw + (size_t)wib * STAGES * TILEB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_raw + (size_t)nwarps * STAGES * TILEB) + wib * STAGES;
  const int64_t ntiles = n * 4 / TILEB;
  const int64_t nw = (int64_t)gridDim.x * nwarps;
  int64_t t = (int64_t)blockIdx.x * nwarps + wib;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < STAGES; ++s)
      if (t + s * nw < ntiles) tma_load_1d(ring + s * TILEB, (const char*)g + (t + s * nw) * TILEB, TILEB, &bars[s]);
  }
  __syncwarp();
  uint32_t acc = 0, parity = 0;
  int stage = 0;
  for (; t < ntiles; t += nw) {
    mbar_wait(&bars[stage], (parity >> stage) & 1u);
    parity ^= 1u << stage;
    const float4* tile = reinterpret_cast<const float4*>(ring + stage * TILEB);
#pragma unroll 4
    for (int k = lane; k < TILEB / 16; k += 32) {
      const float4 x = tile[k];
      acc ^= __float_as_uint(x.x) ^ __float_as_uint(x.w);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0 && t + STAGES * nw < ntiles)
      tma_load_1d(ring + stage * TILEB, (const char*)g + (t + STAGES * nw) * TILEB, TILEB, &bars[stage]);
    stage = stage + 1 == STAGES ? 0 : stage + 1;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

extern "C" int kb_tma_read(const float* g, int64_t n, uint32_t* out, int stages, int tileb, int warps, int ctas_per_sm,
                           int sms, void* st) {
  const int smem = warps * stages * tileb + warps * stages * 8;
  cudaStream_t s = (cudaStream_t)st;
  const void* fn = nullptr;
#define C(S, T) if (stages == S && tileb == T) fn = (const void*)k_tma_read<S, T>;
  C(2, 4096) C(3, 4096) C(4, 4096) C(2, 8192) C(3, 8192) C(2, 16384) C(4, 2048) C(8, 2048)
#undef C
  if (!fn) return -1;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  void* args[] = {&g, &n, &out};
  cudaError_t e = cudaLaunchKernel(fn, dim3(sms * ctas_per_sm), dim3(warps * 32), args, smem, s);
  return (int)e;
}

// ---- cp.async (LDGSTS) per-warp ring streaming read ----
template <int STAGES>
__global__ void k_cpasync_read(const float* __restrict__ g, int64_t n, uint32_t* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  float4* ring = reinterpret_cast<float4*>(s_raw) + (size_t)wib * STAGES * 256;
  const int64_t ntiles = n / 1024;
  const int64_t nw = (int64_t)gridDim.x * nwarps;
  int64_t t = (int64_t)blockIdx.x * nwarps + wib;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  auto issue = [&](int64_t tt, int s) {
    if (tt < ntiles) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + s * 256 + k * 32 + lane);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(g4 + tt * 256 + k * 32 + lane) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < STAGES - 1; ++s) issue(t + s * nw, s);
  uint32_t acc = 0;
  int stage = 0;
  for (; t < ntiles; t += nw) {
    issue(t + (STAGES - 1) * nw, (stage + STAGES - 1) % STAGES);
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
    __syncwarp();
    const float4* tile = ring + stage * 256;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 x = tile[k * 32 + lane];
      acc ^= __float_as_uint(x.x) ^ __float_as_uint(x.w);
    }
    __syncwarp();
    stage = stage + 1 == STAGES ? 0 : stage + 1;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

extern "C" int kb_cpasync_read(const float* g, int64_t n, uint32_t* out, int stages, int warps, int ctas_per_sm,
                               int sms, void* st) {
  const int smem = warps * stages * 4096;
  const void* fn = nullptr;
  if (stages == 2) fn = (const void*)k_cpasync_read<2>;
  if (stages == 3) fn = (const void*)k_cpasync_read<3>;
  if (stages == 4) fn = (const void*)k_cpasync_read<4>;
  if (!fn) return -1;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  void* args[] = {&g, &n, &out};
  return (int)cudaLaunchKernel(fn, dim3(sms * ctas_per_sm), dim3(warps * 32), args, smem, (cudaStream_t)st);
}
