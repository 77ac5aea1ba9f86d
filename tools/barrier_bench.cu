// barrier_bench.cu — latency of cross-GPU flag barriers over NVLink (experiment, 2+ ranks).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC tools/barrier_bench.cu -o tools/libbarrier.so
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

struct BArgs {
  uint32_t* flags[8];  // every rank's flag array [W][G], mapped here
  int world, rank, iters, mode;
  unsigned long long* out;  // [G] ns per barrier
};

__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_barrier(BArgs a) {
  const int G = gridDim.x, b = blockIdx.x;
  __shared__ uint64_t t0;
  if (threadIdx.x == 0) t0 = gt();
  __syncthreads();
  for (int it = 1; it <= a.iters; ++it) {
    __syncthreads();
    if (threadIdx.x < a.world) {
      const int q = threadIdx.x;
      uint32_t* remote = a.flags[q] + a.rank * G + b;
      uint32_t* mine = a.flags[a.rank] + q * G + b;
      if (a.mode == 0) {
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(remote), "r"((uint32_t)it) : "memory");
      } else if (a.mode == 1) {
        __threadfence_system();
        asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(remote), "r"((uint32_t)it) : "memory");
      } else if (a.mode == 2) {
        __threadfence();
        asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(remote), "r"((uint32_t)it) : "memory");
      } else {
        asm volatile("red.release.sys.global.max.u32 [%0], %1;" ::"l"(remote), "r"((uint32_t)it) : "memory");
      }
      uint32_t v;
      const uint64_t tstart = gt();
      int spins = 0;
      do {
        if (++spins % 1024 == 0 && gt() - tstart > 2000000000ull) break;  // 2 s bail-out: never hang the GPU
        if (a.mode == 2)
          asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
        else
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      } while ((int32_t)(v - (uint32_t)it) < 0);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) a.out[b] = (gt() - t0) / a.iters;
}

extern "C" void* bb_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  cudaMemset(p, 0, bytes);
  cudaDeviceSynchronize();
  return p;
}
extern "C" int bb_ipc_handle(void* ptr, void* out64) {
  return (int)cudaIpcGetMemHandle((cudaIpcMemHandle_t*)out64, ptr);
}
extern "C" int bb_ipc_open(const void* h64, void** out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, h64, sizeof h);
  return (int)cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess);
}
extern "C" int bb_run(void* const* flags, int world, int rank, int iters, int mode, int grid, int threads,
                      unsigned long long* out) {
  BArgs a{};
  for (int q = 0; q < world; ++q) a.flags[q] = (uint32_t*)flags[q];
  a.world = world;
  a.rank = rank;
  a.iters = iters;
  a.mode = mode;
  a.out = out;
  void* args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_barrier, dim3(grid), dim3(threads), args, 0, 0);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaDeviceSynchronize();
}
