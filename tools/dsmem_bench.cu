// dsmem_bench.cu — random 4-byte LOAD throughput from a table held three ways (evidence for the
// decode design; not part of libs2.so):
//   l2      __ldg gathers from a global (L2-resident) table — what k_decode does
//   dsmem   ld.shared::cluster gathers from a table distributed over a thread-block cluster's
//           shared memory (cluster x 192 KB: 16 x 192 KB = 3 MB holds the ResNet-50 sketch)
//   smem    CTA-local shared-memory gathers (ceiling)
// Each thread draws per_thread random cells (xorshift32) with ILP loads in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/dsmem_bench.cu -o /tmp/dsmem_bench
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t xs32(uint32_t& s) {
  s ^= s << 13;
  s ^= s >> 17;
  s ^= s << 5;
  return s;
}
__device__ __forceinline__ uint32_t cell_of(uint32_t r, uint32_t cells) { return __umulhi(r, cells); }
__device__ __forceinline__ uint32_t seed_of(uint64_t tid, uint64_t seed) {
  return (uint32_t)((tid + 1) * 0x9E3779B97F4A7C15ull >> 32) ^ (uint32_t)seed | 1u;
}

template <int ILP>
__global__ void k_l2(const float* __restrict__ table, uint32_t cells, int per_thread, uint64_t seed, float* out) {
  uint32_t s = seed_of((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, seed);
  float acc = 0.f;
  for (int k = 0; k < per_thread; k += ILP) {
    float v[ILP];
#pragma unroll
    for (int u = 0; u < ILP; ++u) v[u] = __ldg(table + cell_of(xs32(s), cells));
#pragma unroll
    for (int u = 0; u < ILP; ++u) acc += v[u];
  }
  if (acc == 12345.f) out[0] = acc;
}

__device__ __forceinline__ float ld_dsmem(uint32_t cta_addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(cta_addr));
  return v;
}

// table distributed over the cluster: cell c lives in rank c / cpc at offset c % cpc
template <int ILP>
__global__ void k_dsmem(uint32_t cpc, int per_thread, uint64_t seed, float* out) {
  extern __shared__ float t[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t nrank = cl.num_blocks();
  for (uint32_t i = threadIdx.x; i < cpc; i += blockDim.x) t[i] = (float)i;
  cl.sync();
  const uint32_t local = (uint32_t)__cvta_generic_to_shared(t);
  uint32_t base[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(local), "r"(r < (int)nrank ? r : 0));
    base[r] = a;
  }
  uint32_t s = seed_of((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, seed);
  float acc = 0.f;
  const uint32_t cells = cpc * nrank;
  for (int k = 0; k < per_thread; k += ILP) {
    float v[ILP];
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
      const uint32_t c = cell_of(xs32(s), cells);
      const uint32_t rk = c / cpc, off = c - rk * cpc;
      uint32_t b = base[0];
#pragma unroll
      for (int r = 1; r < 16; ++r) b = rk == (uint32_t)r ? base[r] : b;
      v[u] = ld_dsmem(b + 4 * off);
    }
#pragma unroll
    for (int u = 0; u < ILP; ++u) acc += v[u];
  }
  cl.sync();
  if (acc == 12345.f) out[0] = acc;
}

template <int ILP>
__global__ void k_smem(uint32_t cells, int per_thread, uint64_t seed, float* out) {
  extern __shared__ float t[];
  for (uint32_t i = threadIdx.x; i < cells; i += blockDim.x) t[i] = (float)i;
  __syncthreads();
  uint32_t s = seed_of((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, seed);
  float acc = 0.f;
  for (int k = 0; k < per_thread; k += ILP) {
    float v[ILP];
#pragma unroll
    for (int u = 0; u < ILP; ++u) v[u] = t[cell_of(xs32(s), cells)];
#pragma unroll
    for (int u = 0; u < ILP; ++u) acc += v[u];
  }
  if (acc == 12345.f) out[0] = acc;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *table, *out;
  cudaMalloc(&table, 64u << 20);
  cudaMemset(table, 0, 64u << 20);
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 10, per_thread = 512;
  printf("{\"sms\": %d, \"results\": [\n", sms);
  {
    const int threads = 512, grid = sms * 4;
    k_l2<4><<<grid, threads>>>(table, 786432u, per_thread, 1, out);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_l2<4><<<grid, threads>>>(table, 786432u, per_thread, r, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    const double n = (double)grid * threads * per_thread * reps;
    printf("  {\"kind\": \"l2_gather\", \"table_MB\": 3.15, \"Gload_per_s\": %.1f, \"err\": \"%s\"},\n",
           n / (time_ms(e0, e1) * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  for (int csize : {1, 2, 4, 8, 16}) {
    for (int threads : {512, 1024}) {
      const uint32_t cpc = 49152u;  // 192 KB per CTA
      const size_t smem = cpc * 4;
      auto kern = k_dsmem<4>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (csize > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((sms / csize) * csize);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csize;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t err = cudaLaunchKernelEx(&cfg, kern, cpc, per_thread, (uint64_t)1, out);
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, kern, cpc, per_thread, (uint64_t)r, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      const double n = (double)cfg.gridDim.x * threads * per_thread * reps;
      printf("  {\"kind\": \"dsmem_gather\", \"cluster\": %d, \"threads\": %d, \"table_MB\": %.2f, \"Gload_per_s\": %.1f, "
             "\"err\": \"%s\"},\n",
             csize, threads, csize * cpc * 4 / 1e6, n / (time_ms(e0, e1) * 1e-3) / 1e9,
             cudaGetErrorString(err != cudaSuccess ? err : cudaGetLastError()));
    }
  }
  {
    const uint32_t cells = 49152u;
    const size_t smem = cells * 4;
    cudaFuncSetAttribute(k_smem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int threads = 1024, grid = sms;
    k_smem<4><<<grid, threads, smem>>>(cells, per_thread, 1, out);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_smem<4><<<grid, threads, smem>>>(cells, per_thread, r, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    const double n = (double)grid * threads * per_thread * reps;
    printf("  {\"kind\": \"smem_gather\", \"table_KB_per_cta\": 192, \"Gload_per_s\": %.1f, \"err\": \"%s\"}\n",
           n / (time_ms(e0, e1) * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  printf("]}\n");
  return 0;
}
