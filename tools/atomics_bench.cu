// atomics_bench.cu — random fp32 add throughput into a count-sketch table, three ways
// (evidence for the sketch-insert design; not part of libs2.so):
//   l2      red.global.add.f32 into a global table (L2-resident), what k_compress does
//   smem    atomicAdd on a CTA-private shared-memory table (privatised sketch; the table
//           must fit one CTA's shared memory — 3 MB does not, so this is the ceiling of a
//           privatised design, not a drop-in)
//   dsmem   atom.shared::cluster.add.f32 into a table distributed over the shared memory of
//           a thread-block cluster (16 CTAs x 192 KB = 3 MB: the ResNet-50 sketch fits one
//           cluster) — the only privatisation that holds a 3 MB table on chip
// Every thread draws `per_thread` pseudo-random (cell, +-1) pairs (xorshift32, multiply-high
// range reduction — cheap, so the rates reflect the memory system, not the index math).  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/atomics_bench.cu -o /tmp/atomics_bench
//   /tmp/atomics_bench
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

// cheap per-thread random stream (xorshift32) and multiply-high range reduction: a few integer
// ops per draw, so the rates below measure the memory system, not the index arithmetic
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

__global__ void k_l2(float* table, uint32_t cells, int per_thread, uint64_t seed) {
  uint32_t s = seed_of((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, seed);
  for (int k = 0; k < per_thread; ++k) {
    const uint32_t r = xs32(s);
    atomicAdd(table + cell_of(r, cells), (r & 1u) ? -1.f : 1.f);
  }
}

__global__ void k_smem(float* out, uint32_t cells, int per_thread, uint64_t seed) {
  extern __shared__ float t[];
  for (uint32_t i = threadIdx.x; i < cells; i += blockDim.x) t[i] = 0.f;
  __syncthreads();
  uint32_t s = seed_of((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, seed);
  for (int k = 0; k < per_thread; ++k) {
    const uint32_t r = xs32(s);
    atomicAdd(t + cell_of(r, cells), (r & 1u) ? -1.f : 1.f);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t[0];
}

__global__ void k_dsmem(float* out, uint32_t cells_per_cta, int per_thread, uint64_t seed) {
  extern __shared__ float t[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t nrank = cl.num_blocks();
  for (uint32_t i = threadIdx.x; i < cells_per_cta; i += blockDim.x) t[i] = 0.f;
  cl.sync();
  uint32_t s = seed_of((uint64_t)blockIdx.x * blockDim.x + threadIdx.x, seed);
  for (int k = 0; k < per_thread; ++k) {
    const uint32_t r = xs32(s);
    const uint32_t rank = cell_of(r, nrank), c = cell_of(r * 2654435761u, cells_per_cta);
    float* dst = cl.map_shared_rank(t, rank) + c;
    atomicAdd(dst, (r & 1u) ? -1.f : 1.f);  // remote (or local) shared-memory atomic over DSMEM
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = t[0];
}

// random 4-byte gathers from an L2-resident table, `ilp` independent loads in flight per thread —
// the access pattern of the decode's sketch queries (r gathers per union coordinate)
template <int ILP>
__global__ void k_gather(const float* __restrict__ table, uint32_t cells, int per_thread, uint64_t seed, float* out) {
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
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 512, per_thread = 64, reps = 20;
  printf("{\"sms\": %d, \"results\": [\n", sms);
  // L2 REDs: tables of 3 MB (ResNet-50 sketch) and 21 MB (BERT sketch)
  for (uint32_t cells : {786432u, 5242880u}) {
    const int grid = sms * 4;
    k_l2<<<grid, threads>>>(table, cells, per_thread, 1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_l2<<<grid, threads>>>(table, cells, per_thread, r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    const double n = (double)grid * threads * per_thread * reps;
    printf("  {\"kind\": \"l2_red\", \"table_MB\": %.2f, \"Gatomic_per_s\": %.1f},\n", cells * 4 / 1e6,
           n / (time_ms(e0, e1) * 1e-3) / 1e9);
  }
  // random gathers (the decode's query pattern): 3 MB and 21 MB tables, 1 / 3 / 6 loads in flight
  for (uint32_t cells : {786432u, 5242880u}) {
    for (int ilp : {1, 3, 6}) {
      const int grid = sms * 4;
      auto run = [&](uint64_t sd) {
        if (ilp == 1) k_gather<1><<<grid, threads>>>(table, cells, 48, sd, out);
        else if (ilp == 3) k_gather<3><<<grid, threads>>>(table, cells, 48, sd, out);
        else k_gather<6><<<grid, threads>>>(table, cells, 48, sd, out);
      };
      run(1);
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) run(r);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      const double n = (double)grid * threads * 48 * reps;
      printf("  {\"kind\": \"gather\", \"table_MB\": %.2f, \"ilp\": %d, \"Gload_per_s\": %.1f},\n", cells * 4 / 1e6, ilp,
             n / (time_ms(e0, e1) * 1e-3) / 1e9);
    }
  }
  // CTA-private shared-memory table (48 KB and 192 KB per CTA)
  for (uint32_t cells : {12288u, 49152u}) {
    const size_t smem = cells * 4;
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = sms * (smem <= 49152 ? 4 : 1);
    k_smem<<<grid, threads, smem>>>(out, cells, per_thread, 1);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_smem<<<grid, threads, smem>>>(out, cells, per_thread, r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    const double n = (double)grid * threads * per_thread * reps;
    printf("  {\"kind\": \"smem_private\", \"table_KB_per_cta\": %u, \"Gatomic_per_s\": %.1f, \"err\": \"%s\"},\n",
           cells * 4 / 1024, n / (time_ms(e0, e1) * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  // cluster-distributed table: 8 CTAs x 192 KB = 1.5 MB, 16 CTAs x 192 KB = 3 MB
  for (int csize : {8, 16}) {
    const uint32_t cpc = 49152u;
    const size_t smem = cpc * 4;
    cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (csize > 8) cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
    cudaError_t err = cudaLaunchKernelEx(&cfg, k_dsmem, out, cpc, per_thread, (uint64_t)1);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, k_dsmem, out, cpc, per_thread, (uint64_t)r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    const double n = (double)cfg.gridDim.x * threads * per_thread * reps;
    printf("  {\"kind\": \"dsmem_cluster\", \"cluster\": %d, \"table_MB\": %.2f, \"Gatomic_per_s\": %.1f, "
           "\"err\": \"%s\"}%s\n",
           csize, csize * cpc * 4 / 1e6, n / (time_ms(e0, e1) * 1e-3) / 1e9,
           cudaGetErrorString(err != cudaSuccess ? err : cudaGetLastError()), csize == 16 ? "" : ",");
  }
  printf("]}\n");
  return 0;
}
