// nvlink_bench.cu — all-to-all push bandwidth over NVLink between the GPUs of one box, the
// traffic shape of the exchange's push phases (s2_p2p.cu): every GPU stores `bytes` into each
// of its W-1 peers at once.  Single process, peer access; evidence for the exchange design
// (DESIGN.md §7), not part of libs2.so.
//   mode 0  st.global.v4 (16 B per thread), what k_p2p_push_twoshot does
//   mode 1  st.global.v8 (32 B per thread, sm_100 256-bit stores)
//   mode 2  TMA bulk store: a CTA stages 8 KB in shared memory, then one cp.async.bulk
//           shared::cta -> peer global per peer
//   mode 4  local stores only (launch + fence overhead baseline)
//   mode 3  pull: ld.global.v4 from each peer into local memory (the one-shot's pattern)
// Each timed kernel ends with every CTA's __threadfence_system, so a launch's time includes
// the remote writes becoming visible.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/nvlink_bench.cu -o /tmp/nvlink_bench
//   /tmp/nvlink_bench [W]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

struct Peers {
  char* p[8];
};

__global__ void k_push(Peers dst, const char* __restrict__ src, int64_t bytes, int w, int me, int mode) {
  const int64_t per = (bytes / gridDim.x + 8191) & ~(int64_t)8191;
  const int64_t lo = (int64_t)blockIdx.x * per;
  const int64_t hi = lo + per < bytes ? lo + per : bytes;
  if (mode == 0) {
    for (int64_t i = lo + threadIdx.x * 16; i < hi; i += blockDim.x * 16) {
      const uint4 v = *reinterpret_cast<const uint4*>(src + i);
      for (int q = 0; q < w; ++q)
        if (q != me) *reinterpret_cast<uint4*>(dst.p[q] + me * bytes + i) = v;
    }
  } else if (mode == 1) {
    for (int64_t i = lo + threadIdx.x * 32; i < hi; i += blockDim.x * 32) {
      uint32_t a[8];
      asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7])
                   : "l"(src + i));
      for (int q = 0; q < w; ++q)
        if (q != me)
          asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst.p[q] + me * bytes + i), "r"(a[0]),
                       "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7])
                       : "memory");
    }
  } else if (mode == 2) {
    __shared__ __align__(128) char stage[2][8192];
    int buf = 0;
    for (int64_t c = lo; c < hi; c += 8192, buf ^= 1) {
      const int n = (int)(hi - c < 8192 ? hi - c : 8192);
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncthreads();
      for (int i = threadIdx.x * 16; i < n; i += blockDim.x * 16)
        *reinterpret_cast<uint4*>(stage[buf] + i) = *reinterpret_cast<const uint4*>(src + c + i);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int q = 0; q < w; ++q)
          if (q != me)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst.p[q] + me * bytes + c),
                         "r"((uint32_t)__cvta_generic_to_shared(stage[buf])), "r"(n)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (mode == 4) {  // local stores only: launch + fence overhead baseline
    for (int64_t i = lo + threadIdx.x * 16; i < hi; i += blockDim.x * 16)
      *reinterpret_cast<uint4*>(dst.p[me] + me * bytes + i) = *reinterpret_cast<const uint4*>(src + i);
  } else {
    // pull: read my slot from every peer (they hold `bytes` for me at offset me*bytes)
    for (int64_t i = lo + threadIdx.x * 16; i < hi; i += blockDim.x * 16) {
      uint4 acc = make_uint4(0, 0, 0, 0);
      for (int q = 0; q < w; ++q) {
        if (q == me) continue;
        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(dst.p[q] + me * bytes + i));
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
      }
      *reinterpret_cast<uint4*>(dst.p[me] + me * bytes + i) = acc;
    }
  }
  __syncthreads();
  __threadfence_system();
}

int main(int argc, char** argv) {
  int w = argc > 1 ? atoi(argv[1]) : 4;
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  if (w > ndev) w = ndev;
  if (w < 2) {
    printf("{\"error\": \"needs >= 2 GPUs\"}\n");
    return 0;
  }
  for (int a = 0; a < w; ++a) {
    cudaSetDevice(a);
    for (int b = 0; b < w; ++b)
      if (a != b) cudaDeviceEnablePeerAccess(b, 0);
  }
  const int64_t maxb = 64ll << 20;
  Peers pr{};
  char* src[8];
  cudaStream_t st[8];
  cudaEvent_t e0[8], e1[8];
  for (int a = 0; a < w; ++a) {
    cudaSetDevice(a);
    cudaMalloc(&pr.p[a], maxb * w);
    cudaMalloc(&src[a], maxb);
    cudaMemset(src[a], 1, maxb);
    cudaStreamCreateWithFlags(&st[a], cudaStreamNonBlocking);
    cudaEventCreate(&e0[a]);
    cudaEventCreate(&e1[a]);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"w\": %d, \"results\": [\n", w);
  bool first = true;
  for (int64_t bytes : {(int64_t)(1 << 20), (int64_t)(1600 << 10), (int64_t)(3 << 20), (int64_t)(6 << 20), (int64_t)(32 << 20)}) {
    for (int mode = 0; mode < 5; ++mode) {
      for (int grid : {sms / 2, sms}) {
        for (int threads : {1024}) {
          const int reps = 20;
          for (int a = 0; a < w; ++a) {  // warm-up
            cudaSetDevice(a);
            k_push<<<grid, threads, 0, st[a]>>>(pr, src[a], bytes, w, a, mode);
          }
          for (int a = 0; a < w; ++a) {
            cudaSetDevice(a);
            cudaStreamSynchronize(st[a]);
          }
          for (int a = 0; a < w; ++a) {
            cudaSetDevice(a);
            cudaEventRecord(e0[a], st[a]);
          }
          for (int r = 0; r < reps; ++r)
            for (int a = 0; a < w; ++a) {
              cudaSetDevice(a);
              k_push<<<grid, threads, 0, st[a]>>>(pr, src[a], bytes, w, a, mode);
            }
          float worst = 0.f;
          for (int a = 0; a < w; ++a) {
            cudaSetDevice(a);
            cudaEventRecord(e1[a], st[a]);
            cudaEventSynchronize(e1[a]);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0[a], e1[a]);
            if (ms > worst) worst = ms;
          }
          const double us = worst * 1e3 / reps;
          const double out_bytes = (double)bytes * (w - 1);
          printf("%s  {\"bytes_per_peer\": %lld, \"mode\": %d, \"grid\": %d, \"threads\": %d, \"us\": %.2f, "
                 "\"egress_GBps\": %.1f, \"err\": \"%s\"}",
                 first ? "" : ",\n", (long long)bytes, mode, grid, threads, us, out_bytes / (us * 1e3),
                 cudaGetErrorString(cudaGetLastError()));
          first = false;
        }
      }
    }
  }
  printf("\n]}\n");
  return 0;
}
