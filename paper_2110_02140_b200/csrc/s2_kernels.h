// s2_kernels.h — internal launcher interface between the C ABI (s2_capi.cu) and the kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "s2_common.cuh"

namespace s2 {

// BlockPartition(dim, num_blocks) + CountSketchTable hash parameters (core.py:172-211, sketch.py:86-100)
struct Plan {
  int64_t dim;
  int64_t num_blocks;
  int64_t block_size;  // ceil(dim / num_blocks)
  int64_t words;       // ceil(num_blocks / 32)
  uint64_t seed;
  int injective;
  HashParams hp;
};

constexpr int kMaxWorldSig = 8;
struct DoneSignal {  // see signal_done (s2_kernels.cu); done == nullptr: no signal
  unsigned int* done;
  unsigned int* epoch;
  uint32_t* peer_flags[kMaxWorldSig];
  int world, rank;
};
constexpr int kMaxWorld = 8;
// element bitmap words also stored straight into each peer's inbox slot for this rank
// (remote NVLink stores during the compress); n = 0: none
struct BitmapPush {
  uint32_t* dst[kMaxWorld];
  int n;
  int fence;  // end-of-kernel system fence: 1 every thread, 2 one lane per warp (after __syncwarp)
};
cudaError_t launch_compress(const Plan& p, const float* g, uint32_t* bitmap, float* table,
                            unsigned long long* counters, int mode, cudaStream_t st, bool prezeroed = false,
                            void* list = nullptr,  // list: dim x 8 B scratch -> split K1 + K2 path
                            const DoneSignal* signal = nullptr, const BitmapPush* push = nullptr);
// bitmaps of every rank (peer-mapped) whose OR the decode reads directly; n = 0: use `bitmap`
struct PeerMaps {
  const uint32_t* p[kMaxWorld];
  int n;
};
cudaError_t launch_decode(const Plan& p, const uint32_t* bitmap, const float* table, int workers,
                          float* out, cudaStream_t st, float* zero_table = nullptr,
                          unsigned long long* zero_counters = nullptr, const PeerMaps* peers = nullptr);
cudaError_t launch_bitmap_or(int64_t words, const uint32_t* stacked, int nmasks, uint32_t* out,
                             cudaStream_t st);
cudaError_t launch_table_sum(int64_t cells, const float* stacked, int ntables, float* out,
                             cudaStream_t st);
cudaError_t launch_selected_count(const Plan& p, const uint32_t* bitmap,
                                  unsigned long long* counters, cudaStream_t st);
int64_t compact_scratch_bytes(const Plan& p);
cudaError_t launch_exclusive_scan(int64_t* a, int64_t n, int64_t* total, cudaStream_t st);
// block_topk (sparse.py:70-80) into `bitmap`; scratch >= topk_scratch_bytes(p)
int64_t topk_scratch_bytes(const Plan& p);
cudaError_t launch_block_topk(const Plan& p, const float* g, int64_t k, uint32_t* bitmap, void* scratch,
                              cudaStream_t st);
cudaError_t launch_compact(const Plan& p, const uint32_t* bitmap, const float* g, int64_t* idx_out,
                           float* val_out, int64_t* count, void* scratch, cudaStream_t st);

// CountSketchTable.insert (vals != NULL) or .query (vals == NULL -> out) on explicit index lists
cudaError_t launch_pairs(const Plan& p, const int64_t* idx, const float* vals, int64_t n, const float* table,
                         float* out, cudaStream_t st);

// NVLink peer-memory exchange (s2_p2p.cu)
struct P2PArgs {
  char* base[kMaxWorld];  // arena base of every rank (self included), mapped in this process
  int64_t off_table[2], off_bitmap[2], off_union[2];
  int64_t off_flags_a, off_flags_b, off_epoch, off_error;
  int64_t off_tsum[2];  // one-shot: private summed tables
  int64_t off_lsync;    // fused kernel: local arrival counter (u64) + release word (u32)
  int64_t cells;  // table cells, padded to a multiple of 4 * world
  int64_t words;  // bitmap words, padded to a multiple of 4 * world
  int world, rank, cur;
  int oneshot;                // 1: one-shot exchange (single barrier), 0: two-shot
  int table_only;             // 1: bitmaps are OR-ed by the decode from peer memory (no bitmap exchange)
  char* mc;                   // NVLS multicast address of the arena (nullptr: none)
  int nvls;                   // 1: reduce in the NVSwitch (multimem.ld_reduce / multimem.st)
  int hier;                   // 1: hierarchical barriers (CTA 0 <-> peers, local release)
  int csig;                   // 1: barrier 1 = poll of the compress-done flags (signal_done)
  int pipe;                   // 1: pipelined two-shot (per-peer waits, k_p2p_pipe)
  int64_t off_flags_c, off_cdone, off_cepoch;
  int64_t off_inbox[2];       // bitmap push: W slots of `words` words (slot q = rank q's bitmap), or -1
  int push;                   // 1: compress pushes its bitmap into the peers' inboxes (table-only exchange)
  unsigned long long* trace;  // optional: per-CTA globaltimer stamps [G][8] (S2_P2P_TRACE=1)
};
cudaError_t launch_p2p_aggregate(const P2PArgs& a, int grid, cudaStream_t st);
struct DecodeCtx;
cudaError_t xdecode_grid(const HashParams& hp, int world, int oneshot, int* grid);
// fused exchange + decode (W > 1); cudaErrorNotSupported for (rows, world) without an instantiation
cudaError_t launch_xdecode(const P2PArgs& a, const DecodeCtx& dc, const HashParams& hp, int grid, float* zt,
                           int64_t zt_n4, unsigned long long* zc, cudaStream_t st);

}  // namespace s2
