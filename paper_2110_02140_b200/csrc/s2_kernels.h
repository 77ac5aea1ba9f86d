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

constexpr int kMaxWorld = 8;
// late_wait: the kernel may run while its stream predecessor (the previous reduce's decode) is
// still running — it neither reads what that kernel writes nor writes what it reads (s2_reduce's
// buffer rotation) — and waits for it only before exiting, so "this kernel complete" still implies
// "every earlier kernel of the stream complete"
cudaError_t launch_compress(const Plan& p, const float* g, uint32_t* bitmap, float* table,
                            unsigned long long* counters, int mode, cudaStream_t st, bool prezeroed = false,
                            bool late_wait = false);
// s2_reduce's decode also reports the step's health: `poison` (the exchange arena's sticky error
// word, or null) turns the whole output into NaN — a timed-out exchange never yields a silently
// wrong gradient — and `status` (device or mapped pinned host word, or null) receives
// S2_STATUS_NONFINITE if this rank's compress saw NaN/Inf (counters[S2_CNT_NONFINITE]) and
// S2_STATUS_EXCHANGE if the exchange timed out.
// `fence_zero`: fence the prologue's zeroing of the next table before dependents may launch (set
// when the compress that follows on the stream uses that very table: s2_reduce_many's two streams).
struct DecodeHealth {
  const uint32_t* poison;
  const unsigned long long* counters;
  uint32_t* status;
  int fence_zero;
};
cudaError_t launch_decode(const Plan& p, const uint32_t* bitmap, const float* table, int workers,
                          float* out, cudaStream_t st, float* zero_table = nullptr,
                          unsigned long long* zero_counters = nullptr, const DecodeHealth* health = nullptr);
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
  int64_t off_table[4];   // sketch tables and bitmaps rotate over 4 slots (s2_reduce), the rest over 2
  int64_t off_bitmap[4], off_union[2];
  int64_t off_flags_a, off_flags_b, off_epoch, off_error;
  int64_t off_tsum[2];  // one-shot: private summed tables
  int64_t cells;  // table cells, padded to a multiple of 4 * world
  int64_t words;  // bitmap words, padded to a multiple of 4 * world
  int world, rank, cur;  // cur: slot of union / tsum / inbox (step & 1)
  int tcur;              // table and bitmap slot (step & 3)
  int oneshot;                    // 1: one-shot exchange (single barrier), 0: two-shot
  int push;                       // 1: data pushed into the peers' inboxes before each flag (else pulled after)
  int64_t off_inbox[2];           // push: W slots (one-shot: whole table+bitmap; two-shot: one slice)
  unsigned long long timeout_ns;  // cross-rank barrier spin limit (then: sticky error, NaN output)
  unsigned long long* trace;      // optional: per-CTA globaltimer stamps [G][8] (S2_P2P_TRACE=1)
};
cudaError_t launch_p2p_aggregate(const P2PArgs& a, int grid, cudaStream_t st);

// Load the kernels a peer-memory plan will launch (cudaFuncGetAttributes forces CUDA's lazy module
// loading now).  A lazy load inside a launch can wait for running kernels; when one host thread
// drives several ranks (the single-GPU harness) that wait would hold back the launches the
// spinning exchange is waiting for.
cudaError_t preload_compress(const Plan& p);
cudaError_t preload_decode(const Plan& p);
cudaError_t preload_p2p(const P2PArgs& a);

}  // namespace s2
