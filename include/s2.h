/*
 * s2.h — C ABI of libs2.so, the B200 (sm_100a) sparse-sketch reduce of S2 Reducer.
 *
 * Drop-in boundary for the reference's sparse-sketch reducer path
 * (/root/reference/pkg/src/sketchgrad/sparse.py + sketch.py + core.py).  The
 * reference is pure Python/NumPy and has no FFI of its own; each entry point
 * below names the reference function it replaces, and INTEGRATION.md shows the
 * ctypes binding a maintainer adds on the reference side.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Device pointers are CUDA global memory;
 *     `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *   - Every call is stream-ordered and asynchronous unless documented
 *     otherwise; no implicit host synchronisation on the hot path.
 *   - Return value: S2_OK (0) or a status code; s2_last_error() gives the
 *     message of the last failure on the calling thread.  The Python layer
 *     maps S2_EINVAL/S2_EINCOMPAT/S2_ENONFINITE to ValueError with the
 *     reference's message text and the rest to RuntimeError.
 *   - Bitmaps are little-endian uint32 words: bit k of word w is block
 *     32*w + k.  Byte-for-byte this equals the reference wire form
 *     np.packbits(flags, bitorder="little") (sparse.py:60-61) zero-padded to
 *     a multiple of 4 bytes.
 *   - Sketch tables are float32 [rows][cols] row-major (the S2SK wire layout,
 *     sparse.py:129).  The reference accumulates in float64; see DESIGN.md
 *     for the fp32 tolerance contract.
 */
#ifndef S2_H_
#define S2_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S2_OK 0
#define S2_EINVAL 1      /* bad argument (reference: ValueError)                */
#define S2_ENONFINITE 2  /* NaN/Inf in a gradient (core.py:157-158)             */
#define S2_ECUDA 3       /* CUDA runtime failure                                */
#define S2_ENCCL 4       /* NCCL failure                                        */
#define S2_EINCOMPAT 5   /* incompatible payloads / ranks (sparse.py:179-187)  */

#define S2_MAX_ROWS 16

/* counters[] slots written by s2_compress (device, uint64) */
#define S2_CNT_NNZ 0       /* values inserted into the sketch                  */
#define S2_CNT_NONFINITE 1 /* != 0 if the gradient held NaN/Inf                */
#define S2_CNT_SELECTED 2  /* coordinates inside set blocks (alpha * dim)      */
#define S2_NUM_COUNTERS 4

/* status word written by every s2_reduce when set (s2_plan_set_status) */
#define S2_STATUS_NONFINITE 1u /* this rank's gradient held NaN/Inf (core.py:157-158)            */
#define S2_STATUS_EXCHANGE 2u  /* a cross-rank barrier timed out: the output was set to NaN      */

/* mask modes for s2_compress */
#define S2_MASK_NONZERO 0 /* build the bitmap: flag = block holds a non-zero */
#define S2_MASK_GIVEN 1   /* bitmap is an input (e.g. block_topk, sparse.py:70-80)         */

typedef struct s2_plan s2_plan;

const char* s2_last_error(void);
int s2_abi_version(void);

/* ---- L0 hashing, host side (core.py:27-106) -------------------------------- */
uint64_t s2_mix64(uint64_t x);                                /* core.py:27-38  */
uint64_t s2_derive_seed(const uint64_t* parts, int nparts);   /* core.py:44-54  */
int s2_row_seeds(uint64_t seed, int rows, uint64_t* out);     /* sketch.py:96-99 */
/* buckets/signs of `n` indices under one row seed (core.py:89-106); host reference
 * of the device hash, used by tests and the plan builder */
int s2_hash_host(uint64_t row_seed, const int64_t* idx, int64_t n, int64_t cols,
                 int64_t* buckets_out, int8_t* signs_out);

/* ---- plan: BlockPartition(dim, num_blocks) + CountSketchTable(rows, cols, seed)
 *      (core.py:172-211, sketch.py:86-100) ---------------------------------- */
int s2_plan_create(int64_t dim, int64_t num_blocks, int rows, int64_t cols, uint64_t seed,
                   int injective, s2_plan** out);
void s2_plan_destroy(s2_plan* plan);
int64_t s2_plan_bitmap_words(const s2_plan* plan);  /* ceil(num_blocks / 32) */
int64_t s2_plan_block_size(const s2_plan* plan);    /* ceil(dim / num_blocks) */

/* ---- device ops ------------------------------------------------------------- */

/* sparse_compress (sparse.py:151-171) fused with the mask producer.
 *   g        : float32[dim]
 *   bitmap   : uint32[words]; written when mask_mode == S2_MASK_NONZERO, read otherwise
 *   table    : float32[rows*cols]; zeroed here, then the non-zero entries of set
 *              blocks are inserted (sketch.py:102-112)
 *   counters : uint64[S2_NUM_COUNTERS] (device), zeroed here
 */
int s2_compress(const s2_plan* plan, const float* g, uint32_t* bitmap, float* table,
                int mask_mode, uint64_t* counters, void* stream);

/* sparse_decompress (sparse.py:199-214) + CountSketchTable.query (sketch.py:114-128):
 * out[i] = lower-median_j(s_j(i) T[j, h_j(i)]) / workers inside set blocks, else 0. */
int s2_decode(const s2_plan* plan, const uint32_t* bitmap, const float* table, int workers,
              float* out, void* stream);

/* CountSketchTable.insert (sketch.py:102-112) on explicit (index, value) pairs;
 * zero values are skipped; the table is NOT zeroed.  Indices must be in [0, dim). */
int s2_sketch_insert(const s2_plan* plan, const int64_t* idx, const float* vals, int64_t n,
                     float* table, void* stream);
/* CountSketchTable.query (sketch.py:114-128): lower median over rows, no ÷W */
int s2_sketch_query(const s2_plan* plan, const int64_t* idx, int64_t n, const float* table,
                    float* out, void* stream);

/* block_topk (sparse.py:70-80): flags of the k blocks of largest L2 norm (float64 norms,
 * ties to the lower block index) into `bitmap`; scratch >= s2_block_topk_scratch_bytes */
int64_t s2_block_topk_scratch_bytes(const s2_plan* plan);
int s2_block_topk(const s2_plan* plan, const float* g, int64_t k, uint32_t* bitmap, void* scratch,
                  void* stream);

/* BlockMask.union over `nmasks` stacked bitmaps (sparse.py:55-58) */
int s2_bitmap_or(int64_t words, const uint32_t* stacked, int nmasks, uint32_t* out, void* stream);

/* sketch.merge table sum over `ntables` stacked tables (sketch.py:213-216) */
int s2_table_sum(int64_t cells, const float* stacked, int ntables, float* out, void* stream);

/* sizes()[flags].sum() (sparse.py:51-53): selected coordinates of a bitmap, into
 * counters[S2_CNT_SELECTED] (device, accumulated; caller zeroes) */
int s2_selected_count(const s2_plan* plan, const uint32_t* bitmap, uint64_t* counters, void* stream);

/* BlockMask.selected_indices (sparse.py:44-49) when values == NULL, or the
 * compacted (idx, val) pairs sparse_compress inserts (sparse.py:164-168) when
 * g != NULL: ascending int64 indices (and float32 values), count into *count.
 * idx_out == NULL only counts (size the outputs, then call again).
 * scratch: device bytes >= s2_compact_scratch_bytes(plan). */
int64_t s2_compact_scratch_bytes(const s2_plan* plan);
int s2_compact(const s2_plan* plan, const uint32_t* bitmap, const float* g, int64_t* idx_out,
               float* val_out, int64_t* count, void* scratch, void* stream);

/* ---- distributed reduce over NVLink peer memory / NCCL (replaces the in-process
 *      sparse_merge list fold, sparse.py:174-196) -------------------------- */
int s2_nccl_unique_id(void* out /* 128 bytes */);
/* optional, before s2_comm_init*: exchange-kernel CTAs per rank (0 = default: one per SM, or
 * one per two SMs for exchanges <= 8 MB) and the cross-rank barrier timeout in seconds
 * (<= 0: S2_P2P_TIMEOUT_S or 300 s).  After a timeout the plan's outputs are NaN and
 * S2_STATUS_EXCHANGE is reported — never a silently incomplete average. */
int s2_comm_set_options(s2_plan* plan, int exchange_grid, double timeout_s);
int s2_comm_init(s2_plan* plan, int world, int rank, const void* unique_id);
/* comm modes: IPC = the plan allocates its exchange arena, CUDA-IPC handles travel through
 * one NCCL all-gather (default); NCCL = NCCL all-reduce + all-gather + OR kernel;
 * EXTERNAL = no NCCL at all: the caller provides every rank's arena through s2_comm_attach
 * (torch symmetric memory, or W plans driven from one process — the single-GPU multi-rank
 * harness) and checks s2_plan_digest across ranks itself.  unique_id may be NULL. */
#define S2_COMM_IPC 0
#define S2_COMM_NCCL 1
#define S2_COMM_EXTERNAL 2
int s2_comm_init_mode(s2_plan* plan, int world, int rank, const void* unique_id, int mode);
/* bytes of the per-rank exchange arena for `world` ranks (same on every rank) */
int64_t s2_p2p_arena_bytes(s2_plan* plan, int world);
/* EXTERNAL mode: bases[q] = rank q's arena (s2_p2p_arena_bytes bytes, 256-B aligned) as
 * addressable from this process/device; zeroes this rank's arena (stream 0).  Every rank must
 * attach before any rank reduces. */
int s2_comm_attach(s2_plan* plan, const uint64_t* bases, int world);
/* compat_key digest of (dim, num_blocks, rows, cols, seed, injective) (sparse.py:105-109) */
uint64_t s2_plan_digest(const s2_plan* plan);
/* one-time agreement on the digest across ranks over NCCL (IPC / NCCL modes; EXTERNAL: no-op,
 * the caller compares s2_plan_digest) — the distributed compat_key check (sparse.py:179-187) */
int s2_comm_check(s2_plan* plan, void* stream);
/* sketch all-reduce (sum) in place + bitmap all-gather fused with OR into union (NCCL) */
int s2_aggregate(s2_plan* plan, float* table, const uint32_t* bitmap, uint32_t* union_out,
                 void* stream);
/* the whole reduce: compress -> aggregate -> decode (÷ world) using plan-owned
 * scratch; out = float32[dim] averaged gradient.  counters may be NULL (then the
 * plan's own are used, see s2_last_counters).  Plan-owned buffers rotate with period 4
 * (call i uses table / counters slot i % 4 and bitmap slot i % 2 (i % 4 with an exchange
 * arena); its decode zeroes slot (i+2) % 4), so a CUDA graph must capture a multiple of 4 calls.  The compress of call i+1
 * shares no buffer with the decode of call i and overlaps it through programmatic dependent
 * launch, unless g aliases the previous call's out (then it waits; S2_OVERLAP=0 disables). */
int s2_reduce(s2_plan* plan, const float* g, float* out, uint64_t* counters, void* stream);
/* n reduces (gs[k] -> outs[k]), same result as n s2_reduce calls.  With world > 1 they are
 * pipelined: the compress of step k+1 runs while step k's exchange (NVLink, few SMs) is in
 * flight, and step k's decode follows it.  Falls back to n plain calls when an input aliases an
 * earlier output of the batch. */
int s2_reduce_many(s2_plan* plan, const float* const* gs, float* const* outs, int n, void* stream);
/* every later s2_reduce's decode ORs its S2_STATUS_* bits (nothing when healthy) into *status
 * (device memory or mapped pinned host memory; NULL disables; the caller zeroes it) — lets a
 * caller check earlier steps without synchronising */
int s2_plan_set_status(s2_plan* plan, uint32_t* status);
/* device pointer to the counters of the most recent s2_reduce(counters = NULL) */
const uint64_t* s2_last_counters(const s2_plan* plan);
/* optional: 4 caller-created cudaEvent_t that s2_reduce records before compress,
 * after compress, after aggregate and after decode (n = 0 disables) */
int s2_plan_set_timing_events(s2_plan* plan, void* const* events, int n);
/* != 0 if a peer-memory barrier timed out (a rank died or diverged); synchronises */
int s2_p2p_error(const s2_plan* plan);
/* debugging: globaltimer stamps [G][8] of the last peer-memory exchange (S2_P2P_TRACE=1) */
int s2_p2p_trace(const s2_plan* plan, uint64_t* host, int64_t n);
/* copy those counters to host (synchronises `stream`) */
int s2_read_counters(const s2_plan* plan, uint64_t* host_out, void* stream);
int s2_plan_world(const s2_plan* plan);

#ifdef __cplusplus
}
#endif
#endif /* S2_H_ */
