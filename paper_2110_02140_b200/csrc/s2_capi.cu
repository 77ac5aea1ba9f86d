// s2_capi.cu — the C ABI of libs2.so (include/s2.h): plans, host hashing,
// stream-ordered device ops and the NCCL/NVLink distributed reduce.
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost a few ns unless a profiler is attached

#include "s2.h"
#include "s2_common.cuh"
#include "s2_kernels.h"
#include "s2_decode.cuh"

using s2::HashParams;
using s2::Plan;

struct s2_plan {
  Plan p;
  // distributed state
  int world = 1;
  int rank = 0;
  ncclComm_t comm = nullptr;
  // plan-owned scratch for s2_reduce / s2_aggregate.  Reduce i uses sketch table and counters
  // slot i % 4 and bitmap slot i % 2 (i % 4 in the exchange arena); its decode zeroes table /
  // counters slot (i + 2) % 4 in its prologue (fenced before it lets dependents launch), so the
  // hot path has no memset launches and the compress of reduce i+1 (or i+2 in s2_reduce_many's
  // two-stream schedule) may overlap the decode of reduce i (late_wait).
  static constexpr int kTableSlots = 4;
  float* tables[kTableSlots] = {};
  unsigned long long* counters[kTableSlots] = {};
  uint64_t step = 0;
  uint32_t* bitmaps[2] = {nullptr, nullptr};
  const float* prev_out = nullptr;  // the previous reduce's output (alias check for late_wait)
  int overlap = -1;                 // S2_OVERLAP (default 1)
  uint32_t* unionmap = nullptr;
  uint32_t* gather = nullptr;  // world * words (all-gather landing buffer)
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // optional phase timing events
  uint32_t* status = nullptr;  // S2_STATUS_* of every reduce (s2_plan_set_status)
  // NVLink peer-memory exchange (world > 1, default): one arena per rank, mapped by every rank
  bool p2p = false;
  char* arena = nullptr;
  char* peer[s2::kMaxWorld] = {};
  s2::P2PArgs pa{};
  int p2p_grid = 0;
  int comm_mode = 0;         // S2_COMM_IPC | S2_COMM_NCCL | S2_COMM_EXTERNAL
  bool arena_owned = false;  // cudaMalloc'd here (IPC) vs attached by the caller (EXTERNAL)
  int opt_grid = 0;          // s2_comm_set_options
  double opt_timeout_s = 0;
  // s2_reduce_many's exchange stream (high priority) and its fork/join events
  cudaStream_t xstream = nullptr;
  static constexpr int kPipeEvents = 4;
  cudaEvent_t ev_c[kPipeEvents] = {};  // compress k done (main stream)
  cudaEvent_t ev_x[kPipeEvents] = {};  // exchange k done (exchange stream)
};

namespace {

thread_local std::string g_err;

// host-side NVTX range over an enqueue (nsys / ncu --nvtx show where each stage was issued)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(S2_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define S2_CUDA(call, what)                      \
  do {                                           \
    cudaError_t e_ = (call);                     \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

#define S2_NCCL(call, what)                                                         \
  do {                                                                              \
    ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess) return fail(S2_ENCCL, "%s: %s", what, ncclGetErrorString(r_)); \
  } while (0)

uint64_t derive(const uint64_t* parts, int n) {  // core.py:44-54
  uint64_t acc = s2::kDeriveInit;
  for (int k = 0; k < n; ++k) acc = s2::mix64(acc + parts[k] * s2::kGolden);
  return acc;
}

int build_hash(uint64_t seed, int rows, int64_t cols, int injective, HashParams* hp) {
  if (rows < 1 || cols < 1)
    return fail(S2_EINVAL, "rows and cols must be >= 1, got %dx%lld", rows, (long long)cols);
  if (rows > S2_MAX_ROWS) return fail(S2_EINVAL, "rows must be <= %d, got %d", S2_MAX_ROWS, rows);
  if (cols >= (int64_t)1 << 32) return fail(S2_EINVAL, "cols must be < 2^32, got %lld", (long long)cols);
  memset(hp, 0, sizeof *hp);
  hp->rows = rows;
  hp->cols = (uint32_t)cols;
  for (int j = 0; j < rows; ++j) {
    const uint64_t parts[2] = {seed, (uint64_t)j};
    hp->seed[j] = derive(parts, 2);  // sketch.py:96-99
  }
  if (injective) {
    hp->mode = s2::kInjective;
  } else if ((cols & (cols - 1)) == 0) {
    hp->mode = s2::kPow2;
  } else {
    int l = 0;
    while (((int64_t)1 << l) < cols) ++l;  // 2^(l-1) < cols < 2^l
    const unsigned __int128 num = (unsigned __int128)1 << (63 + l);
    hp->magic = (uint64_t)(num / (uint64_t)cols) + 1u;  // ceil: cols never divides 2^(63+l)
    hp->shift = (uint32_t)(l - 1);
    hp->mode = s2::kMagic;
  }
  return S2_OK;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

const char* s2_last_error(void) { return g_err.c_str(); }
int s2_abi_version(void) { return 2; }

uint64_t s2_mix64(uint64_t x) { return s2::mix64(x); }

uint64_t s2_derive_seed(const uint64_t* parts, int nparts) { return derive(parts, nparts); }

int s2_row_seeds(uint64_t seed, int rows, uint64_t* out) {
  if (rows < 1 || rows > S2_MAX_ROWS) return fail(S2_EINVAL, "rows must be in [1, %d]", S2_MAX_ROWS);
  for (int j = 0; j < rows; ++j) {
    const uint64_t parts[2] = {seed, (uint64_t)j};
    out[j] = derive(parts, 2);
  }
  return S2_OK;
}

int s2_hash_host(uint64_t row_seed, const int64_t* idx, int64_t n, int64_t cols,
                 int64_t* buckets_out, int8_t* signs_out) {
  HashParams hp;
  int rc = build_hash(0, 1, cols, 0, &hp);
  if (rc) return rc;
  for (int64_t k = 0; k < n; ++k) {
    const uint64_t w = s2::mix64(row_seed + s2::index_term((uint64_t)idx[k]));
    if (buckets_out) buckets_out[k] = s2::bucket_of(w, hp);
    if (signs_out) signs_out[k] = (w >> 63) ? -1 : 1;
  }
  return S2_OK;
}

int s2_plan_create(int64_t dim, int64_t num_blocks, int rows, int64_t cols, uint64_t seed,
                   int injective, s2_plan** out) {
  if (out == nullptr) return fail(S2_EINVAL, "out is NULL");
  *out = nullptr;
  if (dim < 1) return fail(S2_EINVAL, "dim must be >= 1, got %lld", (long long)dim);
  if (num_blocks < 1 || num_blocks > dim)
    return fail(S2_EINVAL, "num_blocks must be in [1, dim=%lld], got %lld", (long long)dim,
                (long long)num_blocks);
  if (dim >= ((int64_t)1 << 32) - 1)
    return fail(S2_EINVAL, "dim must be < 2^32 - 1 on the GPU path, got %lld", (long long)dim);
  HashParams hp;
  int rc = build_hash(seed, rows, cols, injective, &hp);
  if (rc) return rc;
  // injective with cols < dim is legal: HashMapping(injective) raises only when an index it
  // maps is >= buckets (core.py:131-135).  The Python layer raises that ValueError before any
  // kernel runs; the kernels skip (insert) or read 0 for (query) such indices, so a direct
  // C-ABI caller cannot write or read past the table.
  s2_plan* p = new s2_plan();
  p->p.dim = dim;
  p->p.num_blocks = num_blocks;
  p->p.block_size = (dim + num_blocks - 1) / num_blocks;
  p->p.words = (num_blocks + 31) / 32;
  p->p.seed = seed;
  p->p.injective = injective;
  p->p.hp = hp;
  *out = p;
  return S2_OK;
}

static void free_scratch(s2_plan* p) {
  for (int k = 0; k < s2_plan::kTableSlots; ++k) {
    if (!p->p2p) cudaFree(p->tables[k]);
    cudaFree(p->counters[k]);
    p->tables[k] = nullptr;
    p->counters[k] = nullptr;
  }
  for (int k = 0; k < 2; ++k) {
    cudaFree(p->bitmaps[k]);
    p->bitmaps[k] = nullptr;
  }
  cudaFree(p->unionmap);
  cudaFree(p->gather);
  p->unionmap = p->gather = nullptr;
}

static void free_p2p(s2_plan* p) {
  for (int q = 0; q < s2::kMaxWorld; ++q)
    if (p->arena_owned && p->peer[q] && p->peer[q] != p->arena) cudaIpcCloseMemHandle(p->peer[q]);
  for (int q = 0; q < s2::kMaxWorld; ++q) p->peer[q] = nullptr;
  if (p->arena && p->arena_owned) cudaFree(p->arena);
  p->arena = nullptr;
  p->arena_owned = false;
  if (p->p2p) {  // tables pointed into the arena
    for (int k = 0; k < s2_plan::kTableSlots; ++k) p->tables[k] = nullptr;
  }
  p->p2p = false;
}

void s2_plan_destroy(s2_plan* plan) {
  if (plan && plan->xstream) {
    cudaStreamSynchronize(plan->xstream);
    cudaStreamDestroy(plan->xstream);
    for (int k = 0; k < s2_plan::kPipeEvents; ++k) {
      cudaEventDestroy(plan->ev_c[k]);
      cudaEventDestroy(plan->ev_x[k]);
    }
    plan->xstream = nullptr;
  }
  if (!plan) return;
  free_p2p(plan);
  if (plan->comm) ncclCommDestroy(plan->comm);
  free_scratch(plan);
  delete plan;
}

int64_t s2_plan_bitmap_words(const s2_plan* plan) { return plan ? plan->p.words : -1; }
int64_t s2_plan_block_size(const s2_plan* plan) { return plan ? plan->p.block_size : -1; }
int s2_plan_world(const s2_plan* plan) { return plan ? plan->world : -1; }

int s2_compress(const s2_plan* plan, const float* g, uint32_t* bitmap, float* table, int mask_mode,
                uint64_t* counters, void* stream) {
  if (!plan || !g || !bitmap || !table || !counters) return fail(S2_EINVAL, "NULL argument to s2_compress");
  if (mask_mode != S2_MASK_NONZERO && mask_mode != S2_MASK_GIVEN)
    return fail(S2_EINVAL, "unknown mask mode %d", mask_mode);
  if (reinterpret_cast<uintptr_t>(g) & 15) return fail(S2_EINVAL, "gradient must be 16-byte aligned");
  S2_CUDA(s2::launch_compress(plan->p, g, bitmap, table, reinterpret_cast<unsigned long long*>(counters),
                              mask_mode, as_stream(stream), false),
          "s2_compress");
  return S2_OK;
}

int s2_decode(const s2_plan* plan, const uint32_t* bitmap, const float* table, int workers, float* out,
              void* stream) {
  if (!plan || !bitmap || !table || !out) return fail(S2_EINVAL, "NULL argument to s2_decode");
  if (workers < 1) return fail(S2_EINVAL, "workers must be >= 1");  // sparse.py:208-209
  if (reinterpret_cast<uintptr_t>(out) & 15) return fail(S2_EINVAL, "output must be 16-byte aligned");
  S2_CUDA(s2::launch_decode(plan->p, bitmap, table, workers, out, as_stream(stream)), "s2_decode");
  return S2_OK;
}

int s2_bitmap_or(int64_t words, const uint32_t* stacked, int nmasks, uint32_t* out, void* stream) {
  if (nmasks < 1) return fail(S2_EINVAL, "nothing to merge");  // sparse.py:177-178
  S2_CUDA(s2::launch_bitmap_or(words, stacked, nmasks, out, as_stream(stream)), "s2_bitmap_or");
  return S2_OK;
}

int s2_table_sum(int64_t cells, const float* stacked, int ntables, float* out, void* stream) {
  if (ntables < 1) return fail(S2_EINVAL, "nothing to merge");
  S2_CUDA(s2::launch_table_sum(cells, stacked, ntables, out, as_stream(stream)), "s2_table_sum");
  return S2_OK;
}

int s2_selected_count(const s2_plan* plan, const uint32_t* bitmap, uint64_t* counters, void* stream) {
  if (!plan || !bitmap || !counters) return fail(S2_EINVAL, "NULL argument to s2_selected_count");
  S2_CUDA(s2::launch_selected_count(plan->p, bitmap, reinterpret_cast<unsigned long long*>(counters),
                                    as_stream(stream)),
          "s2_selected_count");
  return S2_OK;
}

int64_t s2_block_topk_scratch_bytes(const s2_plan* plan) {
  return plan ? s2::topk_scratch_bytes(plan->p) : -1;
}

int s2_block_topk(const s2_plan* plan, const float* g, int64_t k, uint32_t* bitmap, void* scratch, void* stream) {
  if (!plan || !g || !bitmap || !scratch) return fail(S2_EINVAL, "NULL argument to s2_block_topk");
  if (k < 1 || k > plan->p.num_blocks)
    return fail(S2_EINVAL, "k must be in [1, %lld], got %lld", (long long)plan->p.num_blocks, (long long)k);
  S2_CUDA(s2::launch_block_topk(plan->p, g, k, bitmap, scratch, as_stream(stream)), "s2_block_topk");
  return S2_OK;
}

int64_t s2_compact_scratch_bytes(const s2_plan* plan) {
  return plan ? s2::compact_scratch_bytes(plan->p) : -1;
}

int s2_compact(const s2_plan* plan, const uint32_t* bitmap, const float* g, int64_t* idx_out,
               float* val_out, int64_t* count, void* scratch, void* stream) {
  if (!plan || !bitmap || !count || !scratch) return fail(S2_EINVAL, "NULL argument to s2_compact");
  if (g && (reinterpret_cast<uintptr_t>(g) & 15)) return fail(S2_EINVAL, "gradient must be 16-byte aligned");
  S2_CUDA(s2::launch_compact(plan->p, bitmap, g, idx_out, g ? val_out : nullptr, count, scratch,
                             as_stream(stream)),
          "s2_compact");
  return S2_OK;
}

int s2_sketch_insert(const s2_plan* plan, const int64_t* idx, const float* vals, int64_t n, float* table,
                     void* stream) {
  if (!plan || (n > 0 && (!idx || !vals || !table))) return fail(S2_EINVAL, "NULL argument to s2_sketch_insert");
  S2_CUDA(s2::launch_pairs(plan->p, idx, vals, n, table, nullptr, as_stream(stream)), "s2_sketch_insert");
  return S2_OK;
}

int s2_sketch_query(const s2_plan* plan, const int64_t* idx, int64_t n, const float* table, float* out,
                    void* stream) {
  if (!plan || (n > 0 && (!idx || !table || !out))) return fail(S2_EINVAL, "NULL argument to s2_sketch_query");
  S2_CUDA(s2::launch_pairs(plan->p, idx, nullptr, n, table, out, as_stream(stream)), "s2_sketch_query");
  return S2_OK;
}

// ------------------------------------------------------------ distributed

int s2_nccl_unique_id(void* out) {
  ncclUniqueId id;
  S2_NCCL(ncclGetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out, &id, sizeof id);
  return S2_OK;
}

static int ensure_scratch(s2_plan* p) {
  if (p->tables[0] || p->p2p) return S2_OK;
  const size_t cells4 = ((size_t)p->p.hp.rows * p->p.hp.cols + 3) / 4 * 4;  // decode zeroes float4s
  const size_t wb = sizeof(uint32_t) * ((size_t)p->p.words + 4);
  for (int k = 0; k < s2_plan::kTableSlots; ++k) {
    S2_CUDA(cudaMalloc(&p->tables[k], cells4 * sizeof(float)), "cudaMalloc(table)");
    S2_CUDA(cudaMemset(p->tables[k], 0, cells4 * sizeof(float)), "cudaMemset(table)");
    S2_CUDA(cudaMalloc(&p->counters[k], sizeof(unsigned long long) * S2_NUM_COUNTERS), "cudaMalloc(counters)");
    S2_CUDA(cudaMemset(p->counters[k], 0, sizeof(unsigned long long) * S2_NUM_COUNTERS), "cudaMemset(counters)");
  }
  p->step = 0;
  for (int k = 0; k < 2; ++k) S2_CUDA(cudaMalloc(&p->bitmaps[k], wb), "cudaMalloc(bitmap)");
  S2_CUDA(cudaMalloc(&p->unionmap, wb), "cudaMalloc(union)");
  if (p->world > 1)
    S2_CUDA(cudaMalloc(&p->gather, sizeof(uint32_t) * (size_t)p->p.words * p->world), "cudaMalloc(gather)");
  S2_CUDA(cudaDeviceSynchronize(), "scratch init");
  return S2_OK;
}

static int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// Arena layout (identical on every rank):
//   tables[4] | bitmaps[4] | unions[2] | flags_a[W*8G] | flags_b[W*8G] | epochs[8G] | error | tsum[2]?
//   | inbox[2]? (push exchange)
// (flag and epoch slots for exchange grids of up to 8 CTAs per SM)
static int64_t layout_p2p(s2_plan* plan, int W, int G) {
  const int64_t cells = round_up((int64_t)plan->p.hp.rows * plan->p.hp.cols, 4 * W);
  const int64_t words = round_up(plan->p.words, 4 * W);
  s2::P2PArgs& a = plan->pa;
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    const int64_t o = off;
    off = round_up(off + bytes, 256);
    return o;
  };
  for (int k = 0; k < s2_plan::kTableSlots; ++k) a.off_table[k] = take(cells * 4);
  for (int k = 0; k < s2_plan::kTableSlots; ++k) a.off_bitmap[k] = take(words * 4);
  for (int k = 0; k < 2; ++k) a.off_union[k] = take(words * 4);
  a.off_flags_a = take((int64_t)W * 8 * G * 4);
  a.off_flags_b = take((int64_t)W * 8 * G * 4);
  a.off_epoch = take((int64_t)8 * G * 4);
  a.off_error = take(256);
  const char* os_env = getenv("S2_P2P_ONESHOT_MAXW");
  const int oneshot_maxw = os_env ? atoi(os_env) : 2;
  a.oneshot = (W <= oneshot_maxw && W <= 4) ? 1 : 0;
  for (int k = 0; k < 2; ++k) a.off_tsum[k] = a.oneshot ? take(cells * 4) : -1;  // two-shot: in place
  // push (data stored into the peers' inboxes before each flag) is the default for the two-shot
  // exchange: W = 4 step 84.9 -> 82.0 µs; the one-shot keeps pulling: W = 2 push 67.3 vs pull
  // 66.1 µs (profiles/r02_push_ab.txt).  S2_P2P_PUSH=0/1 forces either.
  const char* pe = getenv("S2_P2P_PUSH");
  a.push = pe ? atoi(pe) : (a.oneshot ? 0 : 1);
  // inbox: one-shot W slots of the whole table + bitmap, two-shot W slots of one slice each
  for (int k = 0; k < 2; ++k) a.off_inbox[k] = a.push ? take((a.oneshot ? W : 1) * (cells + words) * 4) : -1;
  a.cells = cells;
  a.words = words;
  a.world = W;
  a.rank = plan->rank;
  return off;
}

static int sm_count(int* G) {
  int dev = 0;
  S2_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  S2_CUDA(cudaDeviceGetAttribute(G, cudaDevAttrMultiProcessorCount, dev), "sm count");
  return S2_OK;
}

// base pointers known: plan tables into the arena, counters, trace, grid, timeout
static int finish_p2p(s2_plan* plan, int G) {
  s2::P2PArgs& a = plan->pa;
  // exchange-kernel CTAs (1024 threads each): one per two SMs at W <= 2 (pull one-shot), one per
  // four SMs at W > 2 (push two-shot), at every exchange size.  Fewer CTAs cost little or nothing
  // one reduce at a time and leave more of the GPU to the compress and decode that s2_reduce_many
  // overlaps with the exchange (profiles/r02_ab_exchange_grid.txt): per reduce W = 4 ResNet-50
  // 70.2 -> 66.0 µs (one at a time 80.1 / 80.0), BERT 770 (#SMs) -> 707 µs (770 / 775); W = 2
  // GPT-2-M 99 % 616 (#SMs) -> 577 µs (614 / 617), LSTM 351 -> 329 µs (354 / 362).
  plan->p2p_grid = a.world > 2 ? (G >= 4 ? G / 4 : 1) : (G >= 2 ? G / 2 : 1);
  const char* ge = getenv("S2_P2P_GRID");  // override (A/B runs)
  if (ge && atoi(ge) > 0 && atoi(ge) <= 8 * G) plan->p2p_grid = atoi(ge);
  if (plan->opt_grid > 0) plan->p2p_grid = plan->opt_grid;
  double tmo = plan->opt_timeout_s;
  if (tmo <= 0) {
    const char* te = getenv("S2_P2P_TIMEOUT_S");
    tmo = te && atof(te) > 0 ? atof(te) : 300.0;
  }
  a.timeout_ns = (unsigned long long)(tmo * 1e9);
  plan->p2p = true;
  a.trace = nullptr;
  const char* tr = getenv("S2_P2P_TRACE");
  if (tr && atoi(tr)) {
    S2_CUDA(cudaMalloc(&a.trace, sizeof(unsigned long long) * 64 * G), "cudaMalloc(trace)");
    S2_CUDA(cudaMemset(a.trace, 0, sizeof(unsigned long long) * 64 * G), "cudaMemset(trace)");
  }
  for (int k = 0; k < s2_plan::kTableSlots; ++k) {
    plan->tables[k] = reinterpret_cast<float*>(plan->arena + a.off_table[k]);
    S2_CUDA(cudaMalloc(&plan->counters[k], sizeof(unsigned long long) * S2_NUM_COUNTERS), "cudaMalloc(counters)");
    S2_CUDA(cudaMemset(plan->counters[k], 0, sizeof(unsigned long long) * S2_NUM_COUNTERS), "cudaMemset(counters)");
  }
  plan->step = 0;
  S2_CUDA(s2::preload_compress(plan->p), "preload compress");
  S2_CUDA(s2::preload_decode(plan->p), "preload decode");
  S2_CUDA(s2::preload_p2p(plan->pa), "preload exchange");
  S2_CUDA(cudaDeviceSynchronize(), "p2p init");
  return S2_OK;
}

// CUDA-IPC arena: one cudaMalloc per rank, handles exchanged through one ncclAllGather
static int setup_p2p(s2_plan* plan) {
  const int W = plan->world;
  int G = 0;
  int rc = sm_count(&G);
  if (rc) return rc;
  if (plan->opt_grid > 8 * G) return fail(S2_EINVAL, "exchange grid must be <= %d", 8 * G);
  const int64_t off = layout_p2p(plan, W, G);
  s2::P2PArgs& a = plan->pa;
  S2_CUDA(cudaMalloc(&plan->arena, off), "cudaMalloc(arena)");
  S2_CUDA(cudaMemset(plan->arena, 0, off), "cudaMemset(arena)");
  S2_CUDA(cudaDeviceSynchronize(), "arena init");
  plan->arena_owned = true;
  struct Rec {
    cudaIpcMemHandle_t h;
    int64_t bytes;
    int64_t grid;
  } rec{};
  S2_CUDA(cudaIpcGetMemHandle(&rec.h, plan->arena), "cudaIpcGetMemHandle");
  rec.bytes = off;
  rec.grid = G;
  static_assert(sizeof(Rec) % 8 == 0, "rec");
  char* d = nullptr;
  S2_CUDA(cudaMalloc(&d, sizeof(Rec) * (W + 1)), "cudaMalloc(handles)");
  std::vector<Rec> all(W);
  cudaStream_t st = nullptr;
  S2_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  rc = S2_OK;
  if (cudaMemcpyAsync(d, &rec, sizeof rec, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      ncclAllGather(d, d + sizeof(Rec), sizeof(Rec), ncclUint8, plan->comm, st) != ncclSuccess ||
      cudaMemcpyAsync(all.data(), d + sizeof(Rec), sizeof(Rec) * W, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    rc = fail(S2_ENCCL, "IPC handle exchange failed");
  cudaFree(d);
  cudaStreamDestroy(st);
  if (rc) return rc;
  for (int q = 0; q < W; ++q) {
    if (all[q].bytes != off || all[q].grid != G)
      return fail(S2_EINCOMPAT, "incompatible payloads: field 'sketch_params' differs (arena layout of rank %d)", q);
    if (q == plan->rank) {
      plan->peer[q] = plan->arena;
    } else {
      void* p = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&p, all[q].h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle (set S2_AGG=nccl to use NCCL instead)");
      plan->peer[q] = static_cast<char*>(p);
    }
    a.base[q] = plan->peer[q];
  }
  return finish_p2p(plan, G);
}

int s2_comm_set_options(s2_plan* plan, int exchange_grid, double timeout_s) {
  if (!plan) return fail(S2_EINVAL, "NULL plan");
  if (plan->p2p || plan->comm) return fail(S2_EINVAL, "s2_comm_set_options must precede s2_comm_init");
  if (exchange_grid < 0) return fail(S2_EINVAL, "exchange grid must be >= 0, got %d", exchange_grid);
  plan->opt_grid = exchange_grid;
  plan->opt_timeout_s = timeout_s;
  return S2_OK;
}

int s2_comm_init_mode(s2_plan* plan, int world, int rank, const void* unique_id, int mode) {
  if (!plan) return fail(S2_EINVAL, "NULL plan");
  if (mode < S2_COMM_IPC || mode > S2_COMM_EXTERNAL) return fail(S2_EINVAL, "unknown comm mode %d", mode);
  plan->comm_mode = mode;
  return s2_comm_init(plan, world, rank, unique_id);
}

int64_t s2_p2p_arena_bytes(s2_plan* plan, int world) {
  if (!plan || world < 2 || world > s2::kMaxWorld) return -1;
  int G = 0;
  if (sm_count(&G)) return -1;
  const int saved = plan->world;
  const s2::P2PArgs saved_pa = plan->pa;
  plan->world = world;
  const int64_t b = layout_p2p(plan, world, G);
  plan->world = saved;
  plan->pa = saved_pa;
  return b;
}

int s2_comm_attach(s2_plan* plan, const uint64_t* bases, int world) {
  if (!plan || !bases) return fail(S2_EINVAL, "NULL argument to s2_comm_attach");
  if (plan->world != world || world < 2) return fail(S2_EINVAL, "attach: world %d does not match the plan", world);
  if (plan->comm_mode != S2_COMM_EXTERNAL) return fail(S2_EINVAL, "attach needs s2_comm_init_mode(..., S2_COMM_EXTERNAL)");
  if (plan->p2p) return fail(S2_EINVAL, "arenas already attached");
  int G = 0;
  int rc = sm_count(&G);
  if (rc) return rc;
  if (plan->opt_grid > 8 * G) return fail(S2_EINVAL, "exchange grid must be <= %d", 8 * G);
  const int64_t bytes = layout_p2p(plan, world, G);
  s2::P2PArgs& a = plan->pa;
  for (int q = 0; q < world; ++q) {
    if (bases[q] == 0 || (bases[q] & 255)) return fail(S2_EINVAL, "arena %d must be non-NULL and 256-byte aligned", q);
    plan->peer[q] = reinterpret_cast<char*>(bases[q]);
    a.base[q] = plan->peer[q];
  }
  plan->arena = plan->peer[plan->rank];
  plan->arena_owned = false;
  S2_CUDA(cudaMemset(plan->arena, 0, bytes), "cudaMemset(arena)");
  return finish_p2p(plan, G);
}

int s2_comm_init(s2_plan* plan, int world, int rank, const void* unique_id) {
  if (!plan) return fail(S2_EINVAL, "NULL plan");
  if (world < 1 || rank < 0 || rank >= world) return fail(S2_EINVAL, "bad world/rank %d/%d", world, rank);
  if (plan->comm || plan->p2p) return fail(S2_EINVAL, "communicator already initialised");
  free_scratch(plan);
  plan->world = world;
  plan->rank = rank;
  if (world > 1) {
    if (world > s2::kMaxWorld && plan->comm_mode != S2_COMM_NCCL)
      return fail(S2_EINVAL, "peer-memory exchange supports world <= %d", s2::kMaxWorld);
    if (plan->comm_mode == S2_COMM_EXTERNAL) return S2_OK;  // no NCCL: arenas come from s2_comm_attach
    if (!unique_id) return fail(S2_EINVAL, "NULL NCCL unique id");
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof id);
    S2_NCCL(ncclCommInitRank(&plan->comm, world, id, rank), "ncclCommInitRank");
    const char* agg = getenv("S2_AGG");
    const bool nccl_only = (agg && strcmp(agg, "nccl") == 0) || plan->comm_mode == S2_COMM_NCCL;
    if (!nccl_only) {
      int rc = setup_p2p(plan);
      if (rc) return rc;
    }
  }
  return ensure_scratch(plan);
}

uint64_t s2_plan_digest(const s2_plan* plan) {
  if (!plan) return 0;
  const Plan& q = plan->p;
  // compat_key: partition + sketch params (sparse.py:105-109)
  const uint64_t parts[7] = {(uint64_t)q.dim, (uint64_t)q.num_blocks, (uint64_t)q.hp.rows,
                             (uint64_t)q.hp.cols, q.seed, (uint64_t)q.injective, 0x53325348ull};
  return derive(parts, 7);
}

int s2_comm_check(s2_plan* plan, void* stream) {
  if (!plan) return fail(S2_EINVAL, "NULL plan");
  if (plan->world == 1 || plan->comm_mode == S2_COMM_EXTERNAL) return S2_OK;  // EXTERNAL: caller compares
  if (!plan->comm) return fail(S2_EINVAL, "s2_comm_check needs s2_comm_init");
  const uint64_t mine = s2_plan_digest(plan);
  uint64_t* d = nullptr;
  S2_CUDA(cudaMalloc(&d, sizeof(uint64_t) * (plan->world + 1)), "cudaMalloc(check)");
  cudaStream_t st = as_stream(stream);
  int rc = S2_OK;
  std::vector<uint64_t> all(plan->world);
  if (cudaMemcpyAsync(d, &mine, sizeof mine, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      ncclAllGather(d, d + 1, 1, ncclUint64, plan->comm, st) != ncclSuccess ||
      cudaMemcpyAsync(all.data(), d + 1, sizeof(uint64_t) * plan->world, cudaMemcpyDeviceToHost, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    rc = fail(S2_ENCCL, "parameter agreement exchange failed");
  } else {
    for (int r = 0; r < plan->world; ++r)
      if (all[r] != mine) {
        rc = fail(S2_EINCOMPAT, "incompatible payloads: field 'sketch_params' differs (rank %d vs rank %d)",
                  plan->rank, r);
        break;
      }
  }
  cudaFree(d);
  return rc;
}

int s2_aggregate(s2_plan* plan, float* table, const uint32_t* bitmap, uint32_t* union_out, void* stream) {
  if (!plan || !table || !bitmap || !union_out) return fail(S2_EINVAL, "NULL argument to s2_aggregate");
  cudaStream_t st = as_stream(stream);
  const Plan& q = plan->p;
  if (plan->world == 1) {
    if (union_out != bitmap)
      S2_CUDA(cudaMemcpyAsync(union_out, bitmap, sizeof(uint32_t) * q.words, cudaMemcpyDeviceToDevice, st),
              "copy bitmap");
    return S2_OK;
  }
  int rc = ensure_scratch(plan);
  if (rc) return rc;
  if (!plan->comm) return fail(S2_EINVAL, "s2_aggregate needs an NCCL communicator (s2_comm_init)");
  if (!plan->gather)  // peer-memory plans skip the NCCL landing buffer until asked
    S2_CUDA(cudaMalloc(&plan->gather, sizeof(uint32_t) * (size_t)q.words * plan->world), "cudaMalloc(gather)");
  const size_t cells = (size_t)q.hp.rows * q.hp.cols;
  // sketch sum (sketch.py:213-216) and bitmap gather, one NCCL group over NVLink
  S2_NCCL(ncclGroupStart(), "ncclGroupStart");
  S2_NCCL(ncclAllReduce(table, table, cells, ncclFloat32, ncclSum, plan->comm, st), "ncclAllReduce(table)");
  S2_NCCL(ncclAllGather(bitmap, plan->gather, (size_t)q.words, ncclUint32, plan->comm, st),
          "ncclAllGather(bitmap)");
  S2_NCCL(ncclGroupEnd(), "ncclGroupEnd");
  // BlockMask.union (sparse.py:55-58) — NCCL has no bitwise-OR reduction
  S2_CUDA(s2::launch_bitmap_or(q.words, plan->gather, plan->world, union_out, st), "bitmap OR");
  return S2_OK;
}

// One reduce = compress -> exchange -> decode.  The three stages are split so that
// s2_reduce_many can interleave consecutive reduces (compress of step i+1 between the exchange
// and the decode of step i).
struct StepBufs {
  int cur, tc, tz;  // bitmap / union / tsum / inbox slot, table slot, slot the decode zeroes
  float* table;
  uint32_t* bitmap;
  unsigned long long* cnt;
  const uint32_t* un;
  const float* dec_table;
  s2::DecodeHealth health;
};

static int check_reduce_args(s2_plan* plan, const float* g, const float* out) {
  if (!plan || !g || !out) return fail(S2_EINVAL, "NULL argument to s2_reduce");
  if (reinterpret_cast<uintptr_t>(g) & 15) return fail(S2_EINVAL, "gradient must be 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(out) & 15) return fail(S2_EINVAL, "output must be 16-byte aligned");
  if (plan->world > 1 && !plan->p2p && !plan->comm)
    return fail(S2_EINVAL, "world > 1 needs s2_comm_init (and s2_comm_attach in EXTERNAL mode)");
  if (plan->overlap < 0) {
    const char* e = getenv("S2_OVERLAP");
    plan->overlap = e ? atoi(e) : 1;
  }
  return ensure_scratch(plan);
}

static bool overlaps(const void* a, const void* b, size_t n) {
  const char* x = static_cast<const char*>(a);
  const char* y = static_cast<const char*>(b);
  return x != nullptr && y != nullptr && x < y + n && y < x + n;
}

// compress of step plan->step (slots from the step counter); `late`: may overlap its predecessor
static int stage_compress(s2_plan* plan, const float* g, uint64_t* counters, bool late, cudaStream_t st,
                          StepBufs* b) {
  NvtxRange nvtx_("s2 compress");
  b->cur = (int)(plan->step & 1);
  b->tc = (int)(plan->step & 3);
  b->tz = (int)((plan->step + 2) & 3);
  b->table = plan->tables[b->tc];
  b->bitmap = plan->p2p ? reinterpret_cast<uint32_t*>(plan->arena + plan->pa.off_bitmap[b->tc]) : plan->bitmaps[b->cur];
  // caller counters: zeroed by memset; plan counters: zeroed by the decode two reduces back
  b->cnt = counters ? reinterpret_cast<unsigned long long*>(counters) : plan->counters[b->tc];
  S2_CUDA(s2::launch_compress(plan->p, g, b->bitmap, b->table, b->cnt, S2_MASK_NONZERO, st, counters == nullptr,
                              late),
          "s2_reduce/compress");
  return S2_OK;
}

static int stage_exchange(s2_plan* plan, cudaStream_t st, void* stream, StepBufs* b) {
  NvtxRange nvtx_("s2 exchange");
  b->un = b->bitmap;
  b->dec_table = b->table;
  b->health = s2::DecodeHealth{nullptr, b->cnt, plan->status, 0};
  if (plan->world == 1) return S2_OK;
  if (plan->p2p) {
    plan->pa.cur = b->cur;
    plan->pa.tcur = b->tc;
    S2_CUDA(s2::launch_p2p_aggregate(plan->pa, plan->p2p_grid, st), "s2_reduce/p2p aggregate");
    b->un = reinterpret_cast<const uint32_t*>(plan->arena + plan->pa.off_union[b->cur]);
    if (plan->pa.oneshot) b->dec_table = reinterpret_cast<const float*>(plan->arena + plan->pa.off_tsum[b->cur]);
    b->health.poison = reinterpret_cast<const uint32_t*>(plan->arena + plan->pa.off_error);
    return S2_OK;
  }
  int rc = s2_aggregate(plan, b->table, b->bitmap, plan->unionmap, stream);
  if (rc) return rc;
  b->un = plan->unionmap;
  return S2_OK;
}

static int stage_decode(s2_plan* plan, float* out, cudaStream_t st, const StepBufs& b) {
  NvtxRange nvtx_("s2 decode");
  S2_CUDA(s2::launch_decode(plan->p, b.un, b.dec_table, plan->world, out, st, plan->tables[b.tz],
                            plan->counters[b.tz], &b.health),
          "s2_reduce/decode");
  return S2_OK;
}

int s2_reduce(s2_plan* plan, const float* g, float* out, uint64_t* counters, void* stream) {
  NvtxRange nvtx_("s2_reduce");
  int rc = check_reduce_args(plan, g, out);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  // The compress may overlap the previous reduce's decode (it shares no buffer with it) unless its
  // input is that decode's output (g aliasing the previous out) — then it waits up front.
  const bool late = plan->overlap != 0 && !overlaps(g, plan->prev_out, sizeof(float) * (size_t)plan->p.dim);
  StepBufs b{};
  if (plan->ev[0]) cudaEventRecord(plan->ev[0], st);
  if ((rc = stage_compress(plan, g, counters, late, st, &b))) return rc;
  if (plan->ev[1]) cudaEventRecord(plan->ev[1], st);
  if ((rc = stage_exchange(plan, st, stream, &b))) return rc;
  if (plan->ev[2]) cudaEventRecord(plan->ev[2], st);
  if ((rc = stage_decode(plan, out, st, b))) return rc;
  if (plan->ev[3]) cudaEventRecord(plan->ev[3], st);
  plan->prev_out = out;
  plan->step += 1;
  return S2_OK;
}

int s2_reduce_many(s2_plan* plan, const float* const* gs, float* const* outs, int n, void* stream) {
  NvtxRange nvtx_("s2_reduce_many");
  if (!plan || n < 0 || (n > 0 && (!gs || !outs))) return fail(S2_EINVAL, "NULL argument to s2_reduce_many");
  if (n == 0) return S2_OK;
  for (int k = 0; k < n; ++k) {
    int rc = check_reduce_args(plan, gs[k], outs[k]);
    if (rc) return rc;
  }
  // Pipelining needs every input to be independent of every earlier output of the batch, an
  // exchange to hide (world > 1), the overlap switch on, and no timing events.
  const size_t nb = sizeof(float) * (size_t)plan->p.dim;
  bool pipe = plan->world > 1 && plan->overlap != 0 && plan->ev[0] == nullptr;
  for (int k = 1; pipe && k < n; ++k)
    for (int j = 0; j < k && pipe; ++j) pipe = !overlaps(gs[k], outs[j], nb);
  if (!pipe) {
    for (int k = 0; k < n; ++k) {
      int rc = s2_reduce(plan, gs[k], outs[k], nullptr, stream);
      if (rc) return rc;
    }
    return S2_OK;
  }
  cudaStream_t st = as_stream(stream);
  int rc;
  static int streams = -1;  // S2_PIPE_STREAMS=1: the one-stream schedule below (A/B switch)
  if (streams < 0) {
    const char* e = getenv("S2_PIPE_STREAMS");
    streams = e ? atoi(e) : 2;
  }
  if (plan->p2p && n > 1 && streams == 2) {
    // Two streams.  Main: compress(0) compress(1) decode(0) compress(2) decode(1) ... decode(n-1);
    // exchange stream: exchange(0) exchange(1) ..., exchange(k) after compress(k), decode(k) after
    // exchange(k).  Every exchange (NVLink- and latency-bound, a quarter to half of the SMs) runs
    // beside the HBM-bound compress AND decode of the neighbouring reduces, so a batch costs about
    // (compress + decode) per reduce once the exchange is shorter than that.  Buffer safety: table
    // and bitmap slots rotate over 4, union / tsum / inbox over 2; exchange(k+1) touches slots k+1
    // only, while decode(k) reads slots k and zeroes table slot k+2, whose compress follows it
    // (DESIGN.md §7).
    if (!plan->xstream) {
      int lo = 0, hi = 0;
      S2_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
      // highest priority: exchange CTAs take SMs as the neighbouring kernels' CTAs retire (lowest
      // priority measured 1-10 % slower per reduce, profiles/r02_ab_pipe_streams.txt)
      S2_CUDA(cudaStreamCreateWithPriority(&plan->xstream, cudaStreamNonBlocking, hi), "exchange stream");
      for (int k = 0; k < s2_plan::kPipeEvents; ++k) {
        S2_CUDA(cudaEventCreateWithFlags(&plan->ev_c[k], cudaEventDisableTiming), "event");
        S2_CUDA(cudaEventCreateWithFlags(&plan->ev_x[k], cudaEventDisableTiming), "event");
      }
    }
    cudaStream_t xs = plan->xstream;
    StepBufs prev{}, cur{};
    auto exchange = [&](StepBufs* b, int k) -> int {
      cudaEvent_t ec = plan->ev_c[k % s2_plan::kPipeEvents], ex = plan->ev_x[k % s2_plan::kPipeEvents];
      S2_CUDA(cudaEventRecord(ec, st), "record compress");
      S2_CUDA(cudaStreamWaitEvent(xs, ec, 0), "exchange waits compress");
      int r = stage_exchange(plan, xs, xs, b);
      if (r) return r;
      S2_CUDA(cudaEventRecord(ex, xs), "record exchange");
      return S2_OK;
    };
    auto decode = [&](StepBufs b, float* out, int k) -> int {
      S2_CUDA(cudaStreamWaitEvent(st, plan->ev_x[k % s2_plan::kPipeEvents], 0), "decode waits exchange");
      b.health.fence_zero = 1;  // the next compress on this stream uses the table it zeroes
      return stage_decode(plan, out, st, b);
    };
    const bool late0 = !overlaps(gs[0], plan->prev_out, nb);
    if ((rc = stage_compress(plan, gs[0], nullptr, late0, st, &prev))) return rc;
    if ((rc = exchange(&prev, 0))) return rc;
    plan->step += 1;
    for (int k = 1; k < n; ++k) {
      // compress(1) directly follows compress(0): its table was zeroed by the decode two reduces
      // back, whose completion only compress(0)'s exit guarantees, so it waits up front
      if ((rc = stage_compress(plan, gs[k], nullptr, k > 1, st, &cur))) return rc;
      if ((rc = exchange(&cur, k))) return rc;
      if ((rc = decode(prev, outs[k - 1], k - 1))) return rc;
      plan->step += 1;
      prev = cur;
    }
    if ((rc = decode(prev, outs[n - 1], n - 1))) return rc;
    plan->prev_out = outs[n - 1];
    return S2_OK;
  }
  // one stream: compress(0) exchange(0) | compress(1) decode(0) exchange(1) | compress(2) decode(1) ...
  // decode(n-1): each compress runs beside the previous exchange; the decode of step k waits for
  // compress(k+1), which waited for exchange(k) before completing.
  StepBufs prev{}, cur{};
  const bool late0 = !overlaps(gs[0], plan->prev_out, nb);
  if ((rc = stage_compress(plan, gs[0], nullptr, late0, st, &prev))) return rc;
  if ((rc = stage_exchange(plan, st, stream, &prev))) return rc;
  plan->step += 1;
  for (int k = 1; k < n; ++k) {
    if ((rc = stage_compress(plan, gs[k], nullptr, true, st, &cur))) return rc;
    if ((rc = stage_decode(plan, outs[k - 1], st, prev))) return rc;
    if ((rc = stage_exchange(plan, st, stream, &cur))) return rc;
    plan->step += 1;
    prev = cur;
  }
  if ((rc = stage_decode(plan, outs[n - 1], st, prev))) return rc;
  plan->prev_out = outs[n - 1];
  return S2_OK;
}

int s2_plan_set_status(s2_plan* plan, uint32_t* status) {
  if (!plan) return fail(S2_EINVAL, "NULL plan");
  plan->status = status;
  return S2_OK;
}

int s2_p2p_error(const s2_plan* plan) {
  if (!plan || !plan->p2p) return 0;
  uint32_t e = 0;
  cudaMemcpy(&e, plan->arena + plan->pa.off_error, 4, cudaMemcpyDeviceToHost);
  return (int)e;
}

int s2_p2p_trace(const s2_plan* plan, uint64_t* host, int64_t n) {
  if (!plan || !plan->p2p || !plan->pa.trace) return fail(S2_EINVAL, "no p2p trace (set S2_P2P_TRACE=1)");
  const int64_t m = (int64_t)plan->p2p_grid * 64 < n ? (int64_t)plan->p2p_grid * 64 : n;
  S2_CUDA(cudaMemcpy(host, plan->pa.trace, sizeof(uint64_t) * m, cudaMemcpyDeviceToHost), "trace copy");
  return S2_OK;
}

int s2_plan_set_timing_events(s2_plan* plan, void* const* events, int n) {
  if (!plan) return fail(S2_EINVAL, "NULL plan");
  if (n != 0 && n != 4) return fail(S2_EINVAL, "need 0 or 4 events");
  for (int k = 0; k < 4; ++k) plan->ev[k] = n ? reinterpret_cast<cudaEvent_t>(events[k]) : nullptr;
  return S2_OK;
}

int s2_read_counters(const s2_plan* plan, uint64_t* host_out, void* stream) {
  if (!plan || !host_out) return fail(S2_EINVAL, "NULL argument to s2_read_counters");
  if (!plan->counters[0]) {
    memset(host_out, 0, sizeof(uint64_t) * S2_NUM_COUNTERS);
    return S2_OK;
  }
  cudaStream_t st = as_stream(stream);
  S2_CUDA(cudaMemcpyAsync(host_out, plan->counters[(plan->step + 3) & 3], sizeof(uint64_t) * S2_NUM_COUNTERS,
                          cudaMemcpyDeviceToHost, st), "read counters");
  S2_CUDA(cudaStreamSynchronize(st), "read counters");
  return S2_OK;
}

const uint64_t* s2_last_counters(const s2_plan* plan) {
  if (!plan || !plan->counters[0]) return nullptr;
  return reinterpret_cast<const uint64_t*>(plan->counters[(plan->step + 3) & 3]);
}

}  // extern "C"
