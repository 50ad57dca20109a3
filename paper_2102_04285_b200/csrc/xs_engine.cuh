// xs_engine.cuh -- context, workspace and the host-side pipeline contracts.
#pragma once
#include <initializer_list>
#include <cstdio>
#include <functional>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "xs_common.cuh"

namespace xs {

// Device-side counters filled by the scan passes, copied to pinned host
// memory at the few points where the host has to size the next stage.
struct Stats {
  long long n_bad;          // event-rule + dangling-correlation + nesting violations
  long long n_nonzero;      // events with duration > 0
  long long n_ops_nz;       // OPERATION events with duration > 0
  long long n_ops;          // all OPERATION events
  long long n_api;          // ACCEL_API events
  long long n_api_corr;     // ACCEL_API events with a correlation
  long long n_gpu_corr;     // GPU events with a correlation
  long long max_span;       // max over pids of (hi - lo)
  long long bad_api;        // first ACCEL_API index missing from the profile
  long long max_depth;      // deepest OPERATION nesting (per tid)
  long long table_full;     // a hash table ran out of slots
  long long multi_op_pids;  // pids whose OPERATIONs sit on >1 tid
  long long n_trans;        // wrapper transition sites
  long long n_sites;        // correction hook sites
  long long depth_overflow; // merged multi-tid path deeper than the local limit
  long long n_fixed;        // CORRELATION: GPU events with a fixed path
  long long n_pieces;       // CORRELATION: own-path pieces
  long long pad[15];
  long long cat_all[8];     // events per category
  long long cat_nz[8];      // events per category with duration > 0
};

enum Slot : int {
  W_STATS = 0,
  W_SPAN_LO, W_SPAN_HI, W_PID_OPS, W_GROUP_OPS, W_PID_GROUP0,
  W_CORR_STATE, W_CORR_KEY, W_CORR_PID, W_CORR_START,
  W_OP_EV, W_OPK0, W_OPK1, W_OPV0, W_OPV1,
  W_SKEY, W_SVAL, W_SKEY_ALT, W_SVAL_ALT,
  W_DEPTH_SCAN_DESC, W_DEPTH_SCAN_FLAGS, W_TILE_CTR,
  W_DOPEN, W_POPEN, W_DCLOSE, W_PARENT, W_NODE, W_READY, W_DKEY, W_DVAL, W_DKEY_ALT, W_DVAL_ALT,
  W_TRIE_KEYS, W_TRIE_VALS, W_TRIE_PARENT, W_TRIE_NAME, W_TRIE_COUNT,
  W_GS_OFF, W_PK, W_PK_ALT, W_PIDPATH, W_OPBASE,
  W_MKEY, W_MKEY_ALT, W_MSCAN_DESC, W_MSCAN_FLAGS,
  W_HIST, W_HIST_KEY, W_CELL_PID, W_CELL_NODE, W_CELL_MASK, W_CELL_NS, W_CELL_COUNT, W_TRACKED,
  W_CUB_TEMP,
  // correction
  W_TQ_KEY, W_TQ_VAL, W_TQ_KEY_ALT, W_TQ_VAL_ALT, W_TSCAN_DESC, W_TSCAN_FLAGS, W_THEAD, W_TSTAT,
  W_SITE_FLAG, W_SITE_CNT, W_SITE_POS, W_SITE_K, W_SITE_V, W_SITE_K_ALT, W_SITE_V_ALT,
  W_QSCAN_DESC, W_QSCAN_FLAGS, W_QSLOT, W_LENSLOT, W_REMOVED, W_SHORTFALL,
  W_RSCAN_DESC, W_RSCAN_FLAGS, W_SLAB_A, W_SLAB_B, W_SLAB_PRE, W_SLAB_CNT, W_SLAB_BASE,
  W_SITES_LEN, W_TRANS_OUT_PAIR, W_TRANS_OUT_EV,
  // correlation
  W_FIXED_LS, W_FIXED_PATH, W_PIECE_KEY, W_FX_KEY, W_FX_KEY_ALT, W_FX_VAL, W_FX_VAL_ALT,
  W_FXSCAN_DESC, W_FXSCAN_FLAGS, W_FX_OWN, W_RANK_EV,
  // correction (dedicated: xs_remap reads them after an xs_analyze overlap pass)
  W_CORR_LO, W_CORR_HI, W_PTOTAL, W_PID_SLABS, W_SITE_EV, W_SITE_SUB, W_QVAL, W_OUT_LO, W_OUT_HI,
  // transitions
  W_TSKEY, W_TSKEY_ALT, W_HEADPOS, W_TREC_ID, W_TREC_ID_ALT,
  // bucketed sorts
  W_BK_COUNTS, W_BK_FILL, W_BK_OFFS, W_BK_CSTART, W_BK_CFIRST,
  W_CORR_TOTALS, W_NS_DEV, W_STATS_SAVE, W_PID_OPS_ALT, W_GROUP_OPS_ALT, W_PID_GROUP0_ALT,
  W_BS_COUNTS, W_BS_OFFS, W_BS_TAIL, W_BS_CHUNK, W_RMAP_IDX,
  W_CUB_TEMP2, W_OPG, W_OPG_INV, W_TGRP_FLAG, W_TGRP_IDX, W_TILE_CTR_B, W_CUB_TEMP_B, W_BS_COUNTS_B, W_BS_OFFS_B, W_BS_TAIL_B, W_BS_CHUNK_B,
  W_UN_GSPAN, W_UN_ACC, W_UN_SEG, W_UN_KEY, W_UN_KEY_ALT, W_UN_DEPTH, W_UN_RANK, W_UN_IV,
  W_DEEP_OVF, W_DEEP_SCRATCH,
  W_PSCAN_DESC, W_PSCAN_FLAGS, W_PSCAN_CTR, W_PSCAN_DESC_B, W_PSCAN_FLAGS_B, W_PSCAN_CTR_B, W_SEL_COUNT,
  W_KSORT_VAL, W_KSORT_VAL_ALT, W_SYN_IT, W_SYN_NK, W_SYN_PID, W_SYN_K,
  W_NUM_SLOTS
};

// Lock-free (parent node, name) -> node table: the PathTable of
// overlap.py:80-93 as a trie (a name tuple and its trie node are in
// bijection, so ids are internal exactly as in the reference).
struct TrieView {
  uint64_t* keys;  // (parent << 32 | name), ~0 = empty
  int* vals;       // node id, -1 until published
  int* parent;     // [node_cap]
  int* name;       // [node_cap]
  int* count;      // number of nodes (root = 0 pre-created)
  uint64_t mask;   // table capacity - 1
  int node_cap;    // grow trigger: count >= node_cap
  Stats* st;
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

// child of `parent` named `name`, collapsing an adjacent duplicate name
// (_sweep_py.py:22-24).  Returns the node id (0 on table overflow, with
// Stats.table_full raised so the host re-runs with a larger table).
__device__ __forceinline__ int trie_intern(int parent, int name, const TrieView& t) {
  if (parent > 0 && ((volatile int*)t.name)[parent] == name) return parent;
  const uint64_t key = ((uint64_t)(uint32_t)parent << 32) | (uint32_t)name;
  uint64_t h = mix64(key) & t.mask;
  for (uint64_t probe = 0; probe <= t.mask; probe++) {
    uint64_t k = ((volatile uint64_t*)t.keys)[h];
    if (k == ~0ull) {
      unsigned long long prev = atomicCAS((unsigned long long*)&t.keys[h], ~0ull, (unsigned long long)key);
      if (prev == ~0ull) {
        int id = atomicAdd(t.count, 1);
        if (id >= t.node_cap) {
          atomicAdd((unsigned long long*)&t.st->table_full, 1ull);
          id = 0;
        } else {
          t.parent[id] = parent;
          t.name[id] = name;
        }
        __threadfence();
        atomicExch(&t.vals[h], id);
        return id;
      }
      k = prev;
    }
    if (k == key) {
      int id;
      while ((id = ((volatile int*)t.vals)[h]) < 0) {
      }
      __threadfence();
      return id;
    }
    h = (h + 1) & t.mask;
  }
  atomicAdd((unsigned long long*)&t.st->table_full, 1ull);
  return 0;
}

// Results of stage_ops consumed by the sweep.
struct OpsState {
  int64_t m = 0;          // nonzero OPERATION events
  int tb = 0;             // relative-time bits
  const uint64_t* skeys = nullptr;  // per-group endpoint stream keys (group|t|open)
  const uint32_t* svals = nullptr;  // rank of the op at each stream position
  const int* rank_ev = nullptr;     // event row of each rank
  const int* parent = nullptr;      // parent rank (-1 = none)
  const int* node = nullptr;        // trie node of each rank's single-tid chain
  const uint64_t* pk = nullptr;     // op endpoints in (pid, t) order (pid|t|open)
  const int* pidpath = nullptr;     // path node after each run end of pk
  const int64_t* opbase = nullptr;  // [n_pids+1] first pk index of each pid
  TrieView trie{};
};

}  // namespace xs

namespace xs {
struct BucketGeom {  // bucketed sorts (xs_bucket.cuh)
  int key_bits;  // keys occupy [0, key_bits)
  int bb;        // bucket bits
  int shift;     // bucket = key >> shift
  int64_t nbuckets;
};
struct BkPlan {  // a prepared bucketed endpoint sort (xs_overlap.cu)
  bool ready = false;
  BucketGeom g{};
  int64_t nvalid = 0, n_chunks = 0, n = 0;
  bool pid_chunks = false;
  uint64_t* keys = nullptr;
  int64_t* chunk = nullptr;
  int tb = 0, key_bits = 0;
  const int64_t* start = nullptr;
};
}  // namespace xs

struct xs_ctx {
  int device = 0;
  std::string err;
  std::vector<void*> ptr;
  std::vector<size_t> cap;
  xs::Stats* h_stats = nullptr;  // pinned: [0] last fetch, [1] saved correction stats
  int64_t* h_totals = nullptr;   // pinned [4]: W_CORR_TOTALS as of the last correction
  int64_t* h_report = nullptr;   // pinned: removed[np*4] then shortfall[np*4] of the last correction
  size_t h_report_cap = 0;
  long long launches = 0;
  // last overlap result
  long long n_cells = 0;
  int n_nodes = 0;
  int res_pids = 0;
  bool have_overlap = false;
  // last correction
  bool have_correct = false;
  int corr_pids = 0;
  // last transitions
  long long n_trans_out = 0;
  int trie_cap_log2 = 12;
  long long deep_cap = 0;  // ints of global scratch per thread for merged op stacks deeper than MAXD
  bool reuse_ops = false;  // analyze: the original's op stage builds the paths the corrected overlap reuses
  int64_t reuse_bad_n = -1;  // (n, n_pids) of the last trace whose reuse verdict failed
  int reuse_bad_pids = -1;
  int rmap_logw = 4;  // the last correction's sampled slab-index width (windows per pid, log2)
  unsigned attr_done = 0;  // kernels whose >48 KB dynamic shared memory attribute is set on this ctx's device
  int64_t syn_events = 0, syn_kernels = 0;  // sizes of the last xs_synth_plan
  bool force_lsd = false;  // bucketed sort overflowed on this input: use the LSD path
  xs::OpsState ops;
  // optional per-stage device timing (CUDA events on the launching stream)
  bool prof_on = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t pool_next = 0;
  int prof_active = 0;
  std::vector<int> pend_stage;
  std::vector<cudaEvent_t> pend_a, pend_b;
  double prof_ms[32] = {0};
  long long prof_calls[32] = {0};
  // CUDA-graph replay of sync-free pipeline segments (xs::run_segment)
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    std::vector<int> prof_stage;
    std::vector<cudaEvent_t> prof_a, prof_b;
    long long launches = 0;
    xs::OpsState ops;
    long long generation = 0;  // workspace generation the graph's pointers belong to
    unsigned long long used = 0;  // LRU tick
    std::vector<cudaEvent_t> events;  // timing events owned by this graph
  };
  std::map<std::string, GraphEntry> graphs;
  std::set<std::string> graph_seen, graph_bad;
  std::vector<cudaEvent_t> graph_events;  // events of the capture in progress
  unsigned long long graph_tick = 0;
  long long graph_generation = 0;  // generation the cache was last purged at
  bool capturing = false;
  // speculative overlap pass of xs_analyze: ops selected by the original
  // durations, pass-1 counts kept from the original, k_parent_nodes guarded
  const int64_t* spec_select_dur = nullptr;
  const long long* spec_guard_a = nullptr;
  const long long* spec_guard_b = nullptr;
  bool spec_keep_counts = false;
  // speculative INSTANT pass: operations the correction shrank to zero length
  // get sentinel endpoint keys (sorted to the tail, outside every real path)
  // and the op counts come from the corrected pass 1
  bool spec_zero_sentinel = false;
  long long ws_generation = 0;  // bumped on every workspace reallocation
  cudaStream_t priv_stream = nullptr;
  cudaEvent_t join_in = nullptr, join_out = nullptr;
  // endpoint-sort plan issued ahead of the OPERATION stage (stage_overlap_pre)
  xs::BkPlan bk_plan;
  // concurrent pipeline branches (correct_body): side streams, fork/join
  // events, and the scratch bank of the branch being issued (bank 1 remaps the
  // shared scratch slots -- tile counters, CUB temp, bucket-sort tables -- to
  // private copies so two branches never share them)
  cudaStream_t br_stream[2] = {nullptr, nullptr};
  cudaEvent_t br_fork = nullptr, br_join[2] = {nullptr, nullptr};
  int bank = 0;
  bool skip_ops_reset = false;
  // copy stream of xs_analyze_to_host
  cudaStream_t d2h_stream = nullptr;
  cudaEvent_t d2h_fork = nullptr, d2h_join = nullptr;
  // last union (xs_union / xs_utilization), kept for xs_union_intervals_fetch
  const uint64_t* un_keys = nullptr;
  const int* un_depth = nullptr;
  int64_t un_m = 0;
  int un_tb = 0;
  int64_t un_intervals = -1;
};

namespace xs {
enum Stage : int {
  ST_PASS1 = 0, ST_OPS, ST_TRANS_SORT, ST_TRANS_SCAN, ST_SITE_SORT, ST_QUANTIZE, ST_REMOVAL, ST_REMAP,
  ST_KEYGEN, ST_MAIN_SORT, ST_SWEEP, ST_COMPACT, ST_CORR_FX, ST_NUM
};
cudaEvent_t prof_event(xs_ctx* ctx);
void prof_flush(xs_ctx* ctx);
struct ProfScope {  // records [begin, end) of one stage on stream s when profiling is on
  xs_ctx* c;
  int stage;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  ProfScope(xs_ctx* c_, int st, cudaStream_t s_) : c(c_), stage(st), s(s_) {
    if (c->prof_on) {
      a = prof_event(c);
      record(a);
      c->prof_active++;
    }
  }
  // inside a stream capture a plain record is only a dependency edge: the
  // external flag makes the graph record the event each time it is replayed
  void record(cudaEvent_t e) {
    if (c->capturing) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else cudaEventRecord(e, s);
  }
  void end() {
    if (a) {
      cudaEvent_t b = prof_event(c);
      record(b);
      c->pend_stage.push_back(stage);
      c->pend_a.push_back(a);
      c->pend_b.push_back(b);
      c->prof_active--;
      a = nullptr;
    }
  }
  ~ProfScope() { end(); }
};
}  // namespace xs

namespace xs {

struct Run {
  xs_ctx* c;
  cudaStream_t s;
};

#define XS_TRY(expr)                     \
  do {                                   \
    int _st = (expr);                    \
    if (_st != XS_OK) return _st;        \
  } while (0)

#define XS_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ctx->err = std::string(#expr) + ": " + cudaGetErrorString(_e);                   \
      return XS_CUDA_ERROR;                                                            \
    }                                                                                  \
  } while (0)

// launch bookkeeping: every kernel launch in the library goes through this
#define XS_LAUNCH(ctx, kernel, grid, block, smem, stream, ...)                         \
  do {                                                                                 \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                        \
    (ctx)->launches++;                                                                 \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e != cudaSuccess) {                                                           \
      (ctx)->err = std::string(#kernel) + ": " + cudaGetErrorString(_e);               \
      return XS_CUDA_ERROR;                                                            \
    }                                                                                  \
  } while (0)

// Several small fills as ONE kernel launch: inside a captured graph every
// cudaMemsetAsync is its own node (~5 us of dependency latency each on the
// step's critical path; the look-back kernels alone need two per launch).
struct FillSpec {
  void* p;
  unsigned long long bytes;
  int val;  // byte value
};
constexpr int XS_FILL_MAX = 8;
struct FillArgs {
  FillSpec f[XS_FILL_MAX];
  int n;
};
int fill_many(xs_ctx* ctx, cudaStream_t s, std::initializer_list<FillSpec> specs);
// Small device -> page-locked host copies as ONE kernel storing straight into
// the (unified-address) host buffers: each D2H memcpy costs several us of
// copy-engine latency on the step's tail.  Visible to the host after the
// stream synchronises.
struct CopySpec {
  void* dst;  // page-locked host memory (cudaMallocHost)
  const void* src;
  unsigned long long bytes;  // multiple of 8, both pointers 8-aligned
};
struct CopyArgs {
  CopySpec c[XS_FILL_MAX];
  int n;
};
int to_host_many(xs_ctx* ctx, cudaStream_t s, std::initializer_list<CopySpec> specs);

// grow-only workspace slot
int ws_get(xs_ctx* ctx, int slot, size_t bytes, cudaStream_t s, void** out);
template <class T>
inline int ws(xs_ctx* ctx, int slot, size_t count, cudaStream_t s, T** out) {
  void* p = nullptr;
  int st = ws_get(ctx, slot, count * sizeof(T) + 16, s, &p);
  *out = reinterpret_cast<T*>(p);
  return st;
}

int fetch_stats(xs_ctx* ctx, cudaStream_t s);  // D2H of Stats + sync

// stable radix sorts over [0, bits) (CUB onesweep bring-up backend)
int sort_pairs_u64_u32(xs_ctx* ctx, uint64_t** keys, uint64_t** keys_alt, uint32_t** vals, uint32_t** vals_alt,
                       int64_t n, int bits, cudaStream_t s);
int bucket_sort_pairs(xs_ctx* ctx, uint64_t** keys, uint64_t** keys_alt, uint32_t** vals, uint32_t** vals_alt,
                      int64_t n, int key_bits, cudaStream_t s);
int sort_keys_u64(xs_ctx* ctx, uint64_t** keys, uint64_t** keys_alt, int64_t n, int bits, cudaStream_t s);

// pipeline stages (defined in the .cu files)
struct EventView {  // by value: columns are device pointers; start/dur may be overridden (corrected trace)
  xs_events_t ev;
  const int64_t* start;
  const int64_t* dur;
};

int stage_events_async(xs_ctx* ctx, const EventView& v, cudaStream_t s, bool check_api, const xs_profile_t* prof);
int stage_events(xs_ctx* ctx, const EventView& v, cudaStream_t s, bool need_corr_table, bool check_api,
                 const xs_profile_t* prof);
// (pid, correlation) table: the dangling-correlation rule, plus per-GPU-event
// launch instants when need_start (CORRELATION attribution)
int stage_corr_table(xs_ctx* ctx, const EventView& v, cudaStream_t s, bool need_start);
int stage_ops(xs_ctx* ctx, const EventView& v, cudaStream_t s, bool build_paths);
int stage_ops_paths(xs_ctx* ctx, const EventView& v, cudaStream_t s);
int stage_overlap_pre(xs_ctx* ctx, const EventView& v, cudaStream_t s);
int ops_reuse_check(xs_ctx* ctx, const EventView& v, Stats* verdict, cudaStream_t s);
int ops_with_overlap_pre(xs_ctx* ctx, const EventView& v, int attribution, cudaStream_t w);
int stage_overlap(xs_ctx* ctx, const EventView& v, int attribution, cudaStream_t s);
int stage_transitions(xs_ctx* ctx, const EventView& v, int src_mask, int dst_mask, cudaStream_t s);
int stage_correct(xs_ctx* ctx, const EventView& v, const xs_profile_t* prof, int64_t* out_start,
                  int64_t* out_dur, bool corrected_spans, cudaStream_t s);

inline OpsState& ctx_ops(xs_ctx* c) { return c->ops; }
int trie_setup(xs_ctx* ctx, cudaStream_t s, TrieView* t);

__global__ void k_iota_u32(uint32_t* v, int64_t n);

int run_validate(xs_ctx* ctx, const EventView& v, cudaStream_t s, long long* n_bad);
// run `body` (a sync-free stream of launches) eagerly the first time a key is
// seen, capture it into a CUDA graph the second time, replay it afterwards
int run_segment(xs_ctx* ctx, cudaStream_t s, const std::string& key, bool capturable,
                const std::function<int(cudaStream_t)>& body);
std::string segment_key(xs_ctx* ctx, const char* tag, const void* extra, size_t extra_bytes);
constexpr int XS_CAPTURE_ABORT = 100;
constexpr int XS_RETRY_LSD = 101;  // a bucketed sort overflowed: re-run the call with CUB radix sorts
// runs f; on XS_RETRY_LSD runs it once more with every sort on the LSD path
template <class F>
int with_lsd_retry(xs_ctx* ctx, F&& f) {
  int st = f();
  if (st != XS_RETRY_LSD) return st;
  if (getenv("XS_CHECK_BSORT")) fprintf(stderr, "lsd retry\n");
  const bool prev = ctx->force_lsd;
  ctx->force_lsd = true;
  st = f();
  ctx->force_lsd = prev;
  if (st == XS_RETRY_LSD) {
    ctx->err = "radix sort overflow on the LSD path";
    return XS_UNSUPPORTED;
  }
  return st;
}  // internal: an allocation was needed while capturing
int corrected_total_from_spans(xs_ctx* ctx, cudaStream_t s);
int run_overlap(xs_ctx* ctx, const EventView& v, int attribution, cudaStream_t s);

}  // namespace xs
