#include <atomic>
#include <chrono>
#include <algorithm>
#include <cstdio>
// xs_ctx.cu -- C ABI entry points, workspace and sort plumbing.
#include <cub/device/device_radix_sort.cuh>

#include "xs_engine.cuh"

using namespace xs;

namespace xs {

__global__ void k_fill_many(FillArgs a) {
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (int i = 0; i < a.n; i++) {
    unsigned char* p = (unsigned char*)a.f[i].p;
    const unsigned long long nb = a.f[i].bytes;
    const unsigned v8 = (unsigned)a.f[i].val & 0xFFu;
    const unsigned v32 = v8 * 0x01010101u;
    if (((uintptr_t)p & 15) == 0) {  // 16-byte stores + a byte tail
      const unsigned long long n16 = nb >> 4;
      uint4* q = reinterpret_cast<uint4*>(p);
      for (unsigned long long j = tid; j < n16; j += stride) q[j] = make_uint4(v32, v32, v32, v32);
      for (unsigned long long j = (n16 << 4) + tid; j < nb; j += stride) p[j] = (unsigned char)v8;
    } else if (((uintptr_t)p & 7) == 0 && (nb & 7) == 0) {
      unsigned long long* q = reinterpret_cast<unsigned long long*>(p);
      const unsigned long long v64 = ((unsigned long long)v32 << 32) | v32;
      for (unsigned long long j = tid; j < (nb >> 3); j += stride) q[j] = v64;
    } else {
      for (unsigned long long j = tid; j < nb; j += stride) p[j] = (unsigned char)v8;
    }
  }
}

int fill_many(xs_ctx* ctx, cudaStream_t s, std::initializer_list<FillSpec> specs) {
  FillArgs a{};
  unsigned long long most = 0;
  for (const FillSpec& f : specs) {
    if (!f.p || !f.bytes) continue;
    if (a.n == XS_FILL_MAX) {
      ctx->err = "fill_many: too many regions";
      return XS_BAD_ARGUMENT;
    }
    a.f[a.n++] = f;
    most = f.bytes > most ? f.bytes : most;
  }
  if (!a.n) return XS_OK;
  const unsigned long long blocks = (most / 16 + XS_BLOCK - 1) / XS_BLOCK;
  const int grid = (int)(blocks < 1 ? 1 : (blocks > 148 * 8 ? 148 * 8 : blocks));
  XS_LAUNCH(ctx, k_fill_many, grid, XS_BLOCK, 0, s, a);
  return XS_OK;
}

__global__ void k_copy_many(CopyArgs a) {
  const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (int i = 0; i < a.n; i++) {
    unsigned long long* d = (unsigned long long*)a.c[i].dst;
    const unsigned long long* x = (const unsigned long long*)a.c[i].src;
    for (unsigned long long j = tid; j < (a.c[i].bytes >> 3); j += stride) d[j] = x[j];
  }
}

int to_host_many(xs_ctx* ctx, cudaStream_t s, std::initializer_list<CopySpec> specs) {
  CopyArgs a{};
  unsigned long long most = 0;
  for (const CopySpec& c : specs) {
    if (!c.dst || !c.src || !c.bytes) continue;
    if (a.n == XS_FILL_MAX || (c.bytes & 7) || ((uintptr_t)c.dst & 7) || ((uintptr_t)c.src & 7)) {
      ctx->err = "to_host_many: bad region";
      return XS_BAD_ARGUMENT;
    }
    a.c[a.n++] = c;
    most = c.bytes > most ? c.bytes : most;
  }
  if (!a.n) return XS_OK;
  const unsigned long long blocks = (most / 8 + XS_BLOCK - 1) / XS_BLOCK;
  const int grid = (int)(blocks < 1 ? 1 : (blocks > 148 ? 148 : blocks));
  XS_LAUNCH(ctx, k_copy_many, grid, XS_BLOCK, 0, s, a);
  return XS_OK;
}

int ws_get(xs_ctx* ctx, int slot, size_t bytes, cudaStream_t s, void** out) {
  if (ctx->bank == 1) {  // a concurrent branch's private scratch
    switch (slot) {
      case W_TILE_CTR: slot = W_TILE_CTR_B; break;
      case W_CUB_TEMP: slot = W_CUB_TEMP_B; break;
      case W_BS_COUNTS: slot = W_BS_COUNTS_B; break;
      case W_BS_OFFS: slot = W_BS_OFFS_B; break;
      case W_BS_TAIL: slot = W_BS_TAIL_B; break;
      case W_BS_CHUNK: slot = W_BS_CHUNK_B; break;
      case W_PSCAN_DESC: slot = W_PSCAN_DESC_B; break;
      case W_PSCAN_FLAGS: slot = W_PSCAN_FLAGS_B; break;
      case W_PSCAN_CTR: slot = W_PSCAN_CTR_B; break;
      default: break;
    }
  }
  if (bytes < 256) bytes = 256;
  if (ctx->cap[slot] < bytes) {
    if (ctx->capturing) return XS_CAPTURE_ABORT;  // never allocate inside a graph capture
    static const bool dbg = getenv("XS_DEBUG_GRAPH") != nullptr;
    if (dbg) fprintf(stderr, "[xs ws] slot %d grows %zu -> %zu\n", slot, ctx->cap[slot], bytes);
    ctx->ws_generation++;
    if (ctx->ptr[slot]) XS_CUDA(cudaFreeAsync(ctx->ptr[slot], s));
    size_t nb = bytes + bytes / 4;
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, nb, s);
    if (e != cudaSuccess) {
      ctx->err = std::string("workspace allocation failed: ") + cudaGetErrorString(e);
      ctx->ptr[slot] = nullptr;
      ctx->cap[slot] = 0;
      return XS_NO_MEMORY;
    }
    ctx->ptr[slot] = p;
    ctx->cap[slot] = nb;
  }
  *out = ctx->ptr[slot];
  return XS_OK;
}

int fetch_stats(xs_ctx* ctx, cudaStream_t s) {
  Stats* d = nullptr;
  XS_TRY(ws(ctx, W_STATS, 1, s, &d));
  XS_TRY(to_host_many(ctx, s, {{ctx->h_stats, d, sizeof(Stats)}}));
  XS_CUDA(cudaStreamSynchronize(s));
  if (!ctx->pend_stage.empty()) prof_flush(ctx);
  return XS_OK;
}

// One CTA sorts up to SMALL_SORT_MAX (key, value) pairs in shared memory:
// a bitonic network on (key, input position), so the result is STABLE like
// the radix sorts it stands in for (some callers rely on input order among
// equal keys).  Sentinel keys (>= 2^bits) are larger than every real key.
constexpr int SMALL_SORT_MAX = 8192;

__global__ void __launch_bounds__(1024) k_small_sort(uint64_t* keys, uint32_t* vals, int n, int P) {
  extern __shared__ __align__(16) unsigned char raw[];
  uint64_t* sk = reinterpret_cast<uint64_t*>(raw);
  uint32_t* sv = reinterpret_cast<uint32_t*>(sk + P);
  uint16_t* sp = reinterpret_cast<uint16_t*>(sv + P);
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    sk[i] = i < n ? keys[i] : ~0ull;
    sv[i] = i < n && vals ? vals[i] : 0u;
    sp[i] = (uint16_t)i;
  }
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int x = i ^ j;
        if (x > i) {
          const uint64_t a = sk[i], b = sk[x];
          const uint16_t pa = sp[i], pb = sp[x];
          const bool gt = a > b || (a == b && pa > pb);
          if (gt == ((i & k) == 0)) {
            const uint32_t va = sv[i];
            sk[i] = b, sk[x] = a;
            sp[i] = pb, sp[x] = pa;
            sv[i] = sv[x], sv[x] = va;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    keys[i] = sk[i];
    if (vals) vals[i] = sv[i];
  }
}

static int small_sort(xs_ctx* ctx, uint64_t* keys, uint32_t* vals, int64_t n, cudaStream_t s) {
  int P = 1;
  while (P < n) P <<= 1;
  const int smem = P * 14;
  if (!(ctx->attr_done & 4u)) {  // (per context: a context is bound to one device)
    XS_CUDA(cudaFuncSetAttribute(k_small_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, SMALL_SORT_MAX * 14));
    ctx->attr_done |= 4u;
  }
  XS_LAUNCH(ctx, k_small_sort, 1, 1024, smem, s, keys, vals, (int)n, P);
  return XS_OK;
}

int sort_pairs_u64_u32(xs_ctx* ctx, uint64_t** keys, uint64_t** keys_alt, uint32_t** vals, uint32_t** vals_alt,
                       int64_t n, int bits, cudaStream_t s) {
  if (n > 1 && n <= SMALL_SORT_MAX && !getenv("XS_NO_SMALL_SORT")) return small_sort(ctx, *keys, *vals, n, s);
  if (n <= 1 || bits <= 0) return XS_OK;
  if (bits > 64) bits = 64;
  static const bool no_bsort = getenv("XS_NO_BSORT") != nullptr;  // (debug switch)
  if (!ctx->force_lsd && !no_bsort && n >= 2 * 4096 && n < ((int64_t)1 << 31))
    return bucket_sort_pairs(ctx, keys, keys_alt, vals, vals_alt, n, bits, s);
  cub::DoubleBuffer<uint64_t> k(*keys, *keys_alt);
  cub::DoubleBuffer<uint32_t> v(*vals, *vals_alt);
  size_t temp = 0;
  XS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, k, v, (int)n, 0, bits, s));
  void* t = nullptr;
  XS_TRY(ws_get(ctx, W_CUB_TEMP, temp, s, &t));
  XS_CUDA(cub::DeviceRadixSort::SortPairs(t, temp, k, v, (int)n, 0, bits, s));
  ctx->launches += (bits + 7) / 8 + 1;
  if (k.Current() != *keys) {
    std::swap(*keys, *keys_alt);
  }
  if (v.Current() != *vals) {
    std::swap(*vals, *vals_alt);
  }
  return XS_OK;
}

int sort_keys_u64(xs_ctx* ctx, uint64_t** keys, uint64_t** keys_alt, int64_t n, int bits, cudaStream_t s) {
  if (n <= 1 || bits <= 0) return XS_OK;
  if (bits > 64) bits = 64;
  if (n <= SMALL_SORT_MAX) return small_sort(ctx, *keys, nullptr, n, s);
  if (!ctx->force_lsd && n < ((int64_t)1 << 31)) {  // the bucketed sort, keys only (no value column)
    uint32_t *v = nullptr, *v_alt = nullptr;
    return bucket_sort_pairs(ctx, keys, keys_alt, &v, &v_alt, n, bits, s);
  }
  cub::DoubleBuffer<uint64_t> k(*keys, *keys_alt);
  size_t temp = 0;
  XS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp, k, (int)n, 0, bits, s));
  void* t = nullptr;
  XS_TRY(ws_get(ctx, W_CUB_TEMP, temp, s, &t));
  XS_CUDA(cub::DeviceRadixSort::SortKeys(t, temp, k, (int)n, 0, bits, s));
  ctx->launches += (bits + 7) / 8 + 1;
  if (k.Current() != *keys) std::swap(*keys, *keys_alt);
  return XS_OK;
}

static int run_validate_once(xs_ctx* ctx, const EventView& v, cudaStream_t s, long long* n_bad) {
  int st = stage_events(ctx, v, s, true, false, nullptr);
  if (st == XS_INVALID_TRACE) {
    *n_bad = ctx->h_stats->n_bad;
    return XS_OK;
  }
  XS_TRY(st);
  XS_TRY(stage_ops(ctx, v, s, false));
  XS_TRY(fetch_stats(ctx, s));
  if (ctx->h_stats->pad[3] && !ctx->force_lsd) return XS_RETRY_LSD;
  *n_bad = ctx->h_stats->n_bad;
  return XS_OK;
}

int run_validate(xs_ctx* ctx, const EventView& v, cudaStream_t s, long long* n_bad) {
  return with_lsd_retry(ctx, [&] { return run_validate_once(ctx, v, s, n_bad); });
}

int run_overlap(xs_ctx* ctx, const EventView& v, int attribution, cudaStream_t s) {
  ctx->have_overlap = false;
  struct LsdRestore {  // an LSD retry applies to this call only, whatever the exit
    xs_ctx* c;
    bool prev;
    ~LsdRestore() { c->force_lsd = prev; }
  } lsd_restore{ctx, ctx->force_lsd};
  // pass 1 (+ its sync: sizes and per-event rule violations)
  XS_TRY(stage_events(ctx, v, s, false, false, nullptr));
  for (int attempt = 0; attempt < 8; attempt++) {
    // sync-free segment: correlation table, op paths, sort + sweep + compact
    std::string key = segment_key(ctx, "overlap", &v, sizeof(v));
    key.append(reinterpret_cast<const char*>(&attribution), sizeof(attribution));
    XS_TRY(run_segment(ctx, s, key, true, [&](cudaStream_t w) -> int {
      XS_TRY(stage_corr_table(ctx, v, w, attribution == 1));
      XS_TRY(ops_with_overlap_pre(ctx, v, attribution, w));
      return stage_overlap(ctx, v, attribution, w);
    }));
    ctx->res_pids = v.ev.n_pids;
    XS_TRY(fetch_stats(ctx, s));
    if (getenv("XS_DEBUG_STATS")) {  // developer diagnostics
      const Stats& h = *ctx->h_stats;
      fprintf(stderr, "xs_overlap attempt %d: bad %lld nz %lld ops_nz %lld api_corr %lld gpu_corr %lld span %lld "
              "depth %lld full %lld multi %lld depth_ovf %lld lsd %lld nodes %lld\n", attempt, h.n_bad, h.n_nonzero,
              h.n_ops_nz, h.n_api_corr, h.n_gpu_corr, h.max_span, h.max_depth, h.table_full, h.multi_op_pids,
              h.depth_overflow, h.pad[3], h.pad[0]);
    }
    // a bucket overflowed a chunk: every verdict of this attempt (nesting
    // included) came from an unsorted stream -- redo the call via the LSD sort
    if (ctx->h_stats->pad[3] && !ctx->force_lsd) {
      ctx->force_lsd = true;
      // pass 1 found no violation (else stage_events returned): clear what
      // the failed attempt's nesting check counted
      XS_CUDA(cudaMemsetAsync(&((Stats*)ctx->ptr[W_STATS])->n_bad, 0, sizeof(long long), s));
      continue;
    }
    if (ctx->h_stats->n_bad) return XS_INVALID_TRACE;
    if (ctx->h_stats->depth_overflow) {
      // merged multi-tid stacks deeper than the register-sized merge: re-run
      // with a global scratch that holds the deepest one (no depth limit)
      long long need = ctx->h_stats->pad[7];
      long long cap = 1024;
      while (cap < need) cap <<= 1;
      if (cap <= ctx->deep_cap) {
        ctx->err = "deep operation-path scratch could not be sized";
        return XS_NO_MEMORY;
      }
      ctx->deep_cap = cap;
      continue;
    }
    if (!ctx->h_stats->table_full) {
      ctx->have_overlap = true;
      ctx->n_cells = ctx->h_stats->pad[4];
      ctx->n_nodes = ctx->h_stats->pad[0] > 0 ? (int)ctx->h_stats->pad[0] : 1;  // trie nodes allocated
      return XS_OK;
    }
    {  // the path trie ran out of slots: jump to a capacity that holds a node
       // per op segment (the distinct paths are at most that many)
      const int need = bits_for((uint64_t)(4 * ctx->h_stats->n_ops_nz + 4)) + 1;
      ctx->trie_cap_log2 = std::max(ctx->trie_cap_log2 + 2, std::min(need, 30));
    }
  }
  ctx->err = "path table could not be sized";
  return XS_NO_MEMORY;
}

static int ensure_branches(xs_ctx* ctx) {
  if (!ctx->br_fork) {
    for (int b = 0; b < 2; b++) {
      XS_CUDA(cudaStreamCreateWithFlags(&ctx->br_stream[b], cudaStreamNonBlocking));
      XS_CUDA(cudaEventCreateWithFlags(&ctx->br_join[b], cudaEventDisableTiming));
    }
    XS_CUDA(cudaEventCreateWithFlags(&ctx->br_fork, cudaEventDisableTiming));
  }
  return XS_OK;
}

// stage_ops (paths) on a side branch while the INSTANT endpoint sort's first
// phase (histogram, offsets, chunk table, scatter) runs on w: the two only
// meet in the sweep kernel
int ops_with_overlap_pre(xs_ctx* ctx, const EventView& v, int attribution, cudaStream_t w) {
  static const bool serial = getenv("XS_NO_BRANCHES") != nullptr;  // (A/B switch)
  if (attribution != 0 || ctx->force_lsd || serial) return stage_ops(ctx, v, w, true);
  XS_TRY(ensure_branches(ctx));
  XS_CUDA(cudaEventRecord(ctx->br_fork, w));
  XS_CUDA(cudaStreamWaitEvent(ctx->br_stream[1], ctx->br_fork, 0));
  struct Join {
    xs_ctx* c;
    cudaStream_t w;
    ~Join() {
      c->bank = 0;
      cudaEventRecord(c->br_join[1], c->br_stream[1]);
      cudaStreamWaitEvent(w, c->br_join[1], 0);
    }
  } join{ctx, w};
  XS_TRY(stage_ops(ctx, v, ctx->br_stream[1], true));
  ctx->bank = 1;
  return stage_overlap_pre(ctx, v, w);
}

}  // namespace xs

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* xs_status_str(int st) {
  switch (st) {
    case XS_OK: return "ok";
    case XS_INVALID_TRACE: return "invalid trace";
    case XS_UNCALIBRATED: return "uncalibrated hook";
    case XS_CUDA_ERROR: return "cuda error";
    case XS_BAD_ARGUMENT: return "bad argument";
    case XS_UNSUPPORTED: return "unsupported input";
    case XS_NO_MEMORY: return "out of device memory";
    default: return "unknown status";
  }
}

int xs_version(void) { return 1; }

const char* xs_last_error(xs_ctx_t* ctx) { return ctx ? ctx->err.c_str() : ""; }

int xs_ctx_create(int device, xs_ctx_t** out) {
  if (!out) return XS_BAD_ARGUMENT;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return XS_CUDA_ERROR;
  xs_ctx* c = new xs_ctx();
  c->device = device;
  c->ptr.assign(W_NUM_SLOTS, nullptr);
  c->cap.assign(W_NUM_SLOTS, 0);
  e = cudaMallocHost(&c->h_stats, 2 * sizeof(Stats) + 4 * sizeof(int64_t));
  if (e != cudaSuccess) {
    delete c;
    return XS_CUDA_ERROR;
  }
  memset(c->h_stats, 0, 2 * sizeof(Stats) + 4 * sizeof(int64_t));
  c->h_totals = reinterpret_cast<int64_t*>(c->h_stats + 2);
  *out = c;
  return XS_OK;
}

void xs_ctx_destroy(xs_ctx_t* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (auto& kv : ctx->graphs) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    for (cudaEvent_t e : kv.second.events) cudaEventDestroy(e);
  }
  if (ctx->priv_stream) cudaStreamDestroy(ctx->priv_stream);
  for (int b = 0; b < 2; b++) {
    if (ctx->br_stream[b]) cudaStreamDestroy(ctx->br_stream[b]);
    if (ctx->br_join[b]) cudaEventDestroy(ctx->br_join[b]);
  }
  if (ctx->br_fork) cudaEventDestroy(ctx->br_fork);
  if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
  if (ctx->d2h_fork) cudaEventDestroy(ctx->d2h_fork);
  if (ctx->d2h_join) cudaEventDestroy(ctx->d2h_join);
  if (ctx->join_in) cudaEventDestroy(ctx->join_in);
  if (ctx->join_out) cudaEventDestroy(ctx->join_out);
  for (cudaEvent_t e : ctx->graph_events) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  for (void* p : ctx->ptr)
    if (p) cudaFree(p);
  if (ctx->h_stats) cudaFreeHost(ctx->h_stats);
  if (ctx->h_report) cudaFreeHost(ctx->h_report);
  delete ctx;
}

int64_t xs_ctx_workspace_bytes(xs_ctx_t* ctx) {
  int64_t t = 0;
  for (size_t b : ctx->cap) t += (int64_t)b;
  return t;
}

int64_t xs_launch_count(xs_ctx_t* ctx) { return ctx ? ctx->launches : 0; }

static int check_events(xs_ctx_t* ctx, const xs_events_t* ev) {
  if (!ctx || !ev) return XS_BAD_ARGUMENT;
  if (ev->n < 0 || ev->n > (int64_t)1 << 30) {
    ctx->err = "event count out of range (0 .. 2^30 per call)";
    return XS_BAD_ARGUMENT;
  }
  if (ev->n > 0 && (!ev->start || !ev->dur || !ev->pid || !ev->tid || !ev->cat || !ev->name || !ev->corr ||
                    !ev->has_corr || !ev->pid_has_meta || !ev->group_pid)) {
    ctx->err = "null column";
    return XS_BAD_ARGUMENT;
  }
  return XS_OK;
}

int xs_validate(xs_ctx_t* ctx, const xs_events_t* ev, int64_t* n_bad, xs_stream_t stream) {
  XS_TRY(check_events(ctx, ev));
  cudaSetDevice(ctx->device);
  EventView v{*ev, ev->start, ev->dur};
  long long b = 0;
  XS_TRY(run_validate(ctx, v, (cudaStream_t)stream, &b));
  *n_bad = b;
  return XS_OK;
}

int xs_overlap(xs_ctx_t* ctx, const xs_events_t* ev, int attribution, xs_stream_t stream) {
  XS_TRY(check_events(ctx, ev));
  if (attribution != 0 && attribution != 1) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  EventView v{*ev, ev->start, ev->dur};
  return run_overlap(ctx, v, attribution, (cudaStream_t)stream);
}

int xs_overlap_info(xs_ctx_t* ctx, xs_overlap_info_t* info) {
  if (!ctx || !info || !ctx->have_overlap) return XS_BAD_ARGUMENT;
  info->n_cells = ctx->n_cells;
  info->n_nodes = ctx->n_nodes;
  info->n_pids = ctx->res_pids;
  return XS_OK;
}

int xs_overlap_fetch(xs_ctx_t* ctx, int32_t* cell_pid, int32_t* cell_node, int32_t* cell_mask, int64_t* cell_ns,
                     int32_t* node_parent, int32_t* node_name, int64_t* span_lo, int64_t* span_hi,
                     int64_t* tracked, uint8_t* has_events, xs_stream_t stream) {
  if (!ctx || !ctx->have_overlap) return XS_BAD_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  auto cp = [&](void* dst, int slot, size_t bytes) -> int {
    if (!dst || bytes == 0) return XS_OK;
    XS_CUDA(cudaMemcpyAsync(dst, ctx->ptr[slot], bytes, cudaMemcpyDeviceToHost, s));
    return XS_OK;
  };
  size_t nc = (size_t)ctx->n_cells, nn = (size_t)ctx->n_nodes, np = (size_t)ctx->res_pids;
  XS_TRY(cp(cell_pid, W_CELL_PID, nc * 4));
  XS_TRY(cp(cell_node, W_CELL_NODE, nc * 4));
  XS_TRY(cp(cell_mask, W_CELL_MASK, nc * 4));
  XS_TRY(cp(cell_ns, W_CELL_NS, nc * 8));
  XS_TRY(cp(node_parent, W_TRIE_PARENT, nn * 4));
  XS_TRY(cp(node_name, W_TRIE_NAME, nn * 4));
  XS_TRY(cp(span_lo, W_SPAN_LO, np * 8));
  XS_TRY(cp(span_hi, W_SPAN_HI, np * 8));
  XS_TRY(cp(tracked, W_TRACKED, np * 8));
  std::vector<int64_t> lo_tmp;  // has_events derives from the span starts: one sync for everything
  const int64_t* lo = span_lo;
  if (has_events && np && !span_lo) {
    lo_tmp.resize(np);
    XS_TRY(cp(lo_tmp.data(), W_SPAN_LO, np * 8));
    lo = lo_tmp.data();
  }
  XS_CUDA(cudaStreamSynchronize(s));
  if (has_events)
    for (size_t p = 0; p < np; p++) has_events[p] = lo[p] != INT64_MAX;
  return XS_OK;
}

static int correct_branches(xs_ctx* ctx, const EventView& v, cudaStream_t w) {
  // three independent latency-bound stages run as concurrent branches (graph
  // branches when captured): the correlation table, the OPERATION nesting
  // check (part of require_valid) and the wrapper-transition sites; the
  // correction proper joins them
  XS_TRY(ensure_branches(ctx));
  {  // flags the branches raise start clear before they fork
    Stats* stp = (Stats*)ctx->ptr[W_STATS];
    XS_TRY(fill_many(ctx, w, {{&stp->table_full, sizeof(long long), 0}, {&stp->depth_overflow, sizeof(long long), 0},
                              {&stp->pad[3], sizeof(long long), 0},
                              {&stp->pad[7], 2 * sizeof(long long), 0}}));  // (deep-path need, reuse verdict)
  }
  XS_CUDA(cudaEventRecord(ctx->br_fork, w));
  XS_CUDA(cudaStreamWaitEvent(ctx->br_stream[0], ctx->br_fork, 0));
  XS_CUDA(cudaStreamWaitEvent(ctx->br_stream[1], ctx->br_fork, 0));
  struct Join {  // branches rejoin w on every exit (a capture must end joined)
    xs_ctx* c;
    cudaStream_t w;
    ~Join() {
      c->bank = 0;
      c->skip_ops_reset = false;
      for (int b = 0; b < 2; b++) {
        cudaEventRecord(c->br_join[b], c->br_stream[b]);
        cudaStreamWaitEvent(w, c->br_join[b], 0);
      }
    }
  };
  {
    Join join{ctx, w};
    XS_TRY(stage_corr_table(ctx, v, ctx->br_stream[0], false));
    ctx->skip_ops_reset = true;
    // OPERATION nesting is part of require_valid (with reuse_ops, the paths
    // the corrected trace's overlap pass will use are built from this
    // stage's sorted stream concurrently with the correction: correct_paths)
    XS_TRY(stage_ops(ctx, v, ctx->br_stream[1], false));
    ctx->skip_ops_reset = false;
    ctx->bank = 1;
    XS_TRY(stage_transitions(ctx, v, 0x2 /*HIGH_LEVEL*/, 0xC /*BACKEND|SIMULATOR*/, w));
  }
  return XS_OK;
}

// stage_correct on w; with reuse_ops the original trace's op paths are built
// on a side branch meanwhile (private scratch bank), joined before the end
static int correct_with_paths(xs_ctx* ctx, const EventView& v, const xs_profile_t* prof, int64_t* out_start,
                              int64_t* out_dur, cudaStream_t w) {
  if (!ctx->reuse_ops) return stage_correct(ctx, v, prof, out_start, out_dur, false, w);
  XS_TRY(ensure_branches(ctx));
  XS_CUDA(cudaEventRecord(ctx->br_fork, w));
  XS_CUDA(cudaStreamWaitEvent(ctx->br_stream[1], ctx->br_fork, 0));
  struct Join {
    xs_ctx* c;
    cudaStream_t w;
    ~Join() {
      c->bank = 0;
      cudaEventRecord(c->br_join[1], c->br_stream[1]);
      cudaStreamWaitEvent(w, c->br_join[1], 0);
    }
  } join{ctx, w};
  ctx->bank = 1;
  XS_TRY(stage_ops_paths(ctx, v, ctx->br_stream[1]));
  ctx->bank = 0;
  return stage_correct(ctx, v, prof, out_start, out_dur, false, w);
}

static int correct_body(xs_ctx* ctx, const EventView& v, const xs_profile_t* prof, int64_t* out_start,
                        int64_t* out_dur, bool corrected_spans, cudaStream_t w) {
  XS_TRY(correct_branches(ctx, v, w));
  return stage_correct(ctx, v, prof, out_start, out_dur, corrected_spans, w);
}

static int correct_verdict(xs_ctx* ctx, const Stats* h, int64_t* bad_event) {
  if (h->n_bad) return XS_INVALID_TRACE;  // require_valid runs first in the reference
  if (h->bad_api != INT64_MAX) {
    if (bad_event) *bad_event = h->bad_api;
    return XS_UNCALIBRATED;
  }
  ctx->have_correct = true;
  return XS_OK;
}

// queue the D2H of what xs_correct_report returns, to land with the next sync
// the report's host buffer, grown to the current pid count
static int report_buffer(xs_ctx* ctx, size_t* bytes) {
  const size_t b = (size_t)ctx->corr_pids * 4 * 8;
  *bytes = b;
  if (2 * b > ctx->h_report_cap) {
    if (ctx->h_report) XS_CUDA(cudaFreeHost(ctx->h_report));
    ctx->h_report = nullptr;
    ctx->h_report_cap = 0;
    XS_CUDA(cudaMallocHost(&ctx->h_report, 2 * b));
    ctx->h_report_cap = 2 * b;
  }
  return XS_OK;
}

static int prefetch_report(xs_ctx* ctx, cudaStream_t s) {
  size_t b = 0;
  XS_TRY(report_buffer(ctx, &b));
  return to_host_many(ctx, s, {{ctx->h_totals, ctx->ptr[W_CORR_TOTALS], 4 * 8},
                               {ctx->h_report, ctx->ptr[W_REMOVED], b},
                               {ctx->h_report + b / 8, ctx->ptr[W_SHORTFALL], b}});
}

// Pass 1 + its statistics read-back as one graph segment (six eager launches
// left the device waiting on the host for ~18 us at 1M events), then the
// call's one sync: sizes; per-event rule violations stop here.
static int pass1_sync(xs_ctx* ctx, const EventView& v, const xs_profile_t* prof, cudaStream_t s) {
  std::string k1("pass1");
  k1.push_back('\0');
  k1.append(reinterpret_cast<const char*>(&v), sizeof(v));
  k1.append(reinterpret_cast<const char*>(&prof->has_internal), sizeof(prof->has_internal));
  XS_TRY(run_segment(ctx, s, k1, true, [&](cudaStream_t w) -> int {
    XS_TRY(stage_events_async(ctx, v, w, true, prof));
    Stats* d = nullptr;
    XS_TRY(ws(ctx, W_STATS, 1, w, &d));
    return to_host_many(ctx, w, {{ctx->h_stats, d, sizeof(Stats)}});
  }));
  XS_CUDA(cudaStreamSynchronize(s));
  if (!ctx->pend_stage.empty()) prof_flush(ctx);
  return ctx->h_stats->n_bad ? XS_INVALID_TRACE : XS_OK;
}

static int correct_once(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int64_t* out_start,
                          int64_t* out_dur, int64_t* bad_event, cudaStream_t s, bool corrected_spans) {
  ctx->have_correct = false;
  if (bad_event) *bad_event = -1;
  if (!prof || !prof->L || !prof->frac || (prof->words != 1 && prof->words != 2 && prof->words != 4 && prof->words != 8))
    return XS_BAD_ARGUMENT;
  if (ev->n > 0 && (!out_start || !out_dur)) return XS_BAD_ARGUMENT;
  EventView v{*ev, ev->start, ev->dur};
  XS_TRY(pass1_sync(ctx, v, prof, s));
  // the pipeline is safe on a trace whose nesting / correlations / API names
  // turn out bad, so the verdict is read once, after this sync-free segment
  std::string key = segment_key(ctx, "correct", &v, sizeof(v));
  key.append(reinterpret_cast<const char*>(prof), sizeof(*prof));
  key.append(reinterpret_cast<const char*>(&out_start), sizeof(out_start));
  key.append(reinterpret_cast<const char*>(&out_dur), sizeof(out_dur));
  key.push_back(corrected_spans ? 1 : 0);
  XS_TRY(run_segment(ctx, s, key, true, [&](cudaStream_t w) -> int {
    return correct_body(ctx, v, prof, out_start, out_dur, corrected_spans, w);
  }));
  ctx->corr_pids = v.ev.n_pids;
  XS_TRY(prefetch_report(ctx, s));
  XS_TRY(fetch_stats(ctx, s));
  if (ctx->h_stats->pad[3] && !ctx->force_lsd) return XS_RETRY_LSD;  // (before the verdict: order matters to it)
  return correct_verdict(ctx, ctx->h_stats, bad_event);
}

int xs_correct(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int64_t* out_start_dev,
               int64_t* out_dur_dev, int64_t* bad_event, xs_stream_t stream) {
  XS_TRY(check_events(ctx, ev));
  cudaSetDevice(ctx->device);
  return with_lsd_retry(ctx, [&] {
    return correct_once(ctx, ev, prof, out_start_dev, out_dur_dev, bad_event, (cudaStream_t)stream, true);
  });
}

struct SpecScope {  // speculative-pass switches, cleared on every exit path
  xs_ctx* c;
  SpecScope(xs_ctx* c_, const int64_t* dur, const long long* a, const long long* b) : c(c_) {
    c->spec_select_dur = dur;
    c->spec_guard_a = a;
    c->spec_guard_b = b;
    c->spec_keep_counts = true;
  }
  ~SpecScope() {
    c->spec_select_dur = nullptr;
    c->spec_guard_a = c->spec_guard_b = nullptr;
    c->spec_keep_counts = false;
    c->spec_zero_sentinel = false;
  }
};

// correct_trace followed by compute_overlap of the corrected trace.  The
// corrected trace has the original's events, categories, pids and threads, so
// its overlap pass is launched speculatively in the same sync-free segment as
// the correction, sized by the original's pass-1 statistics; the corrected
// trace's own statistics come back with the segment's single sync and any
// difference that matters for sizing (an interval shrunk to zero length, a
// retry flag) sends the overlap pass through the ordinary path instead.
static int analyze_once(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int attribution,
                        int64_t* out_start_dev, int64_t* out_dur_dev, int64_t* out_start_host,
                        int64_t* out_dur_host, int64_t* bad_event, cudaStream_t s);

int xs_analyze(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int attribution,
               int64_t* out_start_dev, int64_t* out_dur_dev, int64_t* bad_event, xs_stream_t stream) {
  XS_TRY(check_events(ctx, ev));
  if (attribution != 0 && attribution != 1) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  return with_lsd_retry(ctx, [&] {
    return analyze_once(ctx, ev, prof, attribution, out_start_dev, out_dur_dev, nullptr, nullptr, bad_event,
                        (cudaStream_t)stream);
  });
}

static int ensure_d2h(xs_ctx* ctx) {
  if (!ctx->d2h_stream) {
    XS_CUDA(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
    XS_CUDA(cudaEventCreateWithFlags(&ctx->d2h_fork, cudaEventDisableTiming));
    XS_CUDA(cudaEventCreateWithFlags(&ctx->d2h_join, cudaEventDisableTiming));
  }
  return XS_OK;
}

int xs_analyze_to_host(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int attribution,
                       int64_t* out_start_dev, int64_t* out_dur_dev, int64_t* out_start_host, int64_t* out_dur_host,
                       int64_t* bad_event, xs_stream_t stream) {
  XS_TRY(check_events(ctx, ev));
  if (attribution != 0 && attribution != 1) return XS_BAD_ARGUMENT;
  if (ev->n > 0 && (!out_start_host || !out_dur_host)) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  XS_TRY(ensure_d2h(ctx));
  const int st = with_lsd_retry(ctx, [&] {
    return analyze_once(ctx, ev, prof, attribution, out_start_dev, out_dur_dev, out_start_host, out_dur_host,
                        bad_event, (cudaStream_t)stream);
  });
  if (ev->n > 0) XS_CUDA(cudaEventSynchronize(ctx->d2h_join));  // (host buffers complete on return)
  return st;
}

int xs_analyze_to_host_async(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int attribution,
                             int64_t* out_start_dev, int64_t* out_dur_dev, int64_t* out_start_host,
                             int64_t* out_dur_host, int64_t* bad_event, xs_stream_t stream) {
  XS_TRY(check_events(ctx, ev));
  if (attribution != 0 && attribution != 1) return XS_BAD_ARGUMENT;
  if (ev->n > 0 && (!out_start_host || !out_dur_host)) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  XS_TRY(ensure_d2h(ctx));
  return with_lsd_retry(ctx, [&] {
    return analyze_once(ctx, ev, prof, attribution, out_start_dev, out_dur_dev, out_start_host, out_dur_host,
                        bad_event, (cudaStream_t)stream);
  });
}

int xs_host_copy_wait(xs_ctx_t* ctx) {
  if (!ctx) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  if (ctx->d2h_join) XS_CUDA(cudaEventSynchronize(ctx->d2h_join));
  return XS_OK;
}

static int analyze_once(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int attribution,
                        int64_t* out_start_dev, int64_t* out_dur_dev, int64_t* out_start_host,
                        int64_t* out_dur_host, int64_t* bad_event, cudaStream_t s) {
  ctx->have_correct = false;
  ctx->have_overlap = false;
  if (bad_event) *bad_event = -1;
  if (!prof || !prof->L || !prof->frac || (prof->words != 1 && prof->words != 2 && prof->words != 4 && prof->words != 8))
    return XS_BAD_ARGUMENT;
  if (ev->n > 0 && (!out_start_dev || !out_dur_dev)) return XS_BAD_ARGUMENT;
  EventView v{*ev, ev->start, ev->dur};
  EventView vc{*ev, out_start_dev, out_dur_dev};
  static const bool host_timing = getenv("XS_HOST_TIMING") != nullptr;  // (developer diagnostics)
  const auto ht0 = std::chrono::steady_clock::now();
  XS_TRY(pass1_sync(ctx, v, prof, s));
  const auto ht1 = std::chrono::steady_clock::now();
  const Stats orig = *ctx->h_stats;
  Stats* st = nullptr;
  Stats* saved = nullptr;
  XS_TRY(ws(ctx, W_STATS, 1, s, &st));
  XS_TRY(ws(ctx, W_STATS_SAVE, 1, s, &saved));
  const bool spec = !ctx->force_lsd && !getenv("XS_NO_SPECULATE");  // (the env switch is for tests)
  const bool no_reuse = getenv("XS_NO_REUSE_OPS") != nullptr;  // (A/B and test switch)
  struct ReuseScope {
    xs_ctx* c;
    ~ReuseScope() { c->reuse_ops = false; }
  } reuse_scope{ctx};
  // a trace whose removal map collapsed op endpoints once (the overlap pass
  // was redone) does not try the reuse again: the same trace would pay the
  // redo on every call
  ctx->reuse_ops = spec && attribution == 0 && !no_reuse && !(ev->n == ctx->reuse_bad_n && ev->n_pids == ctx->reuse_bad_pids);
  std::string key = segment_key(ctx, "analyze", &v, sizeof(v));
  key.append(reinterpret_cast<const char*>(prof), sizeof(*prof));
  key.append(reinterpret_cast<const char*>(&vc), sizeof(vc));
  key.append(reinterpret_cast<const char*>(&attribution), sizeof(attribution));
  key.push_back(spec ? 1 : 0);
  key.push_back(ctx->reuse_ops ? 1 : 0);
  key.append(reinterpret_cast<const char*>(&out_start_host), sizeof(out_start_host));
  key.append(reinterpret_cast<const char*>(&out_dur_host), sizeof(out_dur_host));
  const bool to_host = out_start_host && ev->n > 0;
  auto spec_body = [&](cudaStream_t w) -> int {
    XS_CUDA(cudaMemcpyAsync(saved, st, sizeof(Stats), cudaMemcpyDeviceToDevice, w));
    // INSTANT: ops shrunk to zero length are excluded by sentinel keys, so the
    // pass stays valid; CORRELATION keeps the guard (discard and redo)
    SpecScope sp(ctx, ev->dur, attribution == 1 ? &st->n_ops_nz : nullptr,
                 attribution == 1 ? &saved->n_ops_nz : nullptr);
    ctx->spec_zero_sentinel = attribution == 0;
    // the reuse verdict (is the removal map strictly increasing on the op
    // endpoints?) runs on a side branch: it is only read after the final sync
    struct CheckJoin {
      xs_ctx* c;
      cudaStream_t w;
      bool on;
      ~CheckJoin() {
        if (!on) return;
        cudaEventRecord(c->br_join[0], c->br_stream[0]);
        cudaStreamWaitEvent(w, c->br_join[0], 0);
      }
    } check_join{ctx, w, ctx->reuse_ops};
    if (ctx->reuse_ops) {
      XS_CUDA(cudaEventRecord(ctx->br_fork, w));
      XS_CUDA(cudaStreamWaitEvent(ctx->br_stream[0], ctx->br_fork, 0));
      XS_TRY(ops_reuse_check(ctx, v, saved, ctx->br_stream[0]));  // (into the correction's saved statistics)
    }
    XS_TRY(stage_events_async(ctx, vc, w, false, nullptr));
    // correlations are untouched by the correction: the original's dangling
    // check stands, and only CORRELATION attribution needs launch instants
    if (attribution == 1) XS_TRY(stage_corr_table(ctx, vc, w, true));
    if (ctx->reuse_ops) XS_TRY(stage_overlap_pre(ctx, vc, w));  // paths: the original's (checked below)
    else XS_TRY(ops_with_overlap_pre(ctx, vc, attribution, w));
    XS_TRY(stage_overlap(ctx, vc, attribution, w));
    ctx->res_pids = ev->n_pids;
    return corrected_total_from_spans(ctx, w);
  };
  const auto ht2 = std::chrono::steady_clock::now();
  // Three graph segments launched back to back: a graph's host launch cost
  // grows with its node count (~40 us for the whole step at config 2), and
  // the device starts the first segment while the host submits the rest.
  XS_TRY(run_segment(ctx, s, key + "B", true, [&](cudaStream_t w) -> int { return correct_branches(ctx, v, w); }));
  const auto ht3 = std::chrono::steady_clock::now();
  XS_TRY(run_segment(ctx, s, key + "C", true, [&](cudaStream_t w) -> int {
    return correct_with_paths(ctx, v, prof, out_start_dev, out_dur_dev, w);
  }));
  if (!to_host) {
    if (spec) XS_TRY(run_segment(ctx, s, key + "O", true, spec_body));
  } else {
    // the corrected columns are final after the second segment: their D2H on
    // the copy stream overlaps the overlap pass -- and, for
    // xs_analyze_to_host_async, the caller's next call
    XS_CUDA(cudaEventRecord(ctx->d2h_fork, s));
    XS_CUDA(cudaStreamWaitEvent(ctx->d2h_stream, ctx->d2h_fork, 0));
    XS_CUDA(cudaMemcpyAsync(out_start_host, out_start_dev, ev->n * 8, cudaMemcpyDeviceToHost, ctx->d2h_stream));
    XS_CUDA(cudaMemcpyAsync(out_dur_host, out_dur_dev, ev->n * 8, cudaMemcpyDeviceToHost, ctx->d2h_stream));
    XS_CUDA(cudaEventRecord(ctx->d2h_join, ctx->d2h_stream));
    if (spec) XS_TRY(run_segment(ctx, s, key + "O", true, spec_body));
  }
  if (host_timing) {
    const auto ht4 = std::chrono::steady_clock::now();
    auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
    fprintf(stderr, "[xs host] pass1+sync %.1f us, key %.1f us, first segment launch %.1f us, all launches %.1f us\n",
            us(ht0, ht1), us(ht1, ht2), us(ht2, ht3), us(ht2, ht4));
  }
  ctx->corr_pids = ev->n_pids;
  {  // every small result in one copy kernel, one sync
    size_t b = 0;
    XS_TRY(report_buffer(ctx, &b));
    XS_TRY(to_host_many(ctx, s, {{ctx->h_stats + 1, spec ? saved : nullptr, sizeof(Stats)},
                                 {ctx->h_totals, ctx->ptr[W_CORR_TOTALS], 4 * 8},
                                 {ctx->h_report, ctx->ptr[W_REMOVED], b},
                                 {ctx->h_report + b / 8, ctx->ptr[W_SHORTFALL], b},
                                 {ctx->h_stats, ctx->ptr[W_STATS], sizeof(Stats)}}));
    XS_CUDA(cudaStreamSynchronize(s));
    if (!ctx->pend_stage.empty()) prof_flush(ctx);
  }
  const Stats* hc = spec ? ctx->h_stats + 1 : ctx->h_stats;  // the correction part's statistics
  if (hc->pad[3] && !ctx->force_lsd) return XS_RETRY_LSD;
  XS_TRY(correct_verdict(ctx, hc, bad_event));
  if (spec) {
    const Stats& c = *ctx->h_stats;  // the corrected trace's pass 1 + the overlap flags
    // everything the pass was sized by (the original's pass 1) bounds the
    // corrected trace's counts; INSTANT tolerates ops shrunk to zero length
    const bool shrink_ok = attribution == 0;
    // reused op stage: the original's path flags and the strictness verdict
    const bool reuse_ok = !ctx->reuse_ops || (!hc->pad[8] && !hc->table_full && !hc->depth_overflow);
    bool same = reuse_ok && c.n_bad == 0 && !c.table_full && !c.depth_overflow && !c.pad[3] &&
                (shrink_ok ? c.n_ops_nz <= orig.n_ops_nz : c.n_ops_nz == orig.n_ops_nz) &&
                (shrink_ok ? c.n_nonzero <= orig.n_nonzero : c.n_nonzero == orig.n_nonzero) &&
                (shrink_ok ? c.multi_op_pids <= orig.multi_op_pids : c.multi_op_pids == orig.multi_op_pids) &&
                c.n_api_corr == orig.n_api_corr && c.n_gpu_corr == orig.n_gpu_corr && c.max_span <= orig.max_span;
    for (int k = 0; k < 8; k++) same = same && (shrink_ok ? c.cat_nz[k] <= orig.cat_nz[k] : c.cat_nz[k] == orig.cat_nz[k]);
    if (getenv("XS_DEBUG_STATS"))
      fprintf(stderr, "xs_analyze speculative overlap %s: bad %lld full %lld depth_ovf %lld lsd %lld\n",
              same ? "kept" : "redone", c.n_bad, c.table_full, c.depth_overflow, c.pad[3]);
    if (ctx->reuse_ops && !reuse_ok) {
      ctx->reuse_bad_n = ev->n;
      ctx->reuse_bad_pids = ev->n_pids;
    }
    if (same) {
      ctx->have_overlap = true;
      ctx->n_cells = c.pad[4];
      ctx->n_nodes = c.pad[0] > 0 ? (int)c.pad[0] : 1;  // trie nodes allocated
      return XS_OK;
    }
  }
  int st2 = run_overlap(ctx, vc, attribution, s);
  if (st2 != XS_OK) return st2;
  // corrected_total_ns = sum of the corrected pid spans the overlap pass computed
  XS_TRY(corrected_total_from_spans(ctx, s));
  XS_CUDA(cudaMemcpyAsync(ctx->h_totals, ctx->ptr[W_CORR_TOTALS], 4 * 8, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaStreamSynchronize(s));
  return XS_OK;
}

int xs_correct_report(xs_ctx_t* ctx, xs_correct_info_t* info, int64_t* removed, int64_t* shortfall,
                      xs_stream_t stream) {
  (void)stream;  // everything arrived with the correction's own final sync
  if (!ctx || !ctx->have_correct) return XS_BAD_ARGUMENT;
  if (info) {  // [original_total, corrected_total, n_sites, n_slabs] written by the pipeline
    info->original_total = ctx->h_totals[0];
    info->corrected_total = ctx->h_totals[1];
    info->n_sites = ctx->h_totals[2];
    info->n_slabs = ctx->h_totals[3];
  }
  const size_t b = (size_t)ctx->corr_pids * 4 * 8;
  if (removed && b) memcpy(removed, ctx->h_report, b);
  if (shortfall && b) memcpy(shortfall, ctx->h_report + b / 8, b);
  return XS_OK;
}

int xs_transition_sites(xs_ctx_t* ctx, const xs_events_t* ev, int pair_mask, int64_t* n_out, xs_stream_t stream);
int xs_transition_fetch(xs_ctx_t* ctx, int32_t* pair, int64_t* event, xs_stream_t stream);
int xs_remap(xs_ctx_t* ctx, int64_t n, const int32_t* pid_dev, const int64_t* val_dev, int64_t* out_dev,
             xs_stream_t stream);

}  // extern "C"

// ---------------------------------------------------------------------------
// per-stage device timing
// ---------------------------------------------------------------------------
namespace xs {

cudaEvent_t prof_event(xs_ctx* ctx) {
  if (ctx->capturing) {  // owned by the graph being captured, never pooled
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->graph_events.push_back(e);
    return e;
  }
  // events in flight are never reused before prof_flush
  if (ctx->pool_next == ctx->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->ev_pool.push_back(e);
  }
  return ctx->ev_pool[ctx->pool_next++];
}

void prof_flush(xs_ctx* ctx) {
  for (size_t k = 0; k < ctx->pend_stage.size(); k++) {
    float ms = 0.f;
    if (cudaEventSynchronize(ctx->pend_b[k]) == cudaSuccess &&
        cudaEventElapsedTime(&ms, ctx->pend_a[k], ctx->pend_b[k]) == cudaSuccess) {
      ctx->prof_ms[ctx->pend_stage[k]] += ms;
      ctx->prof_calls[ctx->pend_stage[k]] += 1;
    } else {
      cudaGetLastError();  // a timing miss must not surface as a later launch error
    }
  }
  ctx->pend_stage.clear();
  ctx->pend_a.clear();
  ctx->pend_b.clear();
  if (ctx->prof_active == 0) ctx->pool_next = 0;  // an open scope still owns its start event
}

}  // namespace xs

extern "C" {

static const char* kStageNames[xs::ST_NUM] = {
    "pass1_validate_spans", "operation_paths", "transition_sort", "transition_scan", "site_sort",
    "quantize_scan",        "removal_scan",    "remap",           "endpoint_keygen", "endpoint_sort",
    "sweep_scan_hist",      "cell_compact",    "correlation_prepass"};

int xs_profile_enable(xs_ctx_t* ctx, int on) {
  if (!ctx) return XS_BAD_ARGUMENT;
  xs::prof_flush(ctx);
  ctx->prof_on = on != 0;
  for (int i = 0; i < 32; i++) {
    ctx->prof_ms[i] = 0;
    ctx->prof_calls[i] = 0;
  }
  return XS_OK;
}

int xs_profile_read(xs_ctx_t* ctx, double* ms, int64_t* calls, int n) {
  if (!ctx) return XS_BAD_ARGUMENT;
  xs::prof_flush(ctx);
  for (int i = 0; i < n && i < xs::ST_NUM; i++) {
    if (ms) ms[i] = ctx->prof_ms[i];
    if (calls) calls[i] = ctx->prof_calls[i];
  }
  return xs::ST_NUM;
}

const char* xs_profile_stage_name(int i) { return (i >= 0 && i < xs::ST_NUM) ? kStageNames[i] : ""; }

}  // extern "C"
