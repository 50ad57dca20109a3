// xs_ctx.cu -- C ABI entry points, workspace and sort plumbing.
#include <cub/device/device_radix_sort.cuh>

#include "xs_engine.cuh"

using namespace xs;

namespace xs {

int ws_get(xs_ctx* ctx, int slot, size_t bytes, cudaStream_t s, void** out) {
  if (bytes < 256) bytes = 256;
  if (ctx->cap[slot] < bytes) {
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
  XS_CUDA(cudaMemcpyAsync(ctx->h_stats, d, sizeof(Stats), cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaStreamSynchronize(s));
  if (!ctx->pend_stage.empty()) prof_flush(ctx);
  return XS_OK;
}

int sort_pairs_u64_u32(xs_ctx* ctx, uint64_t** keys, uint64_t** keys_alt, uint32_t** vals, uint32_t** vals_alt,
                       int64_t n, int bits, cudaStream_t s) {
  if (n <= 1 || bits <= 0) return XS_OK;
  if (bits > 64) bits = 64;
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

int run_validate(xs_ctx* ctx, const EventView& v, cudaStream_t s, long long* n_bad) {
  int st = stage_events(ctx, v, s, true, false, nullptr);
  if (st == XS_INVALID_TRACE) {
    *n_bad = ctx->h_stats->n_bad;
    return XS_OK;
  }
  XS_TRY(st);
  XS_TRY(stage_ops(ctx, v, s, false));
  XS_TRY(fetch_stats(ctx, s));
  *n_bad = ctx->h_stats->n_bad;
  return XS_OK;
}

int run_overlap(xs_ctx* ctx, const EventView& v, int attribution, cudaStream_t s) {
  ctx->have_overlap = false;
  XS_TRY(stage_events(ctx, v, s, true, false, nullptr));  // syncs once; per-event rule violations stop here
  for (int attempt = 0; attempt < 8; attempt++) {
    XS_TRY(stage_ops(ctx, v, s, true));
    XS_TRY(stage_overlap(ctx, v, attribution, s));
    // stage_overlap ends with fetch_stats
    if (ctx->h_stats->n_bad) return XS_INVALID_TRACE;
    if (ctx->h_stats->depth_overflow) {
      ctx->err = "merged multi-tid operation path deeper than the device limit";
      return XS_UNSUPPORTED;
    }
    if (ctx->h_stats->pad[3]) {  // a bucket overflowed a chunk: redo this call via the LSD sort
      ctx->force_lsd = true;
      continue;
    }
    if (!ctx->h_stats->table_full) {
      ctx->have_overlap = true;
      ctx->force_lsd = false;
      return XS_OK;
    }
    ctx->trie_cap_log2 += 2;
  }
  ctx->force_lsd = false;
  ctx->err = "path table could not be sized";
  return XS_NO_MEMORY;
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
  e = cudaMallocHost(&c->h_stats, sizeof(Stats));
  if (e != cudaSuccess) {
    delete c;
    return XS_CUDA_ERROR;
  }
  memset(c->h_stats, 0, sizeof(Stats));
  *out = c;
  return XS_OK;
}

void xs_ctx_destroy(xs_ctx_t* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (void* p : ctx->ptr)
    if (p) cudaFree(p);
  if (ctx->h_stats) cudaFreeHost(ctx->h_stats);
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
  if (has_events && np) {
    std::vector<int64_t> lo(np);
    XS_CUDA(cudaMemcpyAsync(lo.data(), ctx->ptr[W_SPAN_LO], np * 8, cudaMemcpyDeviceToHost, s));
    XS_CUDA(cudaStreamSynchronize(s));
    for (size_t p = 0; p < np; p++) has_events[p] = lo[p] != INT64_MAX;
  }
  XS_CUDA(cudaStreamSynchronize(s));
  return XS_OK;
}

static int correct_common(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int64_t* out_start,
                          int64_t* out_dur, int64_t* bad_event, cudaStream_t s, bool corrected_spans) {
  ctx->have_correct = false;
  if (bad_event) *bad_event = -1;
  if (!prof || prof->L <= 0) return XS_BAD_ARGUMENT;
  if (ev->n > 0 && (!out_start || !out_dur)) return XS_BAD_ARGUMENT;
  EventView v{*ev, ev->start, ev->dur};
  XS_TRY(stage_events(ctx, v, s, true, true, prof));  // (sync: sizes; per-event rule violations stop here)
  XS_TRY(stage_ops(ctx, v, s, false));                // OPERATION nesting is part of require_valid
  // the pipeline is safe on a trace whose nesting / correlations / API names
  // turn out bad, so the verdict is read once, after it
  XS_TRY(stage_transitions(ctx, v, 0x2 /*HIGH_LEVEL*/, 0xC /*BACKEND|SIMULATOR*/, s));
  XS_TRY(stage_correct(ctx, v, prof, out_start, out_dur, corrected_spans, s));
  XS_TRY(fetch_stats(ctx, s));
  if (ctx->h_stats->n_bad) return XS_INVALID_TRACE;   // require_valid runs first in the reference
  if (ctx->h_stats->bad_api != INT64_MAX) {
    if (bad_event) *bad_event = ctx->h_stats->bad_api;
    return XS_UNCALIBRATED;
  }
  ctx->have_correct = true;
  return XS_OK;
}

int xs_correct(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int64_t* out_start_dev,
               int64_t* out_dur_dev, int64_t* bad_event, xs_stream_t stream) {
  XS_TRY(check_events(ctx, ev));
  cudaSetDevice(ctx->device);
  return correct_common(ctx, ev, prof, out_start_dev, out_dur_dev, bad_event, (cudaStream_t)stream, true);
}

int xs_analyze(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int attribution,
               int64_t* out_start_dev, int64_t* out_dur_dev, int64_t* bad_event, xs_stream_t stream) {
  XS_TRY(check_events(ctx, ev));
  if (attribution != 0 && attribution != 1) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  XS_TRY(correct_common(ctx, ev, prof, out_start_dev, out_dur_dev, bad_event, s, false));
  EventView v{*ev, out_start_dev, out_dur_dev};
  int st = run_overlap(ctx, v, attribution, s);
  if (st != XS_OK) return st;
  // corrected_total_ns = sum of the corrected pid spans the overlap pass
  // computed; stays on the device until xs_correct_report
  return corrected_total_from_spans(ctx, s);
}

int xs_correct_report(xs_ctx_t* ctx, xs_correct_info_t* info, int64_t* removed, int64_t* shortfall,
                      xs_stream_t stream) {
  if (!ctx || !ctx->have_correct) return XS_BAD_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  if (info) {  // [original_total, corrected_total, n_sites, n_slabs] written by the pipeline
    int64_t tot[4] = {0, 0, 0, 0};
    XS_CUDA(cudaMemcpyAsync(tot, ctx->ptr[W_CORR_TOTALS], sizeof(tot), cudaMemcpyDeviceToHost, s));
    XS_CUDA(cudaStreamSynchronize(s));
    info->original_total = tot[0];
    info->corrected_total = tot[1];
    info->n_sites = tot[2];
    info->n_slabs = tot[3];
  }
  size_t b = (size_t)ctx->corr_pids * 4 * 8;
  if (removed && b) XS_CUDA(cudaMemcpyAsync(removed, ctx->ptr[W_REMOVED], b, cudaMemcpyDeviceToHost, s));
  if (shortfall && b) XS_CUDA(cudaMemcpyAsync(shortfall, ctx->ptr[W_SHORTFALL], b, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaStreamSynchronize(s));
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
