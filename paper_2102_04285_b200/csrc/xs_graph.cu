// xs_graph.cu -- CUDA-graph capture and replay of sync-free pipeline segments.
//
// At config-2 sizes the pipeline is a few dozen short kernels between a
// handful of host syncs, so host launch latency, not the GPU, bounds the step.
// Each segment between syncs is a deterministic function of what the host
// knows at its start: the input/output pointers and sizes, the statistics of
// the preceding sync and the retry flags.  Keyed on exactly that, the first
// sighting runs eagerly (and sizes the workspace), the second is captured into
// a graph, and later calls replay the graph; a graph remembers the workspace
// generation it was captured in and is never replayed after the workspace
// moved (the next sighting captures again).  A
// segment that tries to allocate or synchronize while being captured is
// marked non-capturable and keeps running eagerly.
//
// The cache is bounded: graphs of an older workspace generation hold freed
// pointers and are dropped as soon as the workspace grows, and at most
// kMaxGraphs graphs (least recently replayed first out) are kept, so a
// long-running process analysing many distinct traces does not grow without
// bound.  The sighting and non-capturable sets are bounded the same way.
#include "xs_engine.cuh"

#include <cstdio>
#include <cstdlib>

namespace xs {

std::string segment_key(xs_ctx* ctx, const char* tag, const void* extra, size_t extra_bytes) {
  std::string k(tag);
  k.push_back('\0');
  k.append(reinterpret_cast<const char*>(ctx->h_stats), sizeof(Stats));
  k.append(reinterpret_cast<const char*>(extra), extra_bytes);
  // (no workspace generation: a graph records it and is never replayed
  // across a generation change, and a key seen before a workspace growth is
  // still "seen" -- its next call captures instead of starting over eagerly)
  const long long misc[4] = {ctx->trie_cap_log2, ctx->force_lsd ? 1 : 0, ctx->prof_on ? 1 : 0, ctx->deep_cap};
  k.append(reinterpret_cast<const char*>(misc), sizeof(misc));
  return k;
}

static bool graphs_enabled() {
  static int en = -1;
  if (en < 0) en = getenv("XS_NO_GRAPHS") ? 0 : 1;
  return en == 1;
}

static constexpr size_t kMaxGraphs = 64, kMaxKeys = 4096;

static void drop_graph(xs_ctx* ctx, std::map<std::string, xs_ctx::GraphEntry>::iterator it) {
  if (!ctx->pend_stage.empty()) prof_flush(ctx);  // (pending timings may name this graph's events)
  if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
  for (cudaEvent_t e : it->second.events) cudaEventDestroy(e);
  ctx->graphs.erase(it);
}

// drop graphs of older workspace generations; keep the cache under kMaxGraphs
static void trim_graphs(xs_ctx* ctx, cudaStream_t s) {
  if (ctx->graph_generation != ctx->ws_generation) {
    bool any = false;
    for (auto it = ctx->graphs.begin(); it != ctx->graphs.end();) {
      auto nx = std::next(it);
      if (it->second.generation != ctx->ws_generation) {
        if (!any) cudaStreamSynchronize(s);  // (a replay of it may still be in flight)
        any = true;
        drop_graph(ctx, it);
      }
      it = nx;
    }
    ctx->graph_generation = ctx->ws_generation;
  }
  while (ctx->graphs.size() >= kMaxGraphs) {
    auto victim = ctx->graphs.begin();
    for (auto it = ctx->graphs.begin(); it != ctx->graphs.end(); ++it)
      if (it->second.used < victim->second.used) victim = it;
    cudaStreamSynchronize(s);
    drop_graph(ctx, victim);
  }
  if (ctx->graph_seen.size() > kMaxKeys) ctx->graph_seen.clear();
  if (ctx->graph_bad.size() > kMaxKeys) ctx->graph_bad.clear();
}

static int run_segment_on(xs_ctx* ctx, cudaStream_t s, const std::string& key,
                          const std::function<int(cudaStream_t)>& body0) {
  auto body = [&]() { return body0(s); };
  if (ctx->graph_bad.count(key)) return body();
  auto it = ctx->graphs.find(key);
  if (it != ctx->graphs.end() && it->second.generation != ctx->ws_generation) {
    trim_graphs(ctx, s);  // stale pointers: never replay
    it = ctx->graphs.end();
  }
  if (it != ctx->graphs.end()) {
    it->second.used = ++ctx->graph_tick;
    XS_CUDA(cudaGraphLaunch(it->second.exec, s));
    ctx->ops = it->second.ops;
    ctx->launches += it->second.launches;
    if (ctx->prof_on)
      for (size_t i = 0; i < it->second.prof_stage.size(); i++) {
        ctx->pend_stage.push_back(it->second.prof_stage[i]);
        ctx->pend_a.push_back(it->second.prof_a[i]);
        ctx->pend_b.push_back(it->second.prof_b[i]);
      }
    return XS_OK;
  }
  static const bool dbg = getenv("XS_DEBUG_GRAPH") != nullptr;
  if (dbg) fprintf(stderr, "[xs graph] %s miss (%zu graphs)\n", key.c_str(), ctx->graphs.size());
  // First sighting: eager (a one-off trace never pays capture + instantiate).
  // Second sighting: captured.  If the workspace must grow, the capture
  // aborts at the first allocation (ws_get) and the segment runs eagerly,
  // sizing the workspace; the next call captures.
  if (!ctx->graph_seen.count(key)) {
    ctx->graph_seen.insert(key);
    return body();
  }
  trim_graphs(ctx, s);
  const long long l0 = ctx->launches;
  const size_t p0 = ctx->pend_stage.size();
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    ctx->graph_bad.insert(key);
    return body();
  }
  ctx->capturing = true;
  ctx->graph_events.clear();
  const int st = body();
  ctx->capturing = false;
  std::vector<cudaEvent_t> cap_events;
  cap_events.swap(ctx->graph_events);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &g);
  cudaGraphExec_t exec = nullptr;
  if (st == XS_OK && e == cudaSuccess && g) e = cudaGraphInstantiate(&exec, g, 0);
  if (g) cudaGraphDestroy(g);
  // timing entries recorded while capturing belong to the graph, not to this call
  xs_ctx::GraphEntry ge;
  for (size_t i = p0; i < ctx->pend_stage.size(); i++) {
    ge.prof_stage.push_back(ctx->pend_stage[i]);
    ge.prof_a.push_back(ctx->pend_a[i]);
    ge.prof_b.push_back(ctx->pend_b[i]);
  }
  ctx->pend_stage.resize(p0);
  ctx->pend_a.resize(p0);
  ctx->pend_b.resize(p0);
  if (st != XS_OK || e != cudaSuccess || !exec) {  // workspace growth, or not capturable: eager
    if (exec) cudaGraphExecDestroy(exec);
    for (cudaEvent_t ev : cap_events) cudaEventDestroy(ev);
    cudaGetLastError();
    ctx->err.clear();
    ctx->launches = l0;
    if (st != XS_CAPTURE_ABORT) ctx->graph_bad.insert(key);  // (eager from now on)
    return body();
  }
  ge.exec = exec;
  ge.launches = ctx->launches - l0;
  ge.ops = ctx->ops;
  ge.generation = ctx->ws_generation;
  ge.events = std::move(cap_events);
  ctx->launches = l0;
  ctx->graphs[key] = ge;
  return run_segment_on(ctx, s, key, body0);  // replay it now
}

// The legacy default stream cannot be captured: segments then run on a
// private stream joined to the caller's stream by events.
int run_segment(xs_ctx* ctx, cudaStream_t s, const std::string& key, bool capturable,
                const std::function<int(cudaStream_t)>& body) {
  if (!capturable || !graphs_enabled()) return body(s);
  if (s != 0 && s != cudaStreamLegacy) return run_segment_on(ctx, s, key, body);
  if (!ctx->priv_stream) {
    XS_CUDA(cudaStreamCreateWithFlags(&ctx->priv_stream, cudaStreamNonBlocking));
    XS_CUDA(cudaEventCreateWithFlags(&ctx->join_in, cudaEventDisableTiming));
    XS_CUDA(cudaEventCreateWithFlags(&ctx->join_out, cudaEventDisableTiming));
  }
  XS_CUDA(cudaEventRecord(ctx->join_in, s));
  XS_CUDA(cudaStreamWaitEvent(ctx->priv_stream, ctx->join_in, 0));
  const int st = run_segment_on(ctx, ctx->priv_stream, key, body);
  XS_CUDA(cudaEventRecord(ctx->join_out, ctx->priv_stream));
  XS_CUDA(cudaStreamWaitEvent(s, ctx->join_out, 0));
  return st;
}

}  // namespace xs
