// xs_metrics.cu -- union time of one category and sampled utilization.
//
// Replaces, on the device:
//   metrics._union_ns(trace, category)            metrics.py:41-58
//       (sort (start, end) of the category's nonzero events, merge touching /
//        overlapping intervals, sum lengths) -- trace-wide, or per pid for
//        procview.build_process_tree's gpu_busy_ns (procview.py:68-77)
//   metrics.utilization_samples / sampled_utilization   metrics.py:61-84
//       (a period [lo + kP, lo + (k+1)P) is utilized iff it intersects a GPU
//        event of nonzero duration; equivalently it intersects the union)
//
// One compaction of the category's endpoints into keys
//     per pid : pid | (t - lo[pid]) | close      trace : (t - lo) | close
// (opens sort before closes at equal t, so touching intervals merge exactly
// like the reference's `lo <= cur_hi`), a radix sort, a +-1 prefix sum
// (coverage count), and one reduction:
//   union length  = sum over i of [count_i > 0] * (t_{i+1} - t_i)  (same segment)
//   union intervals start where the count leaves 0 and end where it returns.
// Utilized periods = sum over intervals of (last - first + 1) minus the
// intervals whose first period equals the previous interval's last period.
// Everything is integer; the ratios are formed on the host like the reference.
#include <cub/cub.cuh>

#include "xs_engine.cuh"
#include "xs_prims.cuh"

namespace xs {

__global__ void k_span_reduce(const int64_t* lo, const int64_t* hi, int np, int64_t* out) {
  // out[0] = min lo, out[1] = max hi over pids with events (single block)
  long long l = INT64_MAX, h = INT64_MIN;
  for (int p = threadIdx.x; p < np; p += blockDim.x) {
    if (lo[p] != INT64_MAX) {
      l = lo[p] < l ? lo[p] : l;
      h = hi[p] > h ? hi[p] : h;
    }
  }
  typedef cub::BlockReduce<long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  const long long L = BR(tmp).Reduce(l, cub::Min());
  __syncthreads();
  const long long H = BR(tmp).Reduce(h, cub::Max());
  if (threadIdx.x == 0) {
    out[0] = L;
    out[1] = H;
  }
}

// endpoints of the category's nonzero-duration events, compacted
__global__ void k_union_keys(EventView v, int64_t n, int cat, int per_pid, const int64_t* lo_pid,
                             const int64_t* glo, int tb, uint64_t* keys, unsigned long long* count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool take = i < n && v.ev.cat[i] == cat && v.dur[i] > 0;
  const unsigned act = __ballot_sync(0xffffffffu, take);
  if (!act) return;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == __ffs(act) - 1) base = atomicAdd(count, 2ull * __popc(act));
  base = __shfl_sync(0xffffffffu, base, __ffs(act) - 1);
  if (!take) return;
  const int64_t at = (int64_t)base + 2 * __popc(act & ((1u << lane) - 1));
  const int p = v.ev.pid[i];
  const int64_t org = per_pid ? lo_pid[p] : *glo;
  const uint64_t hi_bits = per_pid ? ((uint64_t)p << (tb + 1)) : 0ull;
  const uint64_t s = (uint64_t)(v.start[i] - org), e = (uint64_t)(v.start[i] + v.dur[i] - org);
  keys[at] = hi_bits | (s << 1);
  keys[at + 1] = hi_bits | (e << 1) | 1ull;
}

struct UnionDelta {
  __device__ int operator()(const uint64_t& k) const { return (k & 1ull) ? -1 : 1; }
};

// acc[0] = sum(last) - sum(first) + #intervals - #shared periods (utilized
// periods), acc[1] = #intervals; per-segment union length into seg_ns
__global__ void k_union_reduce(const uint64_t* keys, const int* depth, int64_t m, int tb, int per_pid,
                               const int64_t* glo, int64_t period, unsigned long long* seg_ns, long long* acc,
                               int64_t* iv_lo, int64_t* iv_hi) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  long long util = 0, nint = 0;
  int seg_k = -1;
  long long seg_v[1] = {0};
  if (i < m) {
    const uint64_t k = keys[i];
    const uint64_t tmask = tb >= 63 ? ~0ull : ((1ull << (tb + 1)) - 1);
    const int64_t t = (int64_t)((k & tmask) >> 1);
    const int seg = per_pid ? (int)(k >> (tb + 1)) : 0;
    const int d = depth[i];
    if (d > 0 && i + 1 < m) {
      const uint64_t kn = keys[i + 1];
      const int segn = per_pid ? (int)(kn >> (tb + 1)) : 0;
      const int64_t tn = (int64_t)((kn & tmask) >> 1);
      if (segn == seg && tn > t) {
        seg_k = seg;
        seg_v[0] = tn - t;
      }
    }
    if (!per_pid) {
      const int dp = i > 0 ? depth[i - 1] : 0;
      if (d == 1 && dp == 0) {  // a union interval starts at t
        nint = 1;
        if (period > 0) {
          const int64_t first = t / period;
          util -= first;
          util += 1;
          if (i > 0) {
            const int64_t tp = (int64_t)((keys[i - 1] & tmask) >> 1);  // previous interval's end
            if ((tp - 1) / period == first) util -= 1;
          }
        }
        if (iv_lo) iv_lo[i] = t;
      }
      if (d == 0) {  // a union interval ends at t
        if (period > 0) util += (t - 1) / period;
        if (iv_hi) iv_hi[i] = t;
      }
    }
  }
  // one add per segment per block (segments are contiguous in key order)
  block_keyed_flush<1>(seg_k, seg_v, [&](int k, const long long* x) {
    if (x[0]) atomicAdd(&seg_ns[k], (unsigned long long)x[0]);
  });
  typedef cub::BlockReduce<long long, XS_BLOCK> BR;
  __shared__ typename BR::TempStorage tmp;
  const long long u = BR(tmp).Sum(util);
  __syncthreads();
  const long long c = BR(tmp).Sum(nint);
  if (threadIdx.x == 0 && (u || c)) {
    atomicAdd((unsigned long long*)&acc[0], (unsigned long long)u);
    atomicAdd((unsigned long long*)&acc[1], (unsigned long long)c);
  }
}

// union interval endpoints -> dense sorted lists (positions are increasing)
__global__ void k_union_intervals(const uint64_t* keys, const int* depth, int64_t m, int tb, const int64_t* glo,
                                  const int* start_rank, const int* end_rank, int64_t* out_lo, int64_t* out_hi) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint64_t tmask = tb >= 63 ? ~0ull : ((1ull << (tb + 1)) - 1);
  const int64_t t = (int64_t)((keys[i] & tmask) >> 1) + *glo;
  const int d = depth[i], dp = i > 0 ? depth[i - 1] : 0;
  if (d == 1 && dp == 0) out_lo[start_rank[i]] = t;
  if (d == 0) out_hi[end_rank[i]] = t;
}

struct IsStart {
  const int* depth;
  __device__ int operator()(const int64_t& i) const { return depth[i] == 1 && (i == 0 || depth[i - 1] == 0); }
};
struct IsEnd {
  const int* depth;
  __device__ int operator()(const int64_t& i) const { return depth[i] == 0; }
};

int run_union(xs_ctx* ctx, const EventView& v, int cat, int per_pid, int64_t period, int64_t* out_ns,
              int64_t* utilized, int64_t* n_intervals, int64_t* span_lo, int64_t* span_hi, cudaStream_t s) {
  XS_TRY(stage_events(ctx, v, s, false, false, nullptr));
  XS_CUDA(cudaMemsetAsync(&((Stats*)ctx->ptr[W_STATS])->pad[3], 0, 8, s));
  const Stats& H = *ctx->h_stats;
  const int np = v.ev.n_pids;
  const int64_t n = v.ev.n;
  const int64_t* lo = (const int64_t*)ctx->ptr[W_SPAN_LO];
  const int64_t* hi = (const int64_t*)ctx->ptr[W_SPAN_HI];
  int64_t* gspan;
  XS_TRY(ws(ctx, W_UN_GSPAN, 4, s, &gspan));
  XS_LAUNCH(ctx, k_span_reduce, 1, 256, 0, s, lo, hi, np, gspan);
  unsigned long long* cnt;
  long long* acc;
  XS_TRY(ws(ctx, W_UN_ACC, 4, s, &cnt));
  acc = (long long*)(cnt + 1);
  XS_CUDA(cudaMemsetAsync(cnt, 0, 4 * 8, s));
  int64_t h_span[2] = {0, 0};
  XS_CUDA(cudaMemcpyAsync(h_span, gspan, 16, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaStreamSynchronize(s));
  if (span_lo) *span_lo = h_span[0];
  if (span_hi) *span_hi = h_span[1];
  const int nseg = per_pid ? np : 1;
  unsigned long long* seg_ns;
  XS_TRY(ws(ctx, W_UN_SEG, nseg + 1, s, &seg_ns));
  XS_CUDA(cudaMemsetAsync(seg_ns, 0, (nseg + 1) * 8, s));
  const int64_t ncat = H.cat_nz[cat];
  const int64_t m = 2 * ncat;
  int64_t h_acc[2] = {0, 0};
  const bool any = n > 0 && h_span[1] > h_span[0] && m > 0;
  if (any) {
    const int tb = bits_for((uint64_t)(per_pid ? H.max_span : h_span[1] - h_span[0]));
    const int pb = bits_for((uint64_t)(np > 0 ? np - 1 : 0));
    if ((per_pid ? pb : 0) + tb + 1 > 64) {
      ctx->err = "timeline too wide for 64-bit union keys";
      return XS_UNSUPPORTED;
    }
    uint64_t *k, *k_alt;
    int* depth;
    XS_TRY(ws(ctx, W_UN_KEY, m + 1, s, &k));
    XS_TRY(ws(ctx, W_UN_KEY_ALT, m + 1, s, &k_alt));
    XS_TRY(ws(ctx, W_UN_DEPTH, m + 1, s, &depth));
    XS_LAUNCH(ctx, k_union_keys, grid_for(n), XS_BLOCK, 0, s, v, n, cat, per_pid, lo, gspan, tb, k, cnt);
    XS_TRY(sort_keys_u64(ctx, &k, &k_alt, m, (per_pid ? pb : 0) + tb + 1, s));
    {
      XS_TRY(scan_inclusive<int>(ctx, map_in((const uint64_t*)k, UnionDelta()), depth, m, s));
    }
    XS_LAUNCH(ctx, k_union_reduce, grid_for(m), XS_BLOCK, 0, s, k, depth, m, tb, per_pid, gspan, period, seg_ns,
              acc, (int64_t*)nullptr, (int64_t*)nullptr);
    XS_CUDA(cudaMemcpyAsync(h_acc, acc, 16, cudaMemcpyDeviceToHost, s));
    ctx->un_keys = k;
    ctx->un_depth = depth;
    ctx->un_m = m;
    ctx->un_tb = tb;
  } else {
    ctx->un_m = 0;
  }
  ctx->un_intervals = per_pid ? -1 : h_acc[1];
  if (out_ns) XS_CUDA(cudaMemcpyAsync(out_ns, seg_ns, nseg * 8, cudaMemcpyDeviceToHost, s));
  long long ovf = 0;  // a bucketed key sort overflowed: the caller re-runs through the LSD sort
  XS_CUDA(cudaMemcpyAsync(&ovf, &((Stats*)ctx->ptr[W_STATS])->pad[3], 8, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaStreamSynchronize(s));
  if (ovf && !ctx->force_lsd) return XS_RETRY_LSD;
  if (utilized) *utilized = h_acc[0];
  if (n_intervals) *n_intervals = h_acc[1];
  return XS_OK;
}

int fetch_union_intervals(xs_ctx* ctx, int64_t* out_lo, int64_t* out_hi, cudaStream_t s) {
  if (ctx->un_intervals < 0) {
    ctx->err = "no trace-wide union computed";
    return XS_BAD_ARGUMENT;
  }
  const int64_t ni = ctx->un_intervals, m = ctx->un_m;
  if (ni == 0) return XS_OK;
  int *rs, *re;
  int64_t *dlo, *dhi;
  XS_TRY(ws(ctx, W_UN_RANK, 2 * m + 2, s, &rs));
  re = rs + m + 1;
  XS_TRY(ws(ctx, W_UN_IV, 2 * ni, s, &dlo));
  dhi = dlo + ni;
  {  // exclusive prefix counts of starts / ends = output slots
    XS_TRY(scan_exclusive<int>(ctx, IsStart{ctx->un_depth}, rs, m, s));
    XS_TRY(scan_exclusive<int>(ctx, IsEnd{ctx->un_depth}, re, m, s));
  }
  const int64_t* gspan = (const int64_t*)ctx->ptr[W_UN_GSPAN];
  XS_LAUNCH(ctx, k_union_intervals, grid_for(m), XS_BLOCK, 0, s, ctx->un_keys, ctx->un_depth, m, ctx->un_tb, gspan,
            rs, re, dlo, dhi);
  XS_CUDA(cudaMemcpyAsync(out_lo, dlo, ni * 8, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaMemcpyAsync(out_hi, dhi, ni * 8, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaStreamSynchronize(s));
  return XS_OK;
}

}  // namespace xs

using namespace xs;

extern "C" {

int xs_union(xs_ctx_t* ctx, const xs_events_t* ev, int category, int per_pid, int64_t* out_ns, int64_t* span_lo,
             int64_t* span_hi, xs_stream_t stream) {
  if (!ctx || !ev || category < 0 || category > 5) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  EventView v{*ev, ev->start, ev->dur};
  return with_lsd_retry(ctx, [&] {
    return run_union(ctx, v, category, per_pid, 0, out_ns, nullptr, nullptr, span_lo, span_hi, (cudaStream_t)stream);
  });
}

int xs_utilization(xs_ctx_t* ctx, const xs_events_t* ev, int64_t period_ns, int64_t* utilized, int64_t* n_intervals,
                   int64_t* span_lo, int64_t* span_hi, xs_stream_t stream) {
  if (!ctx || !ev || period_ns <= 0) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  EventView v{*ev, ev->start, ev->dur};
  int64_t ns = 0;
  return with_lsd_retry(ctx, [&] {
    return run_union(ctx, v, 5, 0, period_ns, &ns, utilized, n_intervals, span_lo, span_hi, (cudaStream_t)stream);
  });
}

int xs_union_intervals_fetch(xs_ctx_t* ctx, int64_t* out_lo, int64_t* out_hi, xs_stream_t stream) {
  if (!ctx || !out_lo || !out_hi) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  return fetch_union_intervals(ctx, out_lo, out_hi, (cudaStream_t)stream);
}

}  // extern "C"
