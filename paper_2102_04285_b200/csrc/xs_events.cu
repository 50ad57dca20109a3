// xs_events.cu -- pass 1 over the event columns.
//
// One streaming read of start/dur/pid/tid/cat (+name for the profile check):
//   * validate_trace event rules (model.py:193-207): negative duration /
//     start, int64 range, unknown pid  -> Stats.n_bad
//   * pid_spans (model.py:125-134): per-pid min start / max end
//   * counts that size every later stage (nonzero events, OPERATIONs, ...)
//   * per-pid and per-(pid,tid) counts of nonzero OPERATIONs
//   * correction: first ACCEL_API whose name the profile lacks
//     (correction.py:70-76, UncalibratedHookError)
// then the (pid, correlation) table of ACCEL_API launches, used for the
// dangling-correlation rule (model.py:186-189, 212-222) and, in CORRELATION
// attribution, the launch instant of each GPU event (overlap.py:148-157: the
// earliest launch by Event.sort_key, whose first field is start -> min start).
#include "xs_engine.cuh"

namespace xs {

constexpr int P1_ITEMS = 4;

__global__ void k_init_pid(int64_t* lo, int64_t* hi, int* pid_ops, int np) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < np) {
    lo[p] = INT64_MAX;
    hi[p] = INT64_MIN;
    pid_ops[p] = 0;
  }
}

__global__ void k_init_stats(Stats* st) {
  if (threadIdx.x == 0) {
    memset(st, 0, sizeof(Stats));
    st->bad_api = INT64_MAX;
  }
}

__device__ __forceinline__ long long warp_sum(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(XS_BLOCK) k_pass1(EventView v, int64_t n, const uint8_t* __restrict__ has_meta,
                                                    const uint8_t* __restrict__ has_internal, int check_api,
                                                    Stats* st, int64_t* lo_out, int64_t* hi_out, int* pid_ops,
                                                    int* group_ops) {
  const int64_t* __restrict__ start = v.start;
  const int64_t* __restrict__ dur = v.dur;
  const int32_t* __restrict__ pid = v.ev.pid;
  const int32_t* __restrict__ tid = v.ev.tid;
  const uint8_t* __restrict__ cat = v.ev.cat;
  const int32_t* __restrict__ name = v.ev.name;
  const uint8_t* __restrict__ has_corr = v.ev.has_corr;

  long long bad = 0, nz = 0, opsnz = 0, ops = 0, api = 0, apic = 0, gpuc = 0;
  long long cat_cnt[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // [0..5] all, [6..11] nonzero
  long long bad_api = INT64_MAX;
  int cur_p = -1, cur_g = -1, cur_pops = 0, cur_gops = 0;
  long long lo = 0, hi = 0;
  const int64_t base = (int64_t)blockIdx.x * XS_BLOCK * P1_ITEMS + threadIdx.x;
#pragma unroll 4
  for (int k = 0; k < P1_ITEMS; k++) {
    int64_t i = base + (int64_t)k * XS_BLOCK;
    if (i >= n) break;
    int64_t s = start[i], d = dur[i];
    int p = pid[i];
    int c = cat[i];
    bad += (d < 0) + (s < 0);
    int64_t dd = d > 0 ? d : 0;
    bad += (s > 0 && dd > INT64_MAX - s);
    bad += !has_meta[p];
    int64_t e = (int64_t)((uint64_t)s + (uint64_t)d);
    if (p != cur_p) {
      if (cur_p >= 0) {
        atomic_min_i64(&lo_out[cur_p], lo);
        atomic_max_i64(&hi_out[cur_p], hi);
        if (cur_pops) atomicAdd(&pid_ops[cur_p], cur_pops);
      }
      cur_p = p;
      lo = s;
      hi = e;
      cur_pops = 0;
    } else {
      lo = s < lo ? s : lo;
      hi = e > hi ? e : hi;
    }
    nz += d > 0;
#pragma unroll
    for (int q = 0; q < 6; q++) {
      cat_cnt[q] += c == q;
      cat_cnt[6 + q] += (c == q) & (d > 0);
    }
    if (c == 0) {
      ops++;
      if (d > 0) {
        opsnz++;
        cur_pops++;
        int g = tid[i];
        if (g != cur_g) {
          if (cur_g >= 0 && cur_gops) atomicAdd(&group_ops[cur_g], cur_gops);
          cur_g = g;
          cur_gops = 0;
        }
        cur_gops++;
      }
    } else if (c == 4) {
      api++;
      apic += has_corr[i];
      if (check_api && !has_internal[name[i]]) bad_api = i < bad_api ? i : bad_api;
    } else if (c == 5) {
      gpuc += has_corr[i];
    }
  }
  // flush the running per-pid reduction: warp-aggregate when the warp agrees
  const unsigned full = 0xffffffffu;
  int p0 = __shfl_sync(full, cur_p, 0);
  bool uniform = __all_sync(full, cur_p == p0);
  if (uniform && p0 >= 0) {
    long long l = lo, h = hi;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      long long l2 = __shfl_xor_sync(full, l, o), h2 = __shfl_xor_sync(full, h, o);
      l = l2 < l ? l2 : l;
      h = h2 > h ? h2 : h;
    }
    long long po = warp_sum(cur_pops);
    if ((threadIdx.x & 31) == 0) {
      atomic_min_i64(&lo_out[p0], l);
      atomic_max_i64(&hi_out[p0], h);
      if (po) atomicAdd(&pid_ops[p0], (int)po);
    }
  } else if (cur_p >= 0) {
    atomic_min_i64(&lo_out[cur_p], lo);
    atomic_max_i64(&hi_out[cur_p], hi);
    if (cur_pops) atomicAdd(&pid_ops[cur_p], cur_pops);
  }
  {
    long long gv[1] = {cur_gops};
    block_keyed_flush<1>(cur_gops ? cur_g : -1, gv, [&](int g, const long long* x) {
      if (x[0]) atomicAdd(&group_ops[g], (int)x[0]);
    });
  }

  block_keyed_flush<12>(0, cat_cnt, [&](int, const long long* x) {
    for (int q = 0; q < 6; q++) {
      if (x[q]) atomicAdd((unsigned long long*)&st->cat_all[q], (unsigned long long)x[q]);
      if (x[6 + q]) atomicAdd((unsigned long long*)&st->cat_nz[q], (unsigned long long)x[6 + q]);
    }
  });

  bad = warp_sum(bad);
  nz = warp_sum(nz);
  opsnz = warp_sum(opsnz);
  ops = warp_sum(ops);
  api = warp_sum(api);
  apic = warp_sum(apic);
  gpuc = warp_sum(gpuc);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    long long b2 = __shfl_xor_sync(full, bad_api, o);
    bad_api = b2 < bad_api ? b2 : bad_api;
  }
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd((unsigned long long*)&st->n_bad, (unsigned long long)bad);
    if (nz) atomicAdd((unsigned long long*)&st->n_nonzero, (unsigned long long)nz);
    if (opsnz) atomicAdd((unsigned long long*)&st->n_ops_nz, (unsigned long long)opsnz);
    if (ops) atomicAdd((unsigned long long*)&st->n_ops, (unsigned long long)ops);
    if (api) atomicAdd((unsigned long long*)&st->n_api, (unsigned long long)api);
    if (apic) atomicAdd((unsigned long long*)&st->n_api_corr, (unsigned long long)apic);
    if (gpuc) atomicAdd((unsigned long long*)&st->n_gpu_corr, (unsigned long long)gpuc);
    if (bad_api != INT64_MAX) atomicMin(&st->bad_api, bad_api);
  }
}

// per-pid span reduction for the max key width; also counts multi-tid op pids
__global__ void k_pid_finish(const int64_t* lo, const int64_t* hi, int np, const int32_t* group_pid,
                             const int* group_ops, int ng, int* pid_group0, Stats* st) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < np && lo[p] != INT64_MAX) atomicMax(&st->max_span, (long long)(hi[p] - lo[p]));
  // first group of each pid (groups are sorted by pid): binary search
  if (p <= np) {
    int a = 0, b = ng;
    while (a < b) {
      int m = (a + b) >> 1;
      if (group_pid[m] < p) a = m + 1;
      else b = m;
    }
    pid_group0[p] = a;
  }
  if (p < np) {
    int a = pid_group0[p];
    int cnt = 0;
    for (int g = a; g < ng && group_pid[g] == p; g++) cnt += group_ops[g] > 0;
    if (cnt > 1) atomicAdd((unsigned long long*)&st->multi_op_pids, 1ull);
  }
}

// ---------------------------------------------------------------------------
// (pid, correlation) -> min launch start, lock-free open addressing with an
// explicit claim state so arbitrary int64 correlation ids are exact keys.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t corr_hash(int p, int64_t corr) {
  uint64_t x = (uint64_t)corr * 0x9E3779B97F4A7C15ull ^ ((uint64_t)(uint32_t)p * 0xC2B2AE3D27D4EB4Full);
  x ^= x >> 31;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 29;
  return x;
}

__global__ void k_corr_insert(EventView v, int64_t n, int* state, int64_t* key, int* kpid, int64_t* kstart,
                              uint64_t mask, Stats* st) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (v.ev.cat[i] != 4 || !v.ev.has_corr[i]) return;
  int p = v.ev.pid[i];
  int64_t corr = v.ev.corr[i];
  int64_t s = v.start[i];
  uint64_t h = corr_hash(p, corr) & mask;
  for (uint64_t probe = 0; probe <= mask; probe++) {
    volatile int* sp = state + h;
    int cur = *sp;
    if (cur == 0) {
      if (atomicCAS(state + h, 0, 1) == 0) {
        key[h] = corr;
        kpid[h] = p;
        kstart[h] = s;
        __threadfence();
        atomicExch(state + h, 2);
        return;
      }
      cur = *sp;
    }
    while (cur == 1) cur = *sp;
    __threadfence();
    if (((volatile int64_t*)key)[h] == corr && ((volatile int*)kpid)[h] == p) {
      atomic_min_i64(&kstart[h], s);
      return;
    }
    h = (h + 1) & mask;
  }
  atomicAdd((unsigned long long*)&st->table_full, 1ull);
}

// GPU events: dangling check; in CORRELATION mode record the launch instant
__global__ void k_corr_query(EventView v, int64_t n, const int* state, const int64_t* key, const int* kpid,
                             const int64_t* kstart, uint64_t mask, Stats* st, int64_t* launch_start) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (v.ev.cat[i] != 5) return;
  if (!v.ev.has_corr[i]) {
    if (launch_start) launch_start[i] = INT64_MIN;
    return;
  }
  int p = v.ev.pid[i];
  int64_t corr = v.ev.corr[i];
  uint64_t h = corr_hash(p, corr) & mask;
  for (uint64_t probe = 0; probe <= mask; probe++) {
    if (state[h] == 0) break;
    if (key[h] == corr && kpid[h] == p) {
      if (launch_start) launch_start[i] = kstart[h];
      return;
    }
    h = (h + 1) & mask;
  }
  atomicAdd((unsigned long long*)&st->n_bad, 1ull);
  if (launch_start) launch_start[i] = INT64_MIN;
}

// pass 1 without its sync: the statistics stay on the device
int stage_events_async(xs_ctx* ctx, const EventView& v, cudaStream_t s, bool check_api, const xs_profile_t* prof) {
  const xs_events_t* ev = &v.ev;
  const int64_t n = ev->n;
  const int np = ev->n_pids, ng = ev->n_groups;
  Stats* st;
  int64_t *lo, *hi;
  int *pid_ops, *group_ops, *pid_group0;
  XS_TRY(ws(ctx, W_STATS, 1, s, &st));
  XS_TRY(ws(ctx, W_SPAN_LO, np + 1, s, &lo));
  XS_TRY(ws(ctx, W_SPAN_HI, np + 1, s, &hi));
  // (a speculative pass keeps the original trace's op counts: its own go to scratch)
  const bool alt = ctx->spec_keep_counts;
  XS_TRY(ws(ctx, alt ? W_PID_OPS_ALT : W_PID_OPS, np + 1, s, &pid_ops));
  XS_TRY(ws(ctx, alt ? W_GROUP_OPS_ALT : W_GROUP_OPS, ng + 1, s, &group_ops));
  XS_TRY(ws(ctx, alt ? W_PID_GROUP0_ALT : W_PID_GROUP0, np + 2, s, &pid_group0));
  XS_LAUNCH(ctx, k_init_stats, 1, 32, 0, s, st);
  XS_LAUNCH(ctx, k_init_pid, grid_for(np + 1), XS_BLOCK, 0, s, lo, hi, pid_ops, np + 1);
  XS_CUDA(cudaMemsetAsync(group_ops, 0, (ng + 1) * sizeof(int), s));
  if (n > 0) {
    ProfScope ps(ctx, ST_PASS1, s);
    const uint8_t* hasint = (check_api && prof) ? prof->has_internal : nullptr;
    int check = (check_api && prof && ev->n_names > 0 && hasint) ? 1 : 0;
    if (check_api && prof && !hasint) check = 0;
    XS_LAUNCH(ctx, k_pass1, grid_for(n, XS_BLOCK * P1_ITEMS), XS_BLOCK, 0, s, v, n, ev->pid_has_meta, hasint,
              check, st, lo, hi, pid_ops, group_ops);
  }
  XS_LAUNCH(ctx, k_pid_finish, grid_for(np + 1), XS_BLOCK, 0, s, lo, hi, np, ev->group_pid, group_ops, ng,
            pid_group0, st);
  return XS_OK;
}

int stage_events(xs_ctx* ctx, const EventView& v, cudaStream_t s, bool need_corr_table, bool check_api,
                 const xs_profile_t* prof) {
  XS_TRY(stage_events_async(ctx, v, s, check_api, prof));
  XS_TRY(fetch_stats(ctx, s));
  if (ctx->h_stats->n_bad) return XS_INVALID_TRACE;
  if (!need_corr_table) return XS_OK;
  return stage_corr_table(ctx, v, s);
}

// (pid, correlation) table build + GPU-event query; no host sync (capturable)
int stage_corr_table(xs_ctx* ctx, const EventView& v, cudaStream_t s) {
  const xs_events_t* ev = &v.ev;
  const int64_t n = ev->n;
  Stats* st = (Stats*)ctx->ptr[W_STATS];
  long long napi = ctx->h_stats->n_api_corr;
  long long ngpu = ctx->h_stats->n_gpu_corr;
  if (ngpu == 0) return XS_OK;
  uint64_t cap = 64;
  while (cap < (uint64_t)(2 * napi + 2)) cap <<= 1;
  int *state, *kpid;
  int64_t *key, *kstart;
  XS_TRY(ws(ctx, W_CORR_STATE, cap, s, &state));
  XS_TRY(ws(ctx, W_CORR_KEY, cap, s, &key));
  XS_TRY(ws(ctx, W_CORR_PID, cap, s, &kpid));
  XS_TRY(ws(ctx, W_CORR_START, cap, s, &kstart));
  XS_CUDA(cudaMemsetAsync(state, 0, cap * sizeof(int), s));
  int64_t* launch = nullptr;
  XS_TRY(ws(ctx, W_FIXED_LS, n + 1, s, &launch));
  if (napi) XS_LAUNCH(ctx, k_corr_insert, grid_for(n), XS_BLOCK, 0, s, v, n, state, key, kpid, kstart, cap - 1, st);
  XS_LAUNCH(ctx, k_corr_query, grid_for(n), XS_BLOCK, 0, s, v, n, state, key, kpid, kstart, cap - 1, st, launch);
  return XS_OK;
}

}  // namespace xs
