// xs_synth.cu -- device synthetic generator (TEST / BENCH INFRASTRUCTURE,
// SURVEY 8(f4)): the DDPG-style workload of synth.ddpg_trace /
// synth.config3_trace with the reference generator's shape (_build_pid /
// _instrument_pid, synth.py:246-375), generated on the
// device so 1B-event configurations build in about a second instead of
// minutes of host time.  Random streams are a counter hash of (seed, pid,
// iteration, draw), not CPython's `random` (parity never depends on them:
// the checkers run on the generated trace itself).
//
// Per pid: iterations of [glue, phase ops (inference: 3 BACKEND calls x 2
// ACCEL_API, simulation: 5 SIMULATOR calls, backprop: 2 BACKEND calls x 4
// ACCEL_API)], each API launching a correlated kernel with probability 0.7
// on one in-order GPU stream (E_k = max(api_start + 500, E_{k-1}) + d_k),
// optional outer op per iteration and phase ops mirrored on tid 1, and one
// ambient HIGH_LEVEL event.  Both twins come out at once: the uninstrumented
// timeline and the instrumented one, x -> x + (amounts of the hook sites
// anchored strictly before x) (InsertionMap, _timeline.py:70-81), GPU events
// shifted only.  With the same constant amounts correct_trace maps the
// instrumented twin back exactly (tests/test_gpu_synth.py).
//
// K1 per (pid, iteration): walk the iteration (every draw in a fixed order,
//    so later walks see the same iteration) -> length, kernels, site total.
// K2 per pid: sequential scans over its iterations (time, rows, kernels,
//    site prefix).
// K3 per (pid, iteration): collect the iteration's sites (time ordered), walk
//    again writing the CPU events of both twins and the kernel launches.
// K4 per pid: the in-order GPU stream over its kernels (sequential max-plus).
// K5 per kernel: the GPU event; its instrumented start re-walks the iteration
//    that holds it.  K6 per pid: the ambient event and the per-twin spans.
#include "xs_engine.cuh"

namespace xs {
namespace {

// symbolic names (the host maps them to ranks of the sorted name table)
enum SynName { NM_KERNEL = 0, NM_SCRIPT, NM_LAUNCH, NM_MEMCPY, NM_INF, NM_INF_B, NM_SIM, NM_SIM_S, NM_BP, NM_BP_B,
               NM_OUTER, NM_COUNT };

struct Phase {
  int op, call, level, calls, apis;
};
__constant__ Phase c_phases[3] = {{NM_INF, NM_INF_B, 2, 3, 2}, {NM_SIM, NM_SIM_S, 3, 5, 0}, {NM_BP, NM_BP_B, 2, 2, 4}};
constexpr int N_PHASES = 3;
enum { GLUE = 0, BACKEND_D, SIMULATOR_D, API_D, API_GAP, KERNEL_D };
__constant__ int c_lo[6] = {1500, 20000, 50000, 5000, 1000, 10000};
__constant__ int c_hi[6] = {2500, 60000, 150000, 15000, 3000, 40000};
constexpr int LAUNCH_DELAY = 500;
constexpr double KERNEL_PROB = 0.7;
constexpr int MAX_SITES = 64;  // per iteration (52 with the outer op and the tid-1 mirror)

__device__ __forceinline__ uint64_t mix(uint64_t z) {  // splitmix64
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Rng {
  uint64_t base;
  uint32_t k;
  __device__ Rng(uint64_t seed, int64_t pid, int64_t it)
      : base(mix(seed ^ mix((uint64_t)pid * 0x100000001B3ull) ^ mix(~(uint64_t)it))), k(0) {}
  __device__ uint64_t next() { return mix(base + (uint64_t)(k++) * 0x632BE59BD9B4E019ull); }
  __device__ int64_t uni(int key) {
    const uint64_t span = (uint64_t)(c_hi[key] - c_lo[key] + 1);
    return c_lo[key] + (int64_t)(next() % span);
  }
  __device__ double unit() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

struct Spec {
  int64_t iterations;
  uint64_t seed;
  int32_t n_pids, outer, tid2, first_pid;
  int64_t ann_start, ann_end, transition, interception, launch, memcpy;
  const int32_t* names;  // [NM_COUNT] name ranks
};

// One iteration starting at time t, in time order: kind 0 op (start, end,
// name, tid), 1 call (start, end, name, level), 2 api (start, end, sel,
// has_kernel, kernel duration), 3 site (anchor, amount).  Returns its end.
template <class F>
__device__ int64_t walk_iteration(const Spec& sp, int64_t pid, int64_t it, int64_t t, F&& emit) {
  Rng r(sp.seed, sp.first_pid + pid, it);
  t += r.uni(GLUE);
  const int64_t it_op0 = t;
  for (int ph = 0; ph < N_PHASES; ph++) {
    const Phase P = c_phases[ph];
    const int64_t os = t;
    if (ph == 0 && sp.outer) emit(3, t, sp.ann_start, 0, 0, 0);  // (sites of ops starting together)
    emit(3, t, sp.ann_start, 0, 0, 0);
    if (sp.tid2) emit(3, t, sp.ann_start, 0, 0, 0);
    t += r.uni(GLUE);
    for (int c = 0; c < P.calls; c++) {
      const int64_t cs = t;
      emit(3, cs, sp.transition, 0, 0, 0);
      if (P.level == 2 && P.apis > 0) {
        t += r.uni(API_GAP);
        for (int a = 0; a < P.apis; a++) {
          const int64_t as = t;
          t += r.uni(API_D);
          const int sel = (int)(r.next() & 1ull);
          const bool hk = r.unit() < KERNEL_PROB;
          const int64_t kd = r.uni(KERNEL_D);
          emit(3, as, sp.interception, 0, 0, 0);
          emit(3, as, sel ? sp.memcpy : sp.launch, 0, 0, 0);
          emit(2, as, t, sel, hk ? 1 : 0, kd);
          t += r.uni(API_GAP);
        }
      } else {
        t += r.uni(P.level == 2 ? BACKEND_D : SIMULATOR_D);
      }
      emit(1, cs, t, P.call, P.level, 0);
      t += r.uni(GLUE);
    }
    emit(0, os, t, P.op, 0, 0);
    if (sp.tid2) emit(0, os, t, P.op, 1, 0);
    if (ph == N_PHASES - 1 && sp.outer) emit(0, it_op0, t, NM_OUTER, 0, 0);
    emit(3, t, sp.ann_end, 0, 0, 0);
    if (sp.tid2) emit(3, t, sp.ann_end, 0, 0, 0);
    if (ph == N_PHASES - 1 && sp.outer) emit(3, t, sp.ann_end, 0, 0, 0);
  }
  return t;
}

__device__ __forceinline__ int cpu_events_per_iteration(const Spec& sp) {
  int n = 0;
  for (int ph = 0; ph < N_PHASES; ph++) n += (sp.tid2 ? 2 : 1) + c_phases[ph].calls * (1 + c_phases[ph].apis);
  return n + (sp.outer ? 1 : 0);
}

__device__ __forceinline__ int group_of(const Spec& sp, int p, int local) { return p * (sp.tid2 ? 3 : 2) + local; }

// the iteration's sites, time ordered (cumulative amounts)
struct SiteList {
  int n;
  int64_t anchor[MAX_SITES];
  int64_t cum[MAX_SITES];  // amounts of sites [0, i]
  __device__ void collect(const Spec& sp, int64_t pid, int64_t it, int64_t t0) {
    n = 0;
    int64_t acc = 0;
    walk_iteration(sp, pid, it, t0, [&](int kind, int64_t a, int64_t b, int64_t, int64_t, int64_t) {
      if (kind != 3 || n >= MAX_SITES) return;
      acc += b;
      anchor[n] = a;
      cum[n] = acc;
      n++;
    });
  }
  __device__ int64_t before(int64_t x) const {  // amounts anchored strictly before x
    int lo = 0, hi = n;  // first anchor >= x
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if (anchor[m] < x) lo = m + 1;
      else hi = m;
    }
    return lo ? cum[lo - 1] : 0;
  }
};

__global__ void k_syn_count(Spec sp, int64_t* it_len, int32_t* it_nk, int64_t* it_site) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)sp.n_pids * sp.iterations) return;
  const int64_t p = g / sp.iterations, it = g % sp.iterations;
  int nk = 0;
  int64_t site = 0;
  it_len[g] = walk_iteration(sp, p, it, 0, [&](int kind, int64_t, int64_t b, int64_t, int64_t d, int64_t) {
    if (kind == 2) nk += (int)d;
    if (kind == 3) site += b;
  });
  it_nk[g] = nk;
  it_site[g] = site;
}

__global__ void k_syn_scan(Spec sp, const int64_t* it_len, const int32_t* it_nk, const int64_t* it_site,
                           int64_t* it_t0, int64_t* it_row0, int64_t* it_k0, int64_t* it_s0, int64_t* pid_rows,
                           int64_t* pid_k, int64_t* pid_tend, int64_t* pid_site) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= sp.n_pids) return;
  const int ncpu = cpu_events_per_iteration(sp);
  int64_t t = 0, row = 0, k = 0, s = 0;
  for (int64_t it = 0; it < sp.iterations; it++) {
    const int64_t g = (int64_t)p * sp.iterations + it;
    it_t0[g] = t;
    it_row0[g] = row;
    it_k0[g] = k;
    it_s0[g] = s;
    t += it_len[g];
    row += ncpu + it_nk[g];
    k += it_nk[g];
    s += it_site[g];
  }
  pid_rows[p] = row + 1;  // + the ambient HIGH_LEVEL event
  pid_k[p] = k;
  pid_tend[p] = t;
  pid_site[p] = s;
}

struct Out {
  int64_t *su, *du, *si, *di;  // start / dur: uninstrumented and instrumented twins
  int32_t *pid, *tid, *name;
  uint8_t *cat, *has;
  int64_t* corr;
};

__device__ __forceinline__ void put(const Out& o, int64_t row, int64_t su, int64_t eu, int64_t si, int64_t ei,
                                    int pid, int group, int cat, int name, int64_t corr, int has) {
  o.su[row] = su;
  o.du[row] = eu - su;
  o.si[row] = si;
  o.di[row] = ei - si;
  o.pid[row] = pid;
  o.tid[row] = group;
  o.cat[row] = (uint8_t)cat;
  o.name[row] = name;
  o.corr[row] = corr;
  o.has[row] = (uint8_t)has;
}

__global__ void k_syn_cpu(Spec sp, const int64_t* it_t0, const int64_t* it_row0, const int64_t* it_k0,
                          const int64_t* it_s0, const int64_t* pid_row0, const int64_t* pid_k0, Out o,
                          int64_t* k_launch, int64_t* k_dur, int64_t* k_corr, int64_t* k_row) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)sp.n_pids * sp.iterations) return;
  const int p = (int)(g / sp.iterations);
  const int64_t it = g % sp.iterations;
  SiteList S;
  S.collect(sp, p, it, it_t0[g]);
  const int64_t sh = it_s0[g];
  auto imap = [&](int64_t x) { return x + sh + S.before(x); };
  int64_t row = pid_row0[p] + it_row0[g];
  int64_t krow = row + cpu_events_per_iteration(sp);  // this iteration's kernels follow its CPU events
  int64_t kidx = pid_k0[p] + it_k0[g];
  int64_t corr = it_k0[g];  // correlation ids 1, 2, ... per pid
  walk_iteration(sp, p, it, it_t0[g], [&](int kind, int64_t a, int64_t b, int64_t c, int64_t d, int64_t e) {
    if (kind == 3) return;
    if (kind == 2) {
      const bool hk = d != 0;
      if (hk) corr++;
      put(o, row++, a, b, imap(a), imap(b), p, group_of(sp, p, 0), 4, sp.names[c ? NM_MEMCPY : NM_LAUNCH],
          hk ? corr : 0, hk ? 1 : 0);
      if (hk) {
        k_launch[kidx] = a + LAUNCH_DELAY;
        k_dur[kidx] = e;
        k_corr[kidx] = corr;
        k_row[kidx] = krow++;
        kidx++;
      }
      return;
    }
    if (kind == 1) {
      put(o, row++, a, b, imap(a), imap(b), p, group_of(sp, p, 0), (int)d, sp.names[c], 0, 0);
      return;
    }
    put(o, row++, a, b, imap(a), imap(b), p, group_of(sp, p, (int)d), 0, sp.names[c], 0, 0);
  });
}

__global__ void k_syn_stream(Spec sp, const int64_t* pid_k0, const int64_t* pid_k, const int64_t* k_launch,
                             const int64_t* k_dur, int64_t* k_start, int64_t* pid_kend) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= sp.n_pids) return;
  int64_t e = 0;  // stream cursor (the reference starts it at 0)
  for (int64_t k = pid_k0[p]; k < pid_k0[p] + pid_k[p]; k++) {
    const int64_t s = k_launch[k] > e ? k_launch[k] : e;
    k_start[k] = s;
    e = s + k_dur[k];
  }
  pid_kend[p] = e;
}

__global__ void k_syn_gpu(Spec sp, int64_t n_k, const int64_t* kpid, const int64_t* it_t0, const int64_t* it_s0,
                          const int64_t* k_start, const int64_t* k_dur, const int64_t* k_corr, const int64_t* k_row,
                          Out o) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_k) return;
  const int p = (int)kpid[k];
  const int64_t x = k_start[k];
  // the iteration holding x: last it_t0 <= x of this pid
  const int64_t* t0 = it_t0 + (int64_t)p * sp.iterations;
  int64_t lo = 0, hi = sp.iterations;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (t0[m] <= x) lo = m + 1;
    else hi = m;
  }
  const int64_t it = lo > 0 ? lo - 1 : 0;
  SiteList S;
  S.collect(sp, p, it, t0[it]);
  const int64_t xi = x + it_s0[(int64_t)p * sp.iterations + it] + S.before(x);
  put(o, k_row[k], x, x + k_dur[k], xi, xi + k_dur[k], p, group_of(sp, p, sp.tid2 ? 2 : 1), 5,
      sp.names[NM_KERNEL], k_corr[k], 1);
}

__global__ void k_syn_ambient(Spec sp, const int64_t* pid_row0, const int64_t* pid_rows, const int64_t* pid_tend,
                              const int64_t* pid_kend, const int64_t* pid_site, Out o, int64_t* span) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= sp.n_pids) return;
  Rng r(sp.seed, sp.first_pid + p, -1);
  const int64_t end = (pid_tend[p] > pid_kend[p] ? pid_tend[p] : pid_kend[p]) + r.uni(GLUE);
  const int64_t endi = end + pid_site[p];  // every site precedes the ambient end
  put(o, pid_row0[p] + pid_rows[p] - 1, 0, end, 0, endi, p, group_of(sp, p, 0), 1, sp.names[NM_SCRIPT], 0, 0);
  span[2 * p] = end;
  span[2 * p + 1] = endi;
}

__global__ void k_syn_kpid(const int64_t* pid_k0, int np, int64_t n_k, int64_t* kpid) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_k) return;
  int lo = 0, hi = np;  // last p with pid_k0[p] <= k
  while (lo < hi) {
    const int m = (lo + hi) >> 1;
    if (pid_k0[m] <= k) lo = m + 1;
    else hi = m;
  }
  kpid[k] = lo - 1;
}

__global__ void k_syn_excl(const int64_t* x, int np, int64_t* out) {  // tiny per-pid exclusive scan
  if (blockIdx.x || threadIdx.x) return;
  int64_t acc = 0;
  for (int p = 0; p < np; p++) {
    out[p] = acc;
    acc += x[p];
  }
  out[np] = acc;
}

}  // namespace
}  // namespace xs

using namespace xs;

extern "C" int xs_synth_plan(xs_ctx_t* ctx, const xs_synth_spec_t* spec, int64_t* n_events, xs_stream_t stream) {
  if (!ctx || !spec || !n_events || spec->n_pids <= 0 || spec->iterations <= 0) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Spec sp{spec->iterations, spec->seed, spec->n_pids, spec->outer_op, spec->second_tid_ops, spec->first_pid,
          spec->ann_start, spec->ann_end, spec->transition, spec->interception, spec->launch, spec->memcpy,
          spec->names};
  const int64_t G = (int64_t)sp.n_pids * sp.iterations;
  const int np = sp.n_pids;
  int64_t *it_len, *it_site, *it_t0, *it_row0, *it_k0, *it_s0, *pid;
  int32_t* it_nk;
  XS_TRY(ws(ctx, W_SYN_IT, 6 * G + 8, s, &it_len));
  it_site = it_len + G;
  it_t0 = it_site + G;
  it_row0 = it_t0 + G;
  it_k0 = it_row0 + G;
  it_s0 = it_k0 + G;
  XS_TRY(ws(ctx, W_SYN_NK, G + 1, s, &it_nk));
  XS_TRY(ws(ctx, W_SYN_PID, 10 * (int64_t)(np + 1), s, &pid));  // rows, k, tend, site, row0, k0, kend, span[2]
  XS_LAUNCH(ctx, k_syn_count, grid_for(G), XS_BLOCK, 0, s, sp, it_len, it_nk, it_site);
  XS_LAUNCH(ctx, k_syn_scan, grid_for(np), XS_BLOCK, 0, s, sp, it_len, it_nk, it_site, it_t0, it_row0, it_k0, it_s0,
            pid, pid + (np + 1), pid + 2 * (np + 1), pid + 3 * (np + 1));
  XS_LAUNCH(ctx, k_syn_excl, 1, 32, 0, s, pid, np, pid + 4 * (np + 1));
  XS_LAUNCH(ctx, k_syn_excl, 1, 32, 0, s, pid + (np + 1), np, pid + 5 * (np + 1));
  int64_t tot[2];
  XS_CUDA(cudaMemcpyAsync(&tot[0], pid + 4 * (np + 1) + np, 8, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaMemcpyAsync(&tot[1], pid + 5 * (np + 1) + np, 8, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaStreamSynchronize(s));
  ctx->syn_events = tot[0];
  ctx->syn_kernels = tot[1];
  *n_events = tot[0];
  return XS_OK;
}

extern "C" int xs_synth_generate(xs_ctx_t* ctx, const xs_synth_spec_t* spec, int64_t* start, int64_t* dur,
                                 int64_t* start_inst, int64_t* dur_inst, int32_t* pid_out, int32_t* tid_out,
                                 uint8_t* cat, int32_t* name, int64_t* corr, uint8_t* has_corr, int64_t* span,
                                 xs_stream_t stream) {
  if (!ctx || !spec || ctx->syn_events <= 0) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  Spec sp{spec->iterations, spec->seed, spec->n_pids, spec->outer_op, spec->second_tid_ops, spec->first_pid,
          spec->ann_start, spec->ann_end, spec->transition, spec->interception, spec->launch, spec->memcpy,
          spec->names};
  const int64_t G = (int64_t)sp.n_pids * sp.iterations;
  const int np = sp.n_pids;
  int64_t* it_len = (int64_t*)ctx->ptr[W_SYN_IT];
  int64_t *it_t0 = it_len + 2 * G, *it_row0 = it_len + 3 * G, *it_k0 = it_len + 4 * G, *it_s0 = it_len + 5 * G;
  int64_t* pid = (int64_t*)ctx->ptr[W_SYN_PID];
  int64_t *pid_rows = pid, *pid_k = pid + (np + 1), *pid_tend = pid + 2 * (np + 1), *pid_site = pid + 3 * (np + 1);
  int64_t *pid_row0 = pid + 4 * (np + 1), *pid_k0 = pid + 5 * (np + 1), *pid_kend = pid + 6 * (np + 1);
  const int64_t nk = ctx->syn_kernels;
  int64_t* kb;
  XS_TRY(ws(ctx, W_SYN_K, 6 * (nk + 1), s, &kb));
  int64_t *k_launch = kb, *k_dur = kb + (nk + 1), *k_corr = kb + 2 * (nk + 1), *k_row = kb + 3 * (nk + 1),
          *k_start = kb + 4 * (nk + 1), *kpid = kb + 5 * (nk + 1);
  Out o{start, dur, start_inst, dur_inst, pid_out, tid_out, name, cat, has_corr, corr};
  XS_LAUNCH(ctx, k_syn_cpu, grid_for(G), XS_BLOCK, 0, s, sp, it_t0, it_row0, it_k0, it_s0, pid_row0, pid_k0, o,
            k_launch, k_dur, k_corr, k_row);
  XS_LAUNCH(ctx, k_syn_stream, grid_for(np), XS_BLOCK, 0, s, sp, pid_k0, pid_k, k_launch, k_dur, k_start, pid_kend);
  if (nk > 0) {
    XS_LAUNCH(ctx, k_syn_kpid, grid_for(nk), XS_BLOCK, 0, s, pid_k0, np, nk, kpid);
    XS_LAUNCH(ctx, k_syn_gpu, grid_for(nk), XS_BLOCK, 0, s, sp, nk, kpid, it_t0, it_s0, k_start, k_dur, k_corr,
              k_row, o);
  }
  XS_LAUNCH(ctx, k_syn_ambient, grid_for(np), XS_BLOCK, 0, s, sp, pid_row0, pid_rows, pid_tend, pid_kend, pid_site,
            o, span);
  return XS_OK;
}
