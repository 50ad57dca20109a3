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

constexpr int P1_ITEMS = 16;

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

// Per-thread pass-1 accumulators.  Small counts are packed four to a 64-bit
// word in 16-bit lanes (a thread sees P1_ITEMS <= 64 events, a warp <= 2048,
// so no lane overflows a warp reduction) and unpacked once per warp.
struct P1Acc {
  unsigned long long cat_all0 = 0, cat_all1 = 0, cat_nz0 = 0, cat_nz1 = 0;  // categories 0-3 / 4-5
  unsigned long long cnt0 = 0;  // bad, nonzero, ops_nz, ops
  unsigned long long cnt1 = 0;  // api, api_corr, gpu_corr
  long long bad_api = INT64_MAX;
  int cur_p = -1, cur_pops = 0;
  // per-(pid, tid) group op counts: a 4-entry register cache (ops of several
  // tids interleave in row order; flushing on every group switch would hammer
  // a handful of global counters with atomics)
  int gk[4] = {-1, -1, -1, -1}, gc[4] = {0, 0, 0, 0};
  long long lo = 0, hi = 0;
};

__device__ __forceinline__ void p1_visit(P1Acc& A, int64_t i, int64_t s, int64_t d, int p, int c, bool meta,
                                         int g, unsigned hc, int nm, int64_t* lo_out, int64_t* hi_out,
                                         int* pid_ops, int* group_ops, const uint8_t* has_internal, int check_api) {
  const int64_t dd = d > 0 ? d : 0;
  const unsigned bad = (d < 0) + (s < 0) + (s > 0 && dd > INT64_MAX - s) + !meta;
  const int64_t e = (int64_t)((uint64_t)s + (uint64_t)d);
  if (p != A.cur_p) {
    if (A.cur_p >= 0) {
      atomic_min_i64(&lo_out[A.cur_p], A.lo);
      atomic_max_i64(&hi_out[A.cur_p], A.hi);
      if (A.cur_pops) atomicAdd(&pid_ops[A.cur_p], A.cur_pops);
    }
    A.cur_p = p;
    A.lo = s;
    A.hi = e;
    A.cur_pops = 0;
  } else {
    A.lo = s < A.lo ? s : A.lo;
    A.hi = e > A.hi ? e : A.hi;
  }
  const bool nzd = d > 0;
  const unsigned long long one = 1ull << (16 * (c & 3));
  if (c < 4) {
    A.cat_all0 += one;
    A.cat_nz0 += nzd ? one : 0ull;
  } else {
    A.cat_all1 += one;
    A.cat_nz1 += nzd ? one : 0ull;
  }
  A.cnt0 += (unsigned long long)bad | ((unsigned long long)nzd << 16) |
            ((unsigned long long)(c == 0 && nzd) << 32) | ((unsigned long long)(c == 0) << 48);
  if (c == 0) {
    if (nzd) {
      A.cur_pops++;
      if (g == A.gk[0]) {
        A.gc[0]++;
      } else if (g == A.gk[1]) {
        A.gc[1]++;
      } else if (g == A.gk[2]) {
        A.gc[2]++;
      } else if (g == A.gk[3]) {
        A.gc[3]++;
      } else {  // evict the last slot, insert at the front
        if (A.gk[3] >= 0 && A.gc[3]) atomicAdd(&group_ops[A.gk[3]], A.gc[3]);
        A.gk[3] = A.gk[2], A.gc[3] = A.gc[2];
        A.gk[2] = A.gk[1], A.gc[2] = A.gc[1];
        A.gk[1] = A.gk[0], A.gc[1] = A.gc[0];
        A.gk[0] = g, A.gc[0] = 1;
      }
    }
  } else if (c == 4) {
    A.cnt1 += 1ull | ((unsigned long long)hc << 16);
    if (check_api && !has_internal[nm]) A.bad_api = i < A.bad_api ? i : A.bad_api;
  } else if (c == 5) {
    A.cnt1 += (unsigned long long)hc << 32;
  }
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

constexpr int P1_VEC = 4;
#ifndef XS_P1_UNROLL
#define XS_P1_UNROLL 2
#endif
constexpr int kP1Unroll = XS_P1_UNROLL;  // vector steps in flight per thread  // events per vector step (16-byte loads)

// One streaming pass; each thread takes P1_ITEMS consecutive events in
// vector steps of 4 (16-byte loads of start/dur/pid, one 4-byte load of the
// categories) when the columns are aligned for it.  Counters reduce per warp
// into shared memory, then one global atomic per counter per CTA.
#ifndef XS_PASS1_MINB
#define XS_PASS1_MINB 1
#endif
template <bool kVec>
__global__ void __launch_bounds__(XS_BLOCK, XS_PASS1_MINB) k_pass1(EventView v, int64_t n, const uint8_t* __restrict__ has_meta,
                                                    const uint8_t* __restrict__ has_internal, int check_api,
                                                    Stats* st, int64_t* lo_out, int64_t* hi_out, int* pid_ops,
                                                    int* group_ops, uint8_t* tflag) {
  __shared__ unsigned long long s_cnt[20];  // cat_all[6], cat_nz[6], bad, nz, ops_nz, ops, api, api_corr, gpu_corr
  __shared__ long long s_bad_api;
  if (threadIdx.x < 20) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_bad_api = INT64_MAX;
  P1Acc A;
  int last_tg = -1;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  __syncthreads();  // s_cnt initialised
  // persistent CTAs over "virtual blocks" of XS_BLOCK * P1_ITEMS events: the
  // per-CTA global atomics on the ~20 shared counters happen once per CTA,
  // not once per 4096 events (same-address atomics serialise in L2)
  const int64_t nvb = (n + (int64_t)XS_BLOCK * P1_ITEMS - 1) / ((int64_t)XS_BLOCK * P1_ITEMS);
  // each CTA walks a contiguous run of virtual blocks, so a thread's running
  // pid only changes at pid boundaries (every change costs global atomics)
  const int64_t per = (nvb + gridDim.x - 1) / gridDim.x;
  const int64_t vb_end = (blockIdx.x + 1) * per < nvb ? (blockIdx.x + 1) * per : nvb;
#pragma unroll 1
  for (int64_t vb = blockIdx.x * per; vb < vb_end; vb++) {
  const int64_t tbase = (vb * XS_BLOCK + threadIdx.x) * P1_ITEMS;
#pragma unroll kP1Unroll
  for (int step = 0; step < P1_ITEMS / P1_VEC; step++) {
    const int64_t i0 = tbase + step * P1_VEC;
    if (i0 >= n) break;
    int64_t s[4], d[4];
    int p[4], c[4], g[4], nm[4];
    unsigned hc[4];
    int cnt = 4;
    if (kVec && i0 + 4 <= n) {
      // every column the visit may need, loaded up front (independent vector
      // loads instead of per-event dependent ones)
      const int4 g4 = *reinterpret_cast<const int4*>(v.ev.tid + i0);
      const int4 n4 = *reinterpret_cast<const int4*>(v.ev.name + i0);
      const uint32_t h4 = *reinterpret_cast<const uint32_t*>(v.ev.has_corr + i0);
      g[0] = g4.x, g[1] = g4.y, g[2] = g4.z, g[3] = g4.w;
      nm[0] = n4.x, nm[1] = n4.y, nm[2] = n4.z, nm[3] = n4.w;
#pragma unroll
      for (int k = 0; k < 4; k++) hc[k] = (h4 >> (8 * k)) & 0xFFu;
      const longlong2 s01 = *reinterpret_cast<const longlong2*>(v.start + i0);
      const longlong2 s23 = *reinterpret_cast<const longlong2*>(v.start + i0 + 2);
      const longlong2 d01 = *reinterpret_cast<const longlong2*>(v.dur + i0);
      const longlong2 d23 = *reinterpret_cast<const longlong2*>(v.dur + i0 + 2);
      const int4 p4 = *reinterpret_cast<const int4*>(v.ev.pid + i0);
      const uint32_t c4 = *reinterpret_cast<const uint32_t*>(v.ev.cat + i0);
      s[0] = s01.x, s[1] = s01.y, s[2] = s23.x, s[3] = s23.y;
      d[0] = d01.x, d[1] = d01.y, d[2] = d23.x, d[3] = d23.y;
      p[0] = p4.x, p[1] = p4.y, p[2] = p4.z, p[3] = p4.w;
#pragma unroll
      for (int k = 0; k < 4; k++) c[k] = (int)((c4 >> (8 * k)) & 0xFFu);
    } else {
      cnt = (int)(n - i0 < 4 ? n - i0 : 4);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (k < cnt) {
          s[k] = v.start[i0 + k];
          d[k] = v.dur[i0 + k];
          p[k] = v.ev.pid[i0 + k];
          c[k] = v.ev.cat[i0 + k];
          g[k] = v.ev.tid[i0 + k];
          nm[k] = v.ev.name[i0 + k];
          hc[k] = v.ev.has_corr[i0 + k];
        }
      }
    }
    int mp = -1;
    bool meta = false;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      if (k < cnt) {
        if (p[k] != mp) {
          mp = p[k];
          meta = has_meta[mp] != 0;
        }
        p1_visit(A, i0 + k, s[k], d[k], p[k], c[k], meta, g[k], hc[k], nm[k], lo_out, hi_out, pid_ops, group_ops,
                 has_internal, check_api);
        // group carries transition records: a cached read first, so the hot
        // groups are written once, not by every event
        if (c[k] >= 1 && c[k] <= 4 && g[k] != last_tg) {
          last_tg = g[k];
          if (!tflag[last_tg]) tflag[last_tg] = 1;
        }
      }
    }
  }
  // fold this virtual block's packed counters (16-bit lanes) into shared memory
  {
    const unsigned long long w0 = warp_sum_u64(A.cat_all0), w1 = warp_sum_u64(A.cat_all1),
                             w2 = warp_sum_u64(A.cat_nz0), w3 = warp_sum_u64(A.cat_nz1),
                             w4 = warp_sum_u64(A.cnt0), w5 = warp_sum_u64(A.cnt1);
    if (lane < 19) {
      // counter layout: 0-5 cat_all, 6-11 cat_nz, 12-15 cnt0 lanes, 16-18 cnt1 lanes
      const unsigned long long word = lane < 4 ? w0 : lane < 6 ? w1 : lane < 10 ? w2 : lane < 12 ? w3 : lane < 16 ? w4 : w5;
      const int sub = lane < 6 ? (lane & 3) : lane < 12 ? ((lane - 6) & 3) : lane < 16 ? lane - 12 : lane - 16;
      const unsigned long long x = (word >> (16 * sub)) & 0xFFFFull;
      if (x) atomicAdd(&s_cnt[lane], x);
    }
    A.cat_all0 = A.cat_all1 = A.cat_nz0 = A.cat_nz1 = A.cnt0 = A.cnt1 = 0;
  }
  }  // virtual blocks
  // running per-pid span / op count: warp-aggregate when the warp agrees,
  // then block-aggregate warps that share a pid (one atomic per pid per CTA)
  __shared__ int s_wp[XS_BLOCK / 32];
  __shared__ long long s_wl[XS_BLOCK / 32], s_wh[XS_BLOCK / 32], s_wo[XS_BLOCK / 32];
  const int p0 = __shfl_sync(full, A.cur_p, 0);
  const int warp = threadIdx.x >> 5;
  if (__all_sync(full, A.cur_p == p0)) {
    long long l = A.lo, h = A.hi;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const long long l2 = __shfl_xor_sync(full, l, o), h2 = __shfl_xor_sync(full, h, o);
      l = l2 < l ? l2 : l;
      h = h2 > h ? h2 : h;
    }
    const long long po = warp_sum(A.cur_pops);
    if (lane == 0) {
      s_wp[warp] = p0;
      s_wl[warp] = l;
      s_wh[warp] = h;
      s_wo[warp] = po;
    }
  } else {
    if (lane == 0) s_wp[warp] = -1;
    if (A.cur_p >= 0) {
      atomic_min_i64(&lo_out[A.cur_p], A.lo);
      atomic_max_i64(&hi_out[A.cur_p], A.hi);
      if (A.cur_pops) atomicAdd(&pid_ops[A.cur_p], A.cur_pops);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int cp = -1;
    long long cl = 0, ch = 0, co = 0;
    for (int w = 0; w <= XS_BLOCK / 32; w++) {
      const int wp = w < XS_BLOCK / 32 ? s_wp[w] : -2;
      if (wp != cp || w == XS_BLOCK / 32) {
        if (cp >= 0) {
          atomic_min_i64(&lo_out[cp], cl);
          atomic_max_i64(&hi_out[cp], ch);
          if (co) atomicAdd(&pid_ops[cp], (int)co);
        }
        cp = wp;
        if (wp >= 0) cl = s_wl[w], ch = s_wh[w], co = s_wo[w];
      } else if (wp >= 0) {
        cl = s_wl[w] < cl ? s_wl[w] : cl;
        ch = s_wh[w] > ch ? s_wh[w] : ch;
        co += s_wo[w];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; q++) {  // group op counts: one add per distinct group per warp
    const int gk = A.gc[q] ? A.gk[q] : -1;
    const unsigned act = __ballot_sync(full, gk >= 0);
    if (gk >= 0) {
      const unsigned peers = __match_any_sync(act, gk);
      const int sum = (int)__reduce_add_sync(peers, (unsigned)A.gc[q]);
      if (lane == __ffs(peers) - 1) atomicAdd(&group_ops[gk], sum);
    }
  }
  long long bad_api = A.bad_api;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const long long b2 = __shfl_xor_sync(full, bad_api, o);
    bad_api = b2 < bad_api ? b2 : bad_api;
  }
  if (lane == 0 && bad_api != INT64_MAX) atomicMin(&s_bad_api, bad_api);
  __syncthreads();
  if (threadIdx.x < 19) {
    const unsigned long long x = s_cnt[threadIdx.x];
    if (x) {
      const int q = threadIdx.x;
      long long* f = q < 6 ? &st->cat_all[q] : q < 12 ? &st->cat_nz[q - 6] : q == 12 ? &st->n_bad
                   : q == 13 ? &st->n_nonzero : q == 14 ? &st->n_ops_nz : q == 15 ? &st->n_ops
                   : q == 16 ? &st->n_api : q == 17 ? &st->n_api_corr : &st->n_gpu_corr;
      unsigned long long* dst = (unsigned long long*)f;
      atomicAdd(dst, x);
    }
  } else if (threadIdx.x == 32 && s_bad_api != INT64_MAX) {
    atomicMin(&st->bad_api, s_bad_api);
  }
}

// per-pid span reduction for the max key width; also counts multi-tid op pids.
// One warp per pid: a pid's groups (hundreds of GPU-stream tids in skewed
// traces) are counted lane-strided.
__global__ void k_pid_finish(const int64_t* lo, const int64_t* hi, int np, const int32_t* group_pid,
                             const int* group_ops, const uint8_t* tflag, int ng, int* pid_group0, Stats* st) {
  const int p = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (p > np) return;
  if (lane == 0 && p < np && lo[p] != INT64_MAX) atomicMax(&st->max_span, (long long)(hi[p] - lo[p]));
  // first group of each pid (groups are sorted by pid): binary search
  int a = 0, b = ng;
  while (a < b) {
    int m = (a + b) >> 1;
    if (group_pid[m] < p) a = m + 1;
    else b = m;
  }
  if (lane == 0) pid_group0[p] = a;
  if (p == np) return;
  int cnt = 0, tcnt = 0;
  for (int g = a + lane; g < ng && group_pid[g] == p; g += 32) {
    cnt += group_ops[g] > 0;
    tcnt += tflag[g] != 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    tcnt += __shfl_xor_sync(0xffffffffu, tcnt, o);
  }
  if (lane) return;
  if (tcnt) atomicAdd((unsigned long long*)&st->pad[6], (unsigned long long)tcnt);  // transition-key groups
  if (cnt > 1) atomicAdd((unsigned long long*)&st->multi_op_pids, 1ull);
  if (cnt) atomicAdd((unsigned long long*)&st->pad[5], (unsigned long long)cnt);  // groups carrying ops
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

// One slot per entry, one DRAM sector per probe: key, pid and claim state
// (+ the min launch start when CORRELATION needs it) live together.  The
// dangling-correlation check alone (INSTANT, validation, correction) uses
// the 16-byte set slots below: half the table to clear and probe.
struct __align__(32) CorrSlot {
  int64_t key;
  int64_t start;
  int pid;
  int state;  // 0 empty, 1 being claimed, 2 published
  int64_t pad;
};

template <class Slot, bool kStart>
__global__ void k_corr_insert(EventView v, int64_t n, Slot* tab, uint64_t mask, Stats* st) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (v.ev.cat[i] != 4 || !v.ev.has_corr[i]) return;
  int p = v.ev.pid[i];
  int64_t corr = v.ev.corr[i];
  uint64_t h = corr_hash(p, corr) & mask;
  for (uint64_t probe = 0; probe <= mask; probe++) {
    Slot* e = tab + h;
    volatile int* sp = &e->state;
    int cur = *sp;
    if (cur == 0) {
      if (atomicCAS(&e->state, 0, 1) == 0) {
        e->key = corr;
        e->pid = p;
        if constexpr (kStart) reinterpret_cast<CorrSlot*>(e)->start = v.start[i];
        __threadfence();
        atomicExch(&e->state, 2);
        return;
      }
      cur = *sp;
    }
    while (cur == 1) cur = *sp;
    __threadfence();
    if (((volatile int64_t*)&e->key)[0] == corr && ((volatile int*)&e->pid)[0] == p) {
      if constexpr (kStart) atomic_min_i64(&reinterpret_cast<CorrSlot*>(e)->start, v.start[i]);
      return;
    }
    h = (h + 1) & mask;
  }
  atomicAdd((unsigned long long*)&st->table_full, 1ull);
}

// Set-only table (the dangling check): a slot is {correlation id, pid tag};
// one 128-bit compare-and-swap claims or matches it (no claim state, no
// fences).  The tag is never 0, so {0, 0} marks an empty slot.
__device__ __forceinline__ uint64_t corr_tag(int p) { return (uint64_t)(uint32_t)p | (1ull << 32); }

__device__ __forceinline__ void cas_b128(longlong2* addr, long long cmp_lo, long long cmp_hi, long long new_lo,
                                         long long new_hi, long long* old_lo, long long* old_hi) {
  asm volatile(
      "{\n\t.reg .b128 d, c, n;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 n, {%4, %5};\n\t"
      "atom.global.cas.b128 d, [%6], c, n;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(*old_lo), "=l"(*old_hi)
      : "l"(cmp_lo), "l"(cmp_hi), "l"(new_lo), "l"(new_hi), "l"(addr)
      : "memory");
}

__global__ void k_corr_set_insert(EventView v, int64_t n, longlong2* tab, uint64_t mask, Stats* st) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (v.ev.cat[i] != 4 || !v.ev.has_corr[i]) return;
  int p = v.ev.pid[i];
  long long corr = v.ev.corr[i];
  long long tag = (long long)corr_tag(p);
  uint64_t h = corr_hash(p, corr) & mask;
  for (uint64_t probe = 0; probe <= mask; probe++) {
    long long lo, hi;
    cas_b128(tab + h, 0, 0, corr, tag, &lo, &hi);
    if (hi == 0 || (lo == corr && hi == tag)) return;
    h = (h + 1) & mask;
  }
  atomicAdd((unsigned long long*)&st->table_full, 1ull);
}

__global__ void k_corr_set_query(EventView v, int64_t n, const longlong2* tab, uint64_t mask, Stats* st) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (v.ev.cat[i] != 5 || !v.ev.has_corr[i]) return;
  int p = v.ev.pid[i];
  long long corr = v.ev.corr[i];
  long long tag = (long long)corr_tag(p);
  uint64_t h = corr_hash(p, corr) & mask;
  for (uint64_t probe = 0; probe <= mask; probe++) {
    const longlong2 e = tab[h];
    if (e.y == 0) break;
    if (e.x == corr && e.y == tag) return;
    h = (h + 1) & mask;
  }
  atomicAdd((unsigned long long*)&st->n_bad, 1ull);
}

// GPU events: dangling check; in CORRELATION mode record the launch instant
template <class Slot, bool kStart>
__global__ void k_corr_query(EventView v, int64_t n, const Slot* tab, uint64_t mask, Stats* st,
                             int64_t* launch_start) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (v.ev.cat[i] != 5) return;
  if (!v.ev.has_corr[i]) {
    if (kStart) launch_start[i] = INT64_MIN;
    return;
  }
  int p = v.ev.pid[i];
  int64_t corr = v.ev.corr[i];
  uint64_t h = corr_hash(p, corr) & mask;
  for (uint64_t probe = 0; probe <= mask; probe++) {
    const Slot e = tab[h];
    if (e.state == 0) break;
    if (e.key == corr && e.pid == p) {
      if constexpr (kStart) launch_start[i] = reinterpret_cast<const CorrSlot&>(e).start;
      return;
    }
    h = (h + 1) & mask;
  }
  atomicAdd((unsigned long long*)&st->n_bad, 1ull);
  if (kStart) launch_start[i] = INT64_MIN;
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
  uint8_t* tflag;  // groups with HIGH_LEVEL/BACKEND/SIMULATOR/ACCEL_API events (dense transition-key groups)
  XS_TRY(ws(ctx, W_TGRP_FLAG, ng + 1, s, &tflag));
  XS_TRY(fill_many(ctx, s, {{group_ops, (unsigned long long)(ng + 1) * sizeof(int), 0}, {tflag, (unsigned long long)ng + 1, 0}}));
  if (n > 0) {
    ProfScope ps(ctx, ST_PASS1, s);
    const uint8_t* hasint = (check_api && prof) ? prof->has_internal : nullptr;
    int check = (check_api && prof && ev->n_names > 0 && hasint) ? 1 : 0;
    if (check_api && prof && !hasint) check = 0;
    const int p1_grid = std::min(grid_for(n, XS_BLOCK * P1_ITEMS), 148 * 8);  // persistent CTAs
    const bool vec = ((uintptr_t)v.start % 16 == 0) && ((uintptr_t)v.dur % 16 == 0) &&
                     ((uintptr_t)ev->pid % 16 == 0) && ((uintptr_t)ev->cat % 4 == 0) &&
                     ((uintptr_t)ev->tid % 16 == 0) && ((uintptr_t)ev->name % 16 == 0) &&
                     ((uintptr_t)ev->has_corr % 4 == 0);
    if (vec)
      XS_LAUNCH(ctx, k_pass1<true>, p1_grid, XS_BLOCK, 0, s, v, n, ev->pid_has_meta, hasint,
                check, st, lo, hi, pid_ops, group_ops, tflag);
    else
      XS_LAUNCH(ctx, k_pass1<false>, p1_grid, XS_BLOCK, 0, s, v, n, ev->pid_has_meta,
                hasint, check, st, lo, hi, pid_ops, group_ops, tflag);
  }
  XS_LAUNCH(ctx, k_pid_finish, grid_for((int64_t)(np + 1) * 32), XS_BLOCK, 0, s, lo, hi, np, ev->group_pid, group_ops, tflag, ng,
            pid_group0, st);
  return XS_OK;
}

int stage_events(xs_ctx* ctx, const EventView& v, cudaStream_t s, bool need_corr_table, bool check_api,
                 const xs_profile_t* prof) {
  XS_TRY(stage_events_async(ctx, v, s, check_api, prof));
  XS_TRY(fetch_stats(ctx, s));
  if (ctx->h_stats->n_bad) return XS_INVALID_TRACE;
  if (!need_corr_table) return XS_OK;
  return stage_corr_table(ctx, v, s, false);
}

// (pid, correlation) table build + GPU-event query; no host sync (capturable)
int stage_corr_table(xs_ctx* ctx, const EventView& v, cudaStream_t s, bool need_start) {
  const xs_events_t* ev = &v.ev;
  const int64_t n = ev->n;
  Stats* st = (Stats*)ctx->ptr[W_STATS];
  long long napi = ctx->h_stats->n_api_corr;
  long long ngpu = ctx->h_stats->n_gpu_corr;
  if (ngpu == 0) return XS_OK;
  uint64_t cap = 64;
  while (cap < (uint64_t)(2 * napi + 2)) cap <<= 1;
  if (need_start) {  // CORRELATION: launch instants per GPU event
    CorrSlot* tab;
    XS_TRY(ws(ctx, W_CORR_STATE, cap, s, &tab));
    XS_CUDA(cudaMemsetAsync(tab, 0, cap * sizeof(CorrSlot), s));
    int64_t* launch = nullptr;
    XS_TRY(ws(ctx, W_FIXED_LS, n + 1, s, &launch));
    if (napi) XS_LAUNCH(ctx, (k_corr_insert<CorrSlot, true>), grid_for(n), XS_BLOCK, 0, s, v, n, tab, cap - 1, st);
    XS_LAUNCH(ctx, (k_corr_query<CorrSlot, true>), grid_for(n), XS_BLOCK, 0, s, v, n, tab, cap - 1, st, launch);
  } else {  // the dangling-correlation rule only
    longlong2* tab;
    XS_TRY(ws(ctx, W_CORR_KEY, cap, s, &tab));
    XS_CUDA(cudaMemsetAsync(tab, 0, cap * sizeof(longlong2), s));
    if (napi) XS_LAUNCH(ctx, k_corr_set_insert, grid_for(n), XS_BLOCK, 0, s, v, n, tab, cap - 1, st);
    XS_LAUNCH(ctx, k_corr_set_query, grid_for(n), XS_BLOCK, 0, s, v, n, tab, cap - 1, st);
  }
  return XS_OK;
}

}  // namespace xs
