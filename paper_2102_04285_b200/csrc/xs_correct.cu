// xs_correct.cu -- correct_trace (correction.py:79-186, _timeline.py:57-132).
//
// Per pid, in Site.order_key order (anchor, subkind, tid, name; stable):
//   quantize   out_i = floor(S_i) - floor(S_{i-1}), S = running exact sum
//              -> segmented int128 scan of amount*L, floor-divided by L
//   caps       each owner has <= 2 sites, first one fixed by subkind:
//              c1 = min(q1, dur); c2 = min(q2, dur - c1)      (139-153)
//   RemovalMap a_i = max(anchor_i, E_{i-1}), b_i = a_i + len_i,
//              E_i = max(E_{i-1}, b_i) = f_i(E_{i-1}),
//              f_i(x) = max(x + max(0,len_i), anchor_i + len_i): (max,+)
//              affine maps compose associatively -> one segmented scan
//   remap      rmap(y) = y - prefix[k] - (y - a_k if a_k < y), k = #slabs
//              with b <= y (bisect_right) -> one binary search per endpoint
// Site order ties follow the reference's stable sort: sites are generated in
// event-index order (ANN/API sites tie only by index); TRANSITION sites that
// tie on the full key are re-ordered by (category, correlation or -1, index),
// which is the order of the H->B list, then H->S, each sorted by
// Event.sort_key (overlap.py:287-288).
#include <cub/device/device_scan.cuh>

#include "xs_engine.cuh"
#include "xs_prims.cuh"

namespace xs {

enum { ANN_START = 0, TRANSITION_HOOK = 1, API_INTERCEPT = 2, API_INTERNAL = 3, ANN_END = 4 };
enum { H_ANN = 0, H_TRANS = 1, H_IC = 2, H_INT = 3 };

// profile amount row of a site: 0..3 by subkind, 4 + name for API_INTERNAL
__device__ __forceinline__ int amount_row(int sub, int name) {
  switch (sub) {
    case ANN_START: return 0;
    case ANN_END: return 1;
    case TRANSITION_HOOK: return 2;
    case API_INTERCEPT: return 3;
    default: return 4 + name;
  }
}

__global__ void k_site_count(EventView v, int64_t n, const uint8_t* tflag, int* cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = v.ev.cat[i];
  cnt[i] = (c == 0 || c == 4) ? 2 : ((tflag[i] & 3) ? 1 : 0);
}

// slot layout: pos[i] (+1) for event i; primary key (pid | anchor | subkind)
__global__ void k_site_gen(EventView v, int64_t n, const int* cnt, const int* pos, const int64_t* lo, int tb,
                           int* site_ev, int* site_row, uint64_t* k1) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || cnt[i] == 0) return;
  const int c = v.ev.cat[i];
  const int at = pos[i];
  const int p = v.ev.pid[i];
  const uint64_t pb = (uint64_t)p << (tb + 3);
  const uint64_t s_rel = (uint64_t)(v.start[i] - lo[p]);
  if (c == 0) {
    const uint64_t e_rel = s_rel + (uint64_t)v.dur[i];
    site_ev[at] = (int)i;
    site_row[at] = amount_row(ANN_START, 0);
    k1[at] = pb | (s_rel << 3) | ANN_START;
    site_ev[at + 1] = (int)i;
    site_row[at + 1] = amount_row(ANN_END, 0);
    k1[at + 1] = pb | (e_rel << 3) | ANN_END;
  } else if (c == 4) {
    site_ev[at] = (int)i;
    site_row[at] = amount_row(API_INTERCEPT, 0);
    k1[at] = pb | (s_rel << 3) | API_INTERCEPT;
    site_ev[at + 1] = (int)i;
    site_row[at + 1] = amount_row(API_INTERNAL, v.ev.name[i]);
    k1[at + 1] = pb | (s_rel << 3) | API_INTERNAL;
  } else {
    site_ev[at] = (int)i;
    site_row[at] = amount_row(TRANSITION_HOOK, 0);
    k1[at] = pb | (s_rel << 3) | TRANSITION_HOOK;
  }
}

__device__ __forceinline__ int64_t site_anchor(const EventView& v, int i, int sub) {
  return sub == ANN_END ? v.start[i] + v.dur[i] : v.start[i];
}

// After the (pid, anchor, subkind) sort, sites tying on it are ordered by the
// rest of Site.order_key, (tid, name), then by the reference's insertion
// order: event index for ANN/API sites; (category, corr or -1, index) for
// TRANSITION sites (the H->B list, then H->S, each Event.sort_key-ordered).
// Runs are tiny (nested ops starting together, APIs on several tids), so one
// thread insertion-sorts each run.
__device__ __forceinline__ bool site_less(const EventView& v, int ix, int iy, bool transition) {
  const int tx = v.ev.tid[ix], ty = v.ev.tid[iy];
  if (tx != ty) return tx < ty;
  const int nx = v.ev.name[ix], ny = v.ev.name[iy];
  if (nx != ny) return nx < ny;
  if (transition) {
    const int cx = v.ev.cat[ix], cy = v.ev.cat[iy];
    if (cx != cy) return cx < cy;
    const int64_t rx = v.ev.has_corr[ix] ? v.ev.corr[ix] : -1;
    const int64_t ry = v.ev.has_corr[iy] ? v.ev.corr[iy] : -1;
    if (rx != ry) return rx < ry;
  }
  return ix < iy;
}

// sort values = slot ids; the unused tail of the upper-bound site arrays
// ([device count, ns)) gets sentinel keys that sort last
__global__ void k_site_tail(uint64_t* k1, uint32_t* sl, int64_t ns, const int64_t* d_ns) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ns) return;
  sl[q] = (uint32_t)q;
  if (q >= *d_ns) k1[q] = ~0ull;
}

__global__ void k_tie_fix(EventView v, const uint64_t* k1, uint32_t* slot, int64_t ns, const int* site_ev) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  // run starts from one key load per thread: neighbours by shuffle
  const uint64_t k = q < ns ? k1[q] : ~0ull;
  uint64_t kp = __shfl_up_sync(0xffffffffu, k, 1), kn = __shfl_down_sync(0xffffffffu, k, 1);
  if (lane == 0) kp = q > 0 && q < ns ? k1[q - 1] : ~k;
  if (lane == 31) kn = q + 1 < ns ? k1[q + 1] : ~k;
  if (q >= ns || k == ~0ull) return;  // unused upper-bound slots sort last
  if (q > 0 && kp == k) return;
  if (q + 1 >= ns || kn != k) return;
  int64_t e = q + 1;
  while (e < ns && k1[e] == k) e++;
  const bool transition = (k & 7u) == TRANSITION_HOOK;
  for (int64_t a = q + 1; a < e; a++) {
    const uint32_t x = slot[a];
    const int ix = site_ev[x];
    int64_t b = a - 1;
    while (b >= q) {
      const uint32_t y = slot[b];
      if (!site_less(v, ix, site_ev[y], transition)) break;
      slot[b + 1] = y;
      b--;
    }
    slot[b + 1] = x;
  }
}

// the quantize scan's element: the fractional parts' running sum modulo L
// (W little-endian words; L < 2^(64W-1), so a sum of two residues never
// overflows W words), segmented per pid by a head flag
template <int W>
struct SegMod {
  uint64_t w[W];
  int head;
  int pad;
};

template <int W>
__device__ __forceinline__ bool mw_less(const uint64_t* a, const uint64_t* b) {
#pragma unroll
  for (int i = W - 1; i >= 0; i--)
    if (a[i] != b[i]) return a[i] < b[i];
  return false;
}

template <int W>
struct SegModOp {
  uint64_t L[W];
  __device__ SegMod<W> operator()(const SegMod<W>& a, const SegMod<W>& b) const {
    SegMod<W> r;
    r.head = a.head | b.head;
    r.pad = 0;
    if (b.head) {
#pragma unroll
      for (int i = 0; i < W; i++) r.w[i] = b.w[i];
      return r;
    }
    add_mod(a.w, b.w, r.w);
    return r;
  }
  __device__ void add_mod(const uint64_t* a, const uint64_t* b, uint64_t* r) const {
    unsigned long long c = 0;
#pragma unroll
    for (int i = 0; i < W; i++) {  // r = a + b (< 2L <= 2^(64W): no carry out)
      const unsigned long long s = a[i] + c;
      const unsigned long long c1 = s < c;
      r[i] = s + b[i];
      c = c1 + (r[i] < s);
    }
    if (!mw_less<W>(r, L)) {  // r -= L
      unsigned long long br = 0;
#pragma unroll
      for (int i = 0; i < W; i++) {
        const unsigned long long d = r[i] - L[i];
        const unsigned long long b1 = r[i] < L[i];
        r[i] = d - br;
        br = b1 | (d < br);
      }
    }
  }
};

// A thread's ITEMS consecutive site keys and slots (ITEMS % 4 == 0, base a
// multiple of ITEMS): 16-byte loads when the run is whole, scalar at the tail.
// `prev` is the key before the run (head detection without re-reading k1).
template <int ITEMS>
__device__ __forceinline__ void load_site_run(const uint64_t* k1, const uint32_t* slot, int64_t base, int64_t ns,
                                              uint64_t (&kv)[ITEMS], uint32_t (&sv)[ITEMS], uint64_t& prev) {
  static_assert(ITEMS % 4 == 0, "vector site loads need ITEMS % 4 == 0");
  prev = base > 0 && base < ns ? k1[base - 1] : 0;  // (no read past the live keys)
  if (base + ITEMS <= ns) {
#pragma unroll
    for (int j = 0; j < ITEMS; j += 2) {
      const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(k1 + base + j);
      kv[j] = x.x;
      kv[j + 1] = x.y;
    }
#pragma unroll
    for (int j = 0; j < ITEMS; j += 4) {
      const uint4 x = *reinterpret_cast<const uint4*>(slot + base + j);
      sv[j] = x.x;
      sv[j + 1] = x.y;
      sv[j + 2] = x.z;
      sv[j + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
      kv[j] = base + j < ns ? k1[base + j] : 0;
      sv[j] = base + j < ns ? slot[base + j] : 0;
    }
  }
}

// site subkind -> row of the profile's whole / frac tables (API_INTERNAL:
// 4 + the event's name)

#ifndef XS_Q_ITEMS
#define XS_Q_ITEMS 8
#endif
constexpr int Q_ITEMS = XS_Q_ITEMS;
// quantize_amounts (_timeline.py:57-67) per pid in site order:
// q_i = floor(S_i) - floor(S_{i-1}) with S the running sum of exact amounts
// = whole_i + [ P_i < frac_i ], P_i the inclusive running sum of the
// fractional numerators modulo L (a carry past L is exactly the floor step)
template <int W>
__global__ void __launch_bounds__(XS_BLOCK) k_quantize(const uint64_t* k1, const uint32_t* slot, const int64_t* d_ns,
                                                       int tb, EventView v, xs_profile_t pr, const int* site_row,
                                                       int64_t* qslot, TileDesc<SegMod<W>>* desc, int* flags,
                                                       int* tile_ctr) {
  const int tile = next_tile(tile_ctr);
  const int64_t ns = *d_ns;
  if ((int64_t)tile * XS_BLOCK * Q_ITEMS >= ns) return;  // tail tiles of the upper-bound grid
  const int64_t base = (int64_t)tile * XS_BLOCK * Q_ITEMS + (int64_t)threadIdx.x * Q_ITEMS;
  SegModOp<W> op;
#pragma unroll
  for (int i = 0; i < W; i++) op.L[i] = pr.L[i];
  int row[Q_ITEMS];
  int hd[Q_ITEMS];
  SegMod<W> id;
#pragma unroll
  for (int i = 0; i < W; i++) id.w[i] = 0;
  id.head = 0;
  id.pad = 0;
  SegMod<W> agg = id;
  const int pshift = tb + 3;
  uint64_t kv[Q_ITEMS], prevk;
  uint32_t sv[Q_ITEMS];
  load_site_run<Q_ITEMS>(k1, slot, base, ns, kv, sv, prevk);
#pragma unroll
  for (int j = 0; j < Q_ITEMS; j++) {
    const int64_t q = base + j;
    row[j] = -1;
    hd[j] = 0;
    if (q < ns) {
      // the subkind is the key's low 3 bits: only API_INTERNAL sites gather
      // their event (for the API name); the rest are profile constants
      const uint64_t kq = kv[j];
      const int sub = (int)(kq & 7u);
      row[j] = sub == API_INTERNAL ? site_row[sv[j]] : amount_row(sub, 0);
      hd[j] = q == 0 || (prevk >> pshift) != (kq >> pshift);
      prevk = kq;
      SegMod<W> e;
#pragma unroll
      for (int i = 0; i < W; i++) e.w[i] = pr.frac[(int64_t)row[j] * W + i];
      if (hd[j] && pr.residue_in) {  // a window's segment starts from the carried residue
        uint64_t r0[W], f0[W];
        const int64_t pp = (int64_t)(kq >> pshift);
#pragma unroll
        for (int i = 0; i < W; i++) {
          r0[i] = pr.residue_in[pp * W + i];
          f0[i] = e.w[i];
        }
        op.add_mod(r0, f0, e.w);
      }
      e.head = hd[j];
      e.pad = 0;
      agg = op(agg, e);
    }
  }
  SegMod<W> run = grid_exclusive(agg, op, id, tile, desc, flags);
#pragma unroll
  for (int j = 0; j < Q_ITEMS; j++) {
    const int64_t q = base + j;
    if (q >= ns) break;
    uint64_t f[W], after[W];
#pragma unroll
    for (int i = 0; i < W; i++) {
      f[i] = pr.frac[(int64_t)row[j] * W + i];
      if (hd[j]) run.w[i] = pr.residue_in ? pr.residue_in[(int64_t)(k1[q] >> pshift) * W + i] : 0;
    }
    op.add_mod(run.w, f, after);
    const int64_t whole = row[j] < 4 ? pr.whole[row[j]] : pr.internal[row[j] - 4];
    qslot[slot[q]] = whole + (mw_less<W>(after, f) ? 1 : 0);
#pragma unroll
    for (int i = 0; i < W; i++) run.w[i] = after[i];
  }
}

template <int W>
static int launch_quantize(xs_ctx* ctx, int64_t tiles, cudaStream_t s, const uint64_t* k1, const uint32_t* sl,
                           const int64_t* d_ns, int tb, const EventView& v, const xs_profile_t& pr,
                           const int* site_row, int64_t* qslot) {
  TileDesc<SegMod<W>>* desc;
  int *flags, *tctr;
  XS_TRY(ws(ctx, W_QSCAN_DESC, tiles + 1, s, &desc));
  XS_TRY(ws(ctx, W_QSCAN_FLAGS, tiles + 1, s, &flags));
  XS_TRY(ws(ctx, W_TILE_CTR, 4, s, &tctr));
  XS_TRY(fill_many(ctx, s, {{flags, (unsigned long long)(tiles + 1) * sizeof(int), 0}, {tctr, sizeof(int), 0}}));
  XS_LAUNCH(ctx, k_quantize<W>, (int)tiles, XS_BLOCK, 0, s, k1, sl, d_ns, tb, v, pr, site_row, qslot, desc, flags,
            tctr);
  return XS_OK;
}

// per owner: budget caps (correction.py:139-153) + shortfall per (pid, hook);
// shortfalls are summed per warp when the warp's owners share a pid (one
// atomic per hook instead of one per capped site: skewed traces cap often)
__global__ void k_caps(EventView v, int64_t n, const int* cnt, const int* pos, const int64_t* qslot, int64_t* lenslot,
                       int64_t* shortfall) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i - threadIdx.x % 32 >= n) return;  // (whole warps leave together)
  int64_t sf[4] = {0, 0, 0, 0};
  int p = -1;
  if (i < n && cnt[i] != 0) {
    int c = v.ev.cat[i];
    int at = pos[i];
    p = v.ev.pid[i];
    int64_t budget = v.dur[i];
    int64_t q1 = qslot[at];
    int64_t c1 = q1 < budget ? q1 : budget;
    budget -= c1;
    lenslot[at] = c1;
    sf[c == 0 ? H_ANN : (c == 4 ? H_IC : H_TRANS)] += q1 - c1;
    if (cnt[i] == 2) {
      int64_t q2 = qslot[at + 1];
      int64_t c2 = q2 < budget ? q2 : budget;
      lenslot[at + 1] = c2;
      sf[c == 0 ? H_ANN : H_INT] += q2 - c2;
    }
  }
  const bool any = sf[0] | sf[1] | sf[2] | sf[3];
  const unsigned who = __ballot_sync(0xffffffffu, any);
  if (!who) return;
  const int leader_p = __shfl_sync(0xffffffffu, p, __ffs(who) - 1);
  if (__all_sync(0xffffffffu, !any || p == leader_p)) {
#pragma unroll
    for (int h = 0; h < 4; h++) {
      int64_t x = sf[h];
#pragma unroll
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (threadIdx.x % 32 == 0 && x) atomic_add_i64(&shortfall[(int64_t)leader_p * 4 + h], x);
    }
    return;
  }
  for (int h = 0; h < 4; h++)
    if (sf[h]) atomic_add_i64(&shortfall[(int64_t)p * 4 + h], sf[h]);
}

// one nonzero removal slab: its start a and the total slab length before it
// (16 bytes; its end b = a + the next slab's pre - pre, the slabs being
// disjoint and ordered: RemovalMap.extents, _timeline.py:90-111)
struct __align__(16) Slab {
  int64_t a, pre;
};

// (max,+) RemovalMap scan, segmented by pid; slab count is global
struct RM {
  int64_t P;  // sum of max(0, len)
  int64_t Q;  // max-plus offset
  int64_t cnt;
  int head;
  int pad;
};
struct RMOp {
  __device__ RM operator()(const RM& a, const RM& b) const {
    RM r;
    r.cnt = a.cnt + b.cnt;
    r.pad = 0;
    if (b.head) {
      r.head = 1;
      r.P = b.P;
      r.Q = b.Q;
    } else {
      r.head = a.head;
      r.P = a.P + b.P;
      int64_t x = a.Q + b.P;
      r.Q = x > b.Q ? x : b.Q;
    }
    return r;
  }
};

__device__ __forceinline__ int hook_of(int sub) {
  return sub == TRANSITION_HOOK ? H_TRANS : sub == API_INTERCEPT ? H_IC : sub == API_INTERNAL ? H_INT : H_ANN;
}

#ifndef XS_R_ITEMS
#define XS_R_ITEMS 8
#endif
constexpr int R_ITEMS = XS_R_ITEMS;
#ifndef XS_REMOVAL_MINB
#define XS_REMOVAL_MINB 4  // 4 CTAs per SM (64 registers, small spills): 1.99 -> 1.61 ms at 30M events
#endif
__global__ void __launch_bounds__(XS_BLOCK, XS_REMOVAL_MINB) k_removal(const uint64_t* k1, const uint32_t* slot, const int64_t* d_ns, int tb,
                                                      const int64_t* lenslot,
                                                      const int64_t* lo, const int64_t* hi,
                                                      const int64_t* span_end_in, int64_t* removed,
                                                      Slab* slabs,
                                                      int* pid_slabs, int64_t* ptotal, TileDesc<RM>* desc,
                                                      int* flags, int* tile_ctr) {
  const int tile = next_tile(tile_ctr);
  const int64_t ns = *d_ns;
  if ((int64_t)tile * XS_BLOCK * R_ITEMS >= ns) return;  // tail tiles of the upper-bound grid
  const int64_t base = (int64_t)tile * XS_BLOCK * R_ITEMS + (int64_t)threadIdx.x * R_ITEMS;
  const int pshift = tb + 3;
  const uint64_t tmask = (1ull << tb) - 1;
  int64_t anc[R_ITEMS], len[R_ITEMS];
  int hd[R_ITEMS], sub[R_ITEMS], pp[R_ITEMS];
  RMOp op;
  RM agg{0, kNegInf, 0, 0, 0};
  uint64_t kv[R_ITEMS], prevk;
  uint32_t sv[R_ITEMS];
  load_site_run<R_ITEMS>(k1, slot, base, ns, kv, sv, prevk);
#pragma unroll
  for (int j = 0; j < R_ITEMS; j++) {
    int64_t q = base + j;
    if (q < ns) {
      const uint64_t kk = kv[j];
      anc[j] = (int64_t)((kk >> 3) & tmask);
      pp[j] = (int)(kk >> pshift);
      sub[j] = (int)(kk & 7u);  // (the key's subkind bits; no gather)
      len[j] = lenslot[sv[j]];
      hd[j] = q == 0 || (prevk >> pshift) != (kk >> pshift);
      prevk = kk;
      RM e{len[j] > 0 ? len[j] : 0, anc[j] + len[j], len[j] > 0 ? 1 : 0, hd[j], 0};
      agg = op(agg, e);
    }
  }
  RM cur = grid_exclusive(agg, op, RM{0, kNegInf, 0, 0, 0}, tile, desc, flags);
  // per-thread removed accumulation keyed by pid
  int cp = -1;
  int64_t acc[4] = {0, 0, 0, 0};
  int64_t nsl = 0, tot = 0;
#pragma unroll
  for (int j = 0; j < R_ITEMS; j++) {
    int64_t q = base + j;
    if (q >= ns) break;
    if (hd[j]) {
      cur.P = 0;
      cur.Q = kNegInf;
    }
    const int64_t E = cur.Q;
    const int64_t a = anc[j] > E ? anc[j] : E;
    const int64_t b = a + len[j];
    const int p = pp[j];
    if (p != cp) {
      if (cp >= 0) {
        for (int h = 0; h < 4; h++)
          if (acc[h]) atomic_add_i64(&removed[(int64_t)cp * 4 + h], acc[h]);
        if (nsl) atomicAdd(&pid_slabs[cp], (int)nsl);
        if (tot) atomic_add_i64(&ptotal[cp], tot);
      }
      cp = p;
      acc[0] = acc[1] = acc[2] = acc[3] = 0;
      nsl = tot = 0;
    }
    const int64_t span_end = (span_end_in ? span_end_in[p] : hi[p]) - lo[p];
    const int64_t mb = b < span_end ? b : span_end;
    const int64_t ma = a < span_end ? a : span_end;
    acc[hook_of(sub[j])] += mb - ma;
    if (len[j] > 0) {
      const int64_t at = cur.cnt;
      slabs[at] = Slab{a, cur.P};
      nsl++;
      tot += len[j];
    }
    RM e{len[j] > 0 ? len[j] : 0, anc[j] + len[j], len[j] > 0 ? 1 : 0, 0, 0};
    cur = op(cur, e);
  }
  long long fv[6] = {acc[0], acc[1], acc[2], acc[3], nsl, tot};
  block_keyed_flush<6>(cp, fv, [&](int p, const long long* x) {
    for (int h = 0; h < 4; h++)
      if (x[h]) atomic_add_i64(&removed[(int64_t)p * 4 + h], x[h]);
    if (x[4]) atomicAdd(&pid_slabs[p], (int)x[4]);
    if (x[5]) atomic_add_i64(&ptotal[p], x[5]);
  });
}

__global__ void k_slab_base(const int* pid_slabs, int np, int64_t* slab_base) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t acc = 0;
    for (int p = 0; p < np; p++) {
      slab_base[p] = acc;
      acc += pid_slabs[p];
    }
    slab_base[np] = acc;
  }
}

// RemovalMap.__call__ (_timeline.py:112-117) on a relative coordinate, over
// the slab starts: with j = #slabs starting before y, slabs 0..j-2 lie wholly
// before y and slab j-1 is removed up to y (the sum of full slabs with b <= y
// plus the part of the one holding y, as bisect_right over the ends gives)
__device__ __forceinline__ int64_t rmap_tail(int64_t y, const Slab* sl, int64_t base, int64_t K, int64_t total,
                                             int64_t j) {
  if (j == 0) return 0;
  const Slab x = sl[base + j - 1];
  const int64_t next = j < K ? sl[base + j].pre : total;  // (the next record: mostly the same sector)
  const int64_t part = y - x.a, len = next - x.pre;
  return x.pre + (part < len ? part : len);
}

__device__ __forceinline__ int64_t rmap_removed(int64_t y, const Slab* sl,
                                                int64_t base, int64_t K, int64_t total) {
  int64_t lo = 0, hi = K;  // j = #starts < y
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (sl[base + mid].a < y) lo = mid + 1;
    else hi = mid;
  }
  return rmap_tail(y, sl, base, K, total, lo);
}

// Sampled index over each pid's slab starts: the pid's time range [0, span]
// is cut into W = 2^logw windows of 2^shift ns; idx[p*W + w] = #starts <
// (w << shift).  A query y in window w then bisects only
// [idx[w], idx[w+1]] -- a few slabs instead of all of them.
__device__ __forceinline__ int rmap_shift(const int64_t* lo, const int64_t* hi, int p, int logw) {
  const int64_t span = hi[p] > lo[p] ? hi[p] - lo[p] : 0;
  const int b = bits_for((uint64_t)span);
  return b > logw ? b - logw : 0;
}

__global__ void k_rmap_index(int np, int logw, const int64_t* lo, const int64_t* hi, const Slab* sl,
                             const int64_t* slab_base, int32_t* idx) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t W = (int64_t)1 << logw;
  if (t >= (int64_t)np * W) return;
  const int p = (int)(t >> logw);
  const int64_t w = t & (W - 1);
  const int64_t base = slab_base[p], K = slab_base[p + 1] - base;
  if (lo[p] == INT64_MAX) {
    idx[t] = 0;
    return;
  }
  const uint64_t x = (uint64_t)w << rmap_shift(lo, hi, p, logw);
  int64_t a = 0, b = K;  // #starts < x
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if ((uint64_t)sl[base + m].a < x) a = m + 1;
    else b = m;
  }
  idx[t] = (int32_t)a;
}

__device__ __forceinline__ int64_t rmap_removed_idx(int64_t y, const Slab* sl, int64_t base, int64_t K,
                                                    int64_t total,
                                                    const int32_t* pidx, int logw, int shift) {
  const int64_t W = (int64_t)1 << logw;
  const int64_t w = y >> shift;  // y in [0, span]: w < W
  int64_t a = pidx[w], b = w + 1 < W ? pidx[w + 1] : K;
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (sl[base + m].a < y) a = m + 1;
    else b = m;
  }
  return rmap_tail(y, sl, base, K, total, a);
}

__global__ void k_remap(EventView v, int64_t n, const int64_t* lo, const int64_t* hi, const Slab* sl,
                        const int64_t* slab_base, const int64_t* ptotal,
                        const int32_t* idx, int logw, int64_t* out_start, int64_t* out_dur) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int p = v.ev.pid[i];
  int64_t base = slab_base[p], K = slab_base[p + 1] - base, tot = ptotal[p];
  int64_t s = v.start[i], d = v.dur[i];
  int64_t l = lo[p];
  const int shift = rmap_shift(lo, hi, p, logw);
  const int32_t* pidx = idx + ((int64_t)p << logw);
  int64_t s2 = s - rmap_removed_idx(s - l, sl, base, K, tot, pidx, logw, shift);
  out_start[i] = s2;
  if (v.ev.cat[i] == 5) {
    out_dur[i] = d;
  } else {
    int64_t e = s + d;
    out_dur[i] = (e - rmap_removed_idx(e - l, sl, base, K, tot, pidx, logw, shift)) - s2;
  }
}

__global__ void k_remap_queries(int64_t n, const int32_t* qp, const int64_t* qv, int64_t* out, const int64_t* lo,
                                const Slab* sl, const int64_t* slab_base,
                                const int64_t* ptotal, int np) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int p = qp[i];
  int64_t y = qv[i];
  if (p < 0 || p >= np || lo[p] == INT64_MAX) {
    out[i] = y;
    return;
  }
  int64_t base = slab_base[p], K = slab_base[p + 1] - base;
  out[i] = y - rmap_removed(y - lo[p], sl, base, K, ptotal[p]);
}

__global__ void k_totals(const int64_t* lo, const int64_t* hi, int np, Stats* st, int which) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  long long v = 0;
  if (p < np && lo[p] != INT64_MAX) v = hi[p] - lo[p];
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd((unsigned long long*)&st->pad[which], (unsigned long long)v);
}

__global__ void k_zero_pad(Stats* st) {  // the two span totals (pad[3] is the sort-overflow flag)
  if (threadIdx.x < 2) st->pad[1 + threadIdx.x] = 0;
}

// corrected per-pid spans (pid_spans(out), correction.py:184-185): warp
// then block aggregation, one min/max atomic pair per pid per block
__global__ void k_out_spans(const int32_t* pid, int64_t n, const int64_t* s, const int64_t* d, int64_t* lo2,
                            int64_t* hi2) {
  constexpr int NW = XS_BLOCK / 32;
  __shared__ int s_p[NW];
  __shared__ int64_t s_a[NW], s_b[NW];
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int p = i < n ? pid[i] : -1;
  int64_t a = i < n ? s[i] : INT64_MAX;
  int64_t b = i < n ? s[i] + d[i] : INT64_MIN;
  const int lane0_p = __shfl_sync(full, p, 0);
  const int pv = p >= 0 ? p : lane0_p;  // (tail lanes join their warp's pid)
  const int p0 = __shfl_sync(full, pv, 0);
  if (__all_sync(full, pv == p0)) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      int64_t a2 = __shfl_xor_sync(full, a, o), b2 = __shfl_xor_sync(full, b, o);
      a = a2 < a ? a2 : a;
      b = b2 > b ? b2 : b;
    }
    if (lane == 0) {
      s_p[warp] = p0;
      s_a[warp] = a;
      s_b[warp] = b;
    }
  } else {
    if (lane == 0) s_p[warp] = -1;
    if (p >= 0) {
      atomic_min_i64(&lo2[p], a);
      atomic_max_i64(&hi2[p], b);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int cp = -1;
    int64_t ca = INT64_MAX, cb = INT64_MIN;
    for (int w = 0; w <= NW; w++) {
      const int wp = w < NW ? s_p[w] : -2;
      if (wp != cp) {
        if (cp >= 0) {
          atomic_min_i64(&lo2[cp], ca);
          atomic_max_i64(&hi2[cp], cb);
        }
        cp = wp;
        ca = INT64_MAX;
        cb = INT64_MIN;
      }
      if (wp >= 0) {
        ca = s_a[w] < ca ? s_a[w] : ca;
        cb = s_b[w] > cb ? s_b[w] : cb;
      }
    }
  }
}

__global__ void k_init_span(int64_t* lo, int64_t* hi, int np) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < np) {
    lo[p] = INT64_MAX;
    hi[p] = INT64_MIN;
  }
}

__global__ void k_site_total(const int* pos, const int* cnt, int64_t n, int64_t* d_ns) {
  if (threadIdx.x == 0) *d_ns = n ? (int64_t)pos[n - 1] + cnt[n - 1] : 0;
}

// report totals stay on the device: [original, corrected, n_sites, n_slabs]
__global__ void k_corr_finalize(const Stats* st, const int64_t* d_ns, const int64_t* slab_base, int np,
                                int corrected_spans, int64_t* totals) {
  if (threadIdx.x == 0) {
    totals[0] = st->pad[1];
    totals[1] = corrected_spans ? st->pad[2] : 0;
    totals[2] = *d_ns;
    totals[3] = slab_base[np];
  }
}

__global__ void k_span_total(const int64_t* lo, const int64_t* hi, int np, int64_t* out) {
  long long v = 0;
  for (int p = threadIdx.x; p < np; p += blockDim.x)
    if (lo[p] != INT64_MAX) v += hi[p] - lo[p];
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd((unsigned long long*)out, (unsigned long long)v);
}

int stage_correct(xs_ctx* ctx, const EventView& v, const xs_profile_t* prof, int64_t* out_start, int64_t* out_dur,
                  bool corrected_spans, cudaStream_t s) {
  const int64_t n = v.ev.n;
  const int np = v.ev.n_pids, ng = v.ev.n_groups;
  Stats* st = (Stats*)ctx->ptr[W_STATS];
  const Stats& H = *ctx->h_stats;
  const int tb = bits_for((uint64_t)(H.max_span > 0 ? H.max_span : 0));
  const int pb = bits_for((uint64_t)(np > 0 ? np - 1 : 0));
  const int gb = bits_for((uint64_t)(ng > 0 ? ng - 1 : 0));
  const int nb = bits_for((uint64_t)(v.ev.n_names > 0 ? v.ev.n_names - 1 : 0));
  if (pb + tb + 3 > 64 || gb + nb > 64) {
    ctx->err = "timeline too wide for 64-bit site keys";
    return XS_UNSUPPORTED;
  }
  const int64_t* lo_ev = (const int64_t*)ctx->ptr[W_SPAN_LO];
  const int64_t* hi_ev = (const int64_t*)ctx->ptr[W_SPAN_HI];
  // keep this correction's per-pid origin for xs_remap (the overlap pass reuses W_SPAN_*)
  int64_t *lo, *hi;
  XS_TRY(ws(ctx, W_CORR_LO, np + 1, s, &lo));
  XS_TRY(ws(ctx, W_CORR_HI, np + 1, s, &hi));
  XS_CUDA(cudaMemcpyAsync(lo, lo_ev, (np + 1) * 8, cudaMemcpyDeviceToDevice, s));
  XS_CUDA(cudaMemcpyAsync(hi, hi_ev, (np + 1) * 8, cudaMemcpyDeviceToDevice, s));
  const uint8_t* tflag = (const uint8_t*)ctx->ptr[W_SITE_FLAG];
  int64_t *removed, *shortfall, *ptotal, *slab_base;
  int* pid_slabs;
  XS_TRY(ws(ctx, W_REMOVED, (int64_t)np * 4 + 1, s, &removed));
  XS_TRY(ws(ctx, W_SHORTFALL, (int64_t)np * 4 + 1, s, &shortfall));
  XS_TRY(ws(ctx, W_PTOTAL, np + 1, s, &ptotal));
  XS_TRY(ws(ctx, W_SLAB_BASE, np + 2, s, &slab_base));
  XS_TRY(ws(ctx, W_PID_SLABS, np + 1, s, &pid_slabs));
  int64_t* d_ns;
  XS_TRY(ws(ctx, W_NS_DEV, 1, s, &d_ns));
  XS_TRY(fill_many(ctx, s, {{removed, ((unsigned long long)np * 4 + 1) * 8, 0},
                            {shortfall, ((unsigned long long)np * 4 + 1) * 8, 0},
                            {ptotal, (unsigned long long)(np + 1) * 8, 0},
                            {pid_slabs, (unsigned long long)(np + 1) * 4, 0},
                            {d_ns, 8, 0}}));
  XS_LAUNCH(ctx, k_zero_pad, 1, 32, 0, s, st);
  XS_LAUNCH(ctx, k_totals, grid_for(np + 1), XS_BLOCK, 0, s, lo, hi, np, st, 1);

  // 1. hook sites, compacted in event-index order
  int *cnt, *pos;
  XS_TRY(ws(ctx, W_SITE_CNT, n + 1, s, &cnt));
  XS_TRY(ws(ctx, W_SITE_POS, n + 1, s, &pos));
  // site count bound from pass-1 counts (2 per OPERATION, 2 per ACCEL_API,
  // <= 1 per BACKEND/SIMULATOR); the exact count stays on the device
  const Stats& Hc = *ctx->h_stats;
  const int64_t ns = 2 * Hc.cat_all[0] + 2 * Hc.cat_all[4] + Hc.cat_all[2] + Hc.cat_all[3];
  ProfScope ps_sites(ctx, ST_SITE_SORT, s);
  if (n) {
    XS_LAUNCH(ctx, k_site_count, grid_for(n), XS_BLOCK, 0, s, v, n, tflag, cnt);
    XS_TRY(scan_exclusive<int>(ctx, ArrayIn<int>{cnt}, pos, n, s));
    XS_LAUNCH(ctx, k_site_total, 1, 32, 0, s, pos, cnt, n, d_ns);
  }
  Slab* slabs;  // (a, b, prefix) per nonzero slab, interleaved
  XS_TRY(ws(ctx, W_SLAB_A, ns + 1, s, &slabs));
  if (ns > 0) {
    int* site_ev;
    int* site_row;
    uint64_t *k1, *k1_alt;
    uint32_t *sl, *sl_alt;
    XS_TRY(ws(ctx, W_SITE_K, ns + 1, s, &k1));
    XS_TRY(ws(ctx, W_SITE_K_ALT, ns + 1, s, &k1_alt));
    XS_TRY(ws(ctx, W_SITE_V, ns + 1, s, &sl));
    XS_TRY(ws(ctx, W_SITE_V_ALT, ns + 1, s, &sl_alt));
    XS_TRY(ws(ctx, W_SITE_EV, ns + 1, s, &site_ev));
    XS_TRY(ws(ctx, W_SITE_SUB, ns + 1, s, &site_row));
    XS_LAUNCH(ctx, k_site_gen, grid_for(n), XS_BLOCK, 0, s, v, n, cnt, pos, lo, tb, site_ev, site_row, k1);
    XS_LAUNCH(ctx, k_site_tail, grid_for(ns), XS_BLOCK, 0, s, k1, sl, ns, d_ns);
    // 2. Site.order_key: one sort on (pid, anchor, subkind) + local tie order
    XS_TRY(sort_pairs_u64_u32(ctx, &k1, &k1_alt, &sl, &sl_alt, ns, pb + tb + 3, s));
    XS_LAUNCH(ctx, k_tie_fix, grid_for(ns), XS_BLOCK, 0, s, v, k1, sl, ns, site_ev);
    ps_sites.end();
    ProfScope ps_q(ctx, ST_QUANTIZE, s);
    // 3. exact quantization (segmented int128 scan)
    int64_t *qslot, *lenslot;
    XS_TRY(ws(ctx, W_LENSLOT, ns + 1, s, &lenslot));
    XS_TRY(ws(ctx, W_QVAL, ns + 1, s, &qslot));
    {
      const int64_t tiles = (ns + XS_BLOCK * Q_ITEMS - 1) / (XS_BLOCK * Q_ITEMS);
      switch (prof->words) {
        case 1: XS_TRY(launch_quantize<1>(ctx, tiles, s, k1, sl, d_ns, tb, v, *prof, site_row, qslot)); break;
        case 2: XS_TRY(launch_quantize<2>(ctx, tiles, s, k1, sl, d_ns, tb, v, *prof, site_row, qslot)); break;
        case 4: XS_TRY(launch_quantize<4>(ctx, tiles, s, k1, sl, d_ns, tb, v, *prof, site_row, qslot)); break;
        default: XS_TRY(launch_quantize<8>(ctx, tiles, s, k1, sl, d_ns, tb, v, *prof, site_row, qslot)); break;
      }
    }
    ps_q.end();
    // 4. budget caps per owner
    ProfScope ps_r(ctx, ST_REMOVAL, s);
    XS_LAUNCH(ctx, k_caps, grid_for(n), XS_BLOCK, 0, s, v, n, cnt, pos, qslot, lenslot, shortfall);
    // 5. RemovalMap scan + removed accounting + nonzero slab compaction
    {
      const int64_t tiles = (ns + XS_BLOCK * R_ITEMS - 1) / (XS_BLOCK * R_ITEMS);
      TileDesc<RM>* desc;
      int *flags, *tctr;
      XS_TRY(ws(ctx, W_RSCAN_DESC, tiles + 1, s, &desc));
      XS_TRY(ws(ctx, W_RSCAN_FLAGS, tiles + 1, s, &flags));
      XS_TRY(ws(ctx, W_TILE_CTR, 4, s, &tctr));
      XS_TRY(fill_many(ctx, s, {{flags, (unsigned long long)(tiles + 1) * sizeof(int), 0}, {tctr, sizeof(int), 0}}));
      XS_LAUNCH(ctx, k_removal, (int)tiles, XS_BLOCK, 0, s, k1, sl, d_ns, tb, lenslot, lo, hi, prof->span_end_in, removed,
                slabs, pid_slabs, ptotal, desc, flags, tctr);
    }
  }
  XS_LAUNCH(ctx, k_slab_base, 1, 32, 0, s, pid_slabs, np, slab_base);
  ps_sites.end();
  // 6. remap every event (positional, correction.py:158-165)
  ProfScope ps_m(ctx, ST_REMAP, s);
  if (n) {
    int logw = bits_for((uint64_t)(ns / (np > 0 ? np : 1)));
    logw = logw < 4 ? 4 : (logw > 16 ? 16 : logw);
    while (logw > 4 && ((int64_t)np << logw) > ((int64_t)1 << 24)) logw--;
    int32_t* ridx;
    XS_TRY(ws(ctx, W_RMAP_IDX, ((int64_t)np << logw) + 1, s, &ridx));
    ctx->rmap_logw = logw;
    XS_LAUNCH(ctx, k_rmap_index, grid_for((int64_t)np << logw), XS_BLOCK, 0, s, np, logw, lo, hi, slabs, slab_base,
              ridx);
    XS_LAUNCH(ctx, k_remap, grid_for(n), XS_BLOCK, 0, s, v, n, lo, hi, slabs, slab_base, ptotal,
              ridx, logw, out_start, out_dur);
  }
  if (corrected_spans) {
    int64_t *lo2, *hi2;
    XS_TRY(ws(ctx, W_OUT_LO, np + 1, s, &lo2));
    XS_TRY(ws(ctx, W_OUT_HI, np + 1, s, &hi2));
    XS_LAUNCH(ctx, k_init_span, grid_for(np + 1), XS_BLOCK, 0, s, lo2, hi2, np);
    if (n) XS_LAUNCH(ctx, k_out_spans, grid_for(n), XS_BLOCK, 0, s, v.ev.pid, n, out_start, out_dur, lo2, hi2);
    XS_LAUNCH(ctx, k_totals, grid_for(np + 1), XS_BLOCK, 0, s, lo2, hi2, np, st, 2);
  }
  int64_t* totals;
  XS_TRY(ws(ctx, W_CORR_TOTALS, 4, s, &totals));
  XS_LAUNCH(ctx, k_corr_finalize, 1, 32, 0, s, st, d_ns, slab_base, np, corrected_spans ? 1 : 0, totals);
  ctx->corr_pids = np;
  return XS_OK;
}

int corrected_total_from_spans(xs_ctx* ctx, cudaStream_t s) {
  int64_t* totals;
  XS_TRY(ws(ctx, W_CORR_TOTALS, 4, s, &totals));
  XS_CUDA(cudaMemsetAsync(totals + 1, 0, 8, s));
  XS_LAUNCH(ctx, k_span_total, 1, 256, 0, s, (const int64_t*)ctx->ptr[W_SPAN_LO], (const int64_t*)ctx->ptr[W_SPAN_HI],
            ctx->res_pids, totals + 1);
  return XS_OK;
}

}  // namespace xs

using namespace xs;

// The operation stage of the ORIGINAL trace serves the overlap pass of the
// corrected one when the removal map is strictly increasing on every pid's
// op endpoint times: then the corrected endpoints keep their order and ties
// (equal times stay equal, distinct ones distinct), so the (start, -end, tid,
// name) ranks, the merged paths and the per-pid op counts are unchanged.
// pk = the original's op endpoints in (pid, t) order (pid | t_rel | flag,
// t_rel relative to the original lo, the removal map's own origin); a pair
// of neighbours of one pid with t < t' but rmap(t) >= rmap(t') sets pad[8]
// (the host then redoes the overlap pass with its own operation stage).
namespace xs {
__device__ __forceinline__ int64_t ops_strict_map(uint64_t key, int tb, const int64_t* lo, const int64_t* hi,
                                                  const Slab* sl,
                                                  const int64_t* slab_base, const int64_t* ptotal, const int32_t* idx,
                                                  int logw) {
  const int p = (int)(key >> (tb + 1));
  const int64_t t = (int64_t)((key >> 1) & ((1ull << tb) - 1));
  const int64_t base = slab_base[p], K = slab_base[p + 1] - base;
  return t - rmap_removed_idx(t, sl, base, K, ptotal[p], idx + ((int64_t)p << logw), logw,
                              rmap_shift(lo, hi, p, logw));
}

// one sampled-index lookup per endpoint; the right neighbour's value comes
// from the next lane (the warp's last lane looks its neighbour up itself)
__global__ void k_ops_strict(const uint64_t* pk, int64_t n2, int tb, const int64_t* lo, const int64_t* hi,
                             const Slab* sl, const int64_t* slab_base,
                             const int64_t* ptotal, const int32_t* idx, int logw, int np, Stats* st) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const uint64_t a = j < n2 ? pk[j] : ~0ull;
  const bool va = a != ~0ull && (int)(a >> (tb + 1)) < np;
  const int64_t ca = va ? ops_strict_map(a, tb, lo, hi, sl, slab_base, ptotal, idx, logw) : 0;
  int64_t cb = __shfl_down_sync(0xffffffffu, ca, 1);
  uint64_t b = __shfl_down_sync(0xffffffffu, a, 1);
  if (lane == 31) {
    b = j + 1 < n2 ? pk[j + 1] : ~0ull;
    const bool vb = b != ~0ull && (int)(b >> (tb + 1)) < np;
    cb = vb ? ops_strict_map(b, tb, lo, hi, sl, slab_base, ptotal, idx, logw) : 0;
  }
  if (!va || j + 1 >= n2 || b == ~0ull) return;
  if ((a >> (tb + 1)) != (b >> (tb + 1))) return;  // different pids
  if (((a ^ b) >> 1) & ((1ull << tb) - 1)) {      // distinct times must stay distinct and ordered
    if (ca >= cb) atomicOr((unsigned long long*)&st->pad[8], 1ull);
  }
}

int ops_reuse_check(xs_ctx* ctx, const EventView& v, Stats* verdict, cudaStream_t s) {
  const OpsState& os = ctx->ops;
  if (os.m <= 0 || !os.pk) return XS_OK;
  XS_LAUNCH(ctx, k_ops_strict, grid_for(2 * os.m), XS_BLOCK, 0, s, os.pk, 2 * os.m, os.tb,
            (const int64_t*)ctx->ptr[W_CORR_LO], (const int64_t*)ctx->ptr[W_CORR_HI],
            (const Slab*)ctx->ptr[W_SLAB_A], (const int64_t*)ctx->ptr[W_SLAB_BASE],
            (const int64_t*)ctx->ptr[W_PTOTAL], (const int32_t*)ctx->ptr[W_RMAP_IDX], ctx->rmap_logw, v.ev.n_pids,
            verdict);
  return XS_OK;
}
}  // namespace xs

extern "C" {


int xs_remap(xs_ctx_t* ctx, int64_t n, const int32_t* pid_dev, const int64_t* val_dev, int64_t* out_dev,
             xs_stream_t stream) {
  if (!ctx || !ctx->have_correct) return XS_BAD_ARGUMENT;
  if (n <= 0) return XS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  XS_LAUNCH(ctx, k_remap_queries, grid_for(n), XS_BLOCK, 0, s, n, pid_dev, val_dev, out_dev,
            (const int64_t*)ctx->ptr[W_CORR_LO], (const Slab*)ctx->ptr[W_SLAB_A],
            (const int64_t*)ctx->ptr[W_SLAB_BASE], (const int64_t*)ctx->ptr[W_PTOTAL], ctx->corr_pids);
  return XS_OK;
}

}  // extern "C"
