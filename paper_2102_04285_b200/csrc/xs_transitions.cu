// xs_transitions.cu -- transition_sites (overlap.py:220-289) on the device.
//
// A dst-category event is a site of pair (src, dst) iff, on its own
// (pid, tid):
//   * it is maximal among same-category events (_maximal_events): no event
//     with an earlier start and end >= its end, and no same-start event with a
//     strictly larger end (equal intervals both count);
//   * its start lies inside the union of nonzero src events (_covered): the
//     count of src events with start <= t < end is > 0.
// One sorted record stream per call: key = group | t_rel | kind with kinds
//   0..2 src close (H,B,S), 3..5 src open, 6..8 query (B,S,A)
// so at one instant closes precede opens precede queries; queries that tie
// on the key are put in descending-end order by a local pass, so inside a
// same-start block the head has the largest end.  One decoupled-lookback scan carries the three
// coverage counts and, per query category, a group-segmented running max of
// ends; an event is contained iff the exclusive max at the head of its run of
// identical (start, end) is >= its end.
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "xs_engine.cuh"
#include "xs_prims.cuh"

namespace xs {

struct TState {
  int cov[3];       // H, B, S coverage counts
  int head;         // segment (group) head seen
  int64_t mx[3];    // running max end for query categories B, S, A (segmented)
  int64_t hp;       // last run-head position (plain max)
};

struct TOp {
  __device__ TState operator()(const TState& a, const TState& b) const {
    TState r;
#pragma unroll
    for (int c = 0; c < 3; c++) r.cov[c] = a.cov[c] + b.cov[c];
    r.head = a.head | b.head;
#pragma unroll
    for (int c = 0; c < 3; c++) r.mx[c] = b.head ? b.mx[c] : (a.mx[c] > b.mx[c] ? a.mx[c] : b.mx[c]);
    r.hp = a.hp > b.hp ? a.hp : b.hp;
    return r;
  }
};

__device__ __forceinline__ TState t_identity() {
  TState r;
  r.cov[0] = r.cov[1] = r.cov[2] = 0;
  r.head = 0;
  r.mx[0] = r.mx[1] = r.mx[2] = INT64_MIN;
  r.hp = -1;
  return r;
}

// records: src endpoints (nonzero src events) + queries (all dst events)
__global__ void k_trec(EventView v, int64_t n, const int64_t* lo, int tb, int src_mask, int dst_mask, const int* tg,
                       uint64_t* key, uint32_t* val, unsigned long long* count) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int c = i < n ? v.ev.cat[i] : 0;
  bool is_src = i < n && c >= 1 && c <= 3 && ((src_mask >> c) & 1) && v.dur[i] > 0;
  bool is_dst = i < n && c >= 2 && c <= 4 && ((dst_mask >> c) & 1);
  int k = (is_src ? 2 : 0) + (is_dst ? 1 : 0);
  unsigned long long at = block_reserve(count, (unsigned)k);  // whole block participates
  if (!k) return;
  int p = v.ev.pid[i];
  uint64_t g = (uint64_t)tg[v.ev.tid[i]];  // dense over the groups carrying such events (order kept)
  uint64_t s = (uint64_t)(v.start[i] - lo[p]);
  uint64_t e = s + (uint64_t)v.dur[i];
  if (is_src) {
    key[at] = (g << (tb + 4)) | (e << 4) | (uint64_t)(c - 1);
    val[at] = (uint32_t)i;
    key[at + 1] = (g << (tb + 4)) | (s << 4) | (uint64_t)(c - 1 + 3);
    val[at + 1] = (uint32_t)i;
    at += 2;
  }
  if (is_dst) {
    key[at] = (g << (tb + 4)) | (s << 4) | (uint64_t)(c - 2 + 6);
    val[at] = (uint32_t)i;
  }
}

// queries with equal (group, start, category): descending end (ties in end
// are identical intervals, whose order does not matter)
__global__ void k_trec_tiefix(const uint64_t* key, uint32_t* val, int64_t m, EventView v) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  const uint64_t k = key[q];
  if ((k & 15u) < 6) return;
  if (q > 0 && key[q - 1] == k) return;
  if (q + 1 >= m || key[q + 1] != k) return;
  int64_t e = q + 1;
  while (e < m && key[e] == k) e++;
  for (int64_t a = q + 1; a < e; a++) {
    const uint32_t x = val[a];
    const int64_t ex = v.start[x] + v.dur[x];
    int64_t b = a - 1;
    while (b >= q) {
      const uint32_t y = val[b];
      if (v.start[y] + v.dur[y] >= ex) break;
      val[b + 1] = y;
      b--;
    }
    val[b + 1] = x;
  }
}

#ifndef XS_T_ITEMS
#define XS_T_ITEMS 4
#endif
constexpr int T_ITEMS = XS_T_ITEMS;
#ifndef XS_TSCAN_MINB
#define XS_TSCAN_MINB 3  // (0.61 -> 0.56 ms at 30M events)
#endif
__global__ void __launch_bounds__(XS_BLOCK, XS_TSCAN_MINB) k_tscan(const uint64_t* __restrict__ key, const uint32_t* __restrict__ val,
                                                    int64_t m, int tb, EventView v, uint8_t* flags_out,
                                                    int32_t* headpos_out, TileDesc<TState>* desc, int* flags,
                                                    int* tile_ctr, int src_mask) {
  const int tile = next_tile(tile_ctr);
  const int64_t base = (int64_t)tile * XS_BLOCK * T_ITEMS + (int64_t)threadIdx.x * T_ITEMS;
  uint64_t k[T_ITEMS];
  uint32_t ev[T_ITEMS];
  int64_t en[T_ITEMS];
  uint64_t kprev = (base > 0 && base - 1 < m) ? key[base - 1] : ~0ull;
  int64_t eprev = INT64_MIN;
  if (base > 0 && base - 1 < m) {
    uint32_t i0 = val[base - 1];
    eprev = v.start[i0] + v.dur[i0];
  }
  TState agg = t_identity();
  TOp op;
#pragma unroll
  for (int j = 0; j < T_ITEMS; j++) {
    int64_t q = base + j;
    k[j] = q < m ? key[q] : ~0ull;
    ev[j] = q < m ? val[q] : 0;
    en[j] = q < m ? v.start[ev[j]] + v.dur[ev[j]] : 0;
  }
#pragma unroll
  for (int j = 0; j < T_ITEMS; j++) {
    int64_t q = base + j;
    if (q >= m) break;
    uint64_t kp = j ? k[j - 1] : kprev;
    int64_t ep = j ? en[j - 1] : eprev;
    TState e = t_identity();
    uint32_t kind = (uint32_t)(k[j] & 15u);
    if (q == 0 || (kp >> (tb + 4)) != (k[j] >> (tb + 4))) e.head = 1;
    if (kind < 3) e.cov[kind] = -1;
    else if (kind < 6) e.cov[kind - 3] = 1;
    else {
      e.mx[kind - 6] = en[j];
      if (q == 0 || kp != k[j] || ep != en[j]) e.hp = q;
    }
    agg = op(agg, e);
  }
  TState cur = grid_exclusive(agg, op, t_identity(), tile, desc, flags);
#pragma unroll
  for (int j = 0; j < T_ITEMS; j++) {
    int64_t q = base + j;
    if (q >= m) break;
    uint64_t kp = j ? k[j - 1] : kprev;
    int64_t ep = j ? en[j - 1] : eprev;
    uint32_t kind = (uint32_t)(k[j] & 15u);
    bool ghead = q == 0 || (kp >> (tb + 4)) != (k[j] >> (tb + 4));
    TState e = t_identity();
    if (ghead) e.head = 1;
    if (kind < 3) e.cov[kind] = -1;
    else if (kind < 6) e.cov[kind - 3] = 1;
    if (kind >= 6) {
      const int qc = kind - 6;
      const bool run_head = q == 0 || kp != k[j] || ep != en[j];
      // exclusive max within the group (a new group resets to -inf)
      const int64_t excl = ghead ? INT64_MIN : cur.mx[qc];
      e.mx[qc] = en[j];
      if (run_head) e.hp = q;
      TState after = op(cur, e);
      if (run_head) {
        const bool contained = excl >= en[j];
        uint8_t f = 0;
        if (!contained) {
          // after includes every src endpoint at t <= start (closes/opens sort first)
          if (qc == 0 && ((src_mask >> 1) & 1) && after.cov[0] > 0) f |= 1;  // H->B
          if (qc == 1 && ((src_mask >> 1) & 1) && after.cov[0] > 0) f |= 2;  // H->S
          if (qc == 2 && ((src_mask >> 2) & 1) && after.cov[1] > 0) f |= 4;  // B->A
          if (qc == 2 && ((src_mask >> 3) & 1) && after.cov[2] > 0) f |= 8;  // S->A
        }
        flags_out[ev[j]] = f;
        headpos_out[q] = -1;
      } else {
        headpos_out[q] = (int32_t)after.hp;
      }
      cur = after;
    } else {
      cur = op(cur, e);
    }
  }
}

// duplicates of one (start, end) run copy the run head's verdict
__global__ void k_tdup(const uint32_t* val, const int32_t* headpos, const uint64_t* key, int64_t m, uint8_t* flags_out) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  if ((key[q] & 15u) < 6) return;
  int32_t h = headpos[q];
  if (h >= 0) flags_out[val[q]] = flags_out[val[h]];
}

struct FlagToInt {
  __device__ int operator()(const uint8_t& f) const { return f ? 1 : 0; }
};

int stage_transitions(xs_ctx* ctx, const EventView& v, int src_mask, int dst_mask, cudaStream_t s) {
  const int64_t n = v.ev.n;
  const int ng = v.ev.n_groups;
  const Stats& H = *ctx->h_stats;
  const int tb = bits_for((uint64_t)(H.max_span > 0 ? H.max_span : 0));
  const int gb = bits_for((uint64_t)(ng > 0 ? ng - 1 : 0));
  uint8_t* site_flag;
  XS_TRY(ws(ctx, W_SITE_FLAG, n + 1, s, &site_flag));
  XS_CUDA(cudaMemsetAsync(site_flag, 0, n + 1, s));
  if (n == 0) return XS_OK;
  if (gb + tb + 4 > 64 || tb + 1 > 64) {
    ctx->err = "timeline too wide for 64-bit transition keys";
    return XS_UNSUPPORTED;
  }
  // record count is known from pass-1 category counts: no device->host sync
  int64_t m = 0;
  for (int c = 1; c <= 3; c++)
    if ((src_mask >> c) & 1) m += 2 * H.cat_nz[c];
  for (int c = 2; c <= 4; c++)
    if ((dst_mask >> c) & 1) m += H.cat_all[c];
  if (m == 0) return XS_OK;
  uint64_t *key, *key_alt;
  uint32_t *val, *val_alt;
  unsigned long long* cnt;
  XS_TRY(ws(ctx, W_TQ_KEY, m + 1, s, &key));
  XS_TRY(ws(ctx, W_TQ_KEY_ALT, m + 1, s, &key_alt));
  XS_TRY(ws(ctx, W_TQ_VAL, m + 1, s, &val));
  XS_TRY(ws(ctx, W_TQ_VAL_ALT, m + 1, s, &val_alt));
  XS_TRY(ws(ctx, W_TSTAT, 4, s, &cnt));
  XS_CUDA(cudaMemsetAsync(cnt, 0, 8, s));
  const int64_t* lo = (const int64_t*)ctx->ptr[W_SPAN_LO];
  ProfScope ps_sort(ctx, ST_TRANS_SORT, s);
  // groups renumbered densely over those with HIGH_LEVEL..ACCEL_API events
  // (pass 1's flags): the key spends its bits on time, not on GPU streams
  int* tg;
  XS_TRY(ws(ctx, W_TGRP_IDX, ng + 1, s, &tg));
  {
    const uint8_t* tflag = (const uint8_t*)ctx->ptr[W_TGRP_FLAG];
    XS_TRY(scan_exclusive<int>(ctx, map_in(tflag, FlagToInt()), tg, ng, s));
  }
  const int tgb = bits_for((uint64_t)(H.pad[6] > 1 ? H.pad[6] - 1 : 0));
  XS_LAUNCH(ctx, k_trec, grid_for(n), XS_BLOCK, 0, s, v, n, lo, tb, src_mask, dst_mask, tg, key, val, cnt);
  // one sort on (group, t, kind); queries tying on it are put in descending
  // end order locally (the head of a same-start run has the largest end)
  XS_TRY(sort_pairs_u64_u32(ctx, &key, &key_alt, &val, &val_alt, m, tgb + tb + 4, s));
  XS_LAUNCH(ctx, k_trec_tiefix, grid_for(m), XS_BLOCK, 0, s, key, val, m, v);
  uint64_t* k1 = key;
  uint32_t* v1 = val;
  TileDesc<TState>* desc;
  int *tflags, *tctr;
  int32_t* headpos;
  const int64_t tiles = (m + XS_BLOCK * T_ITEMS - 1) / (XS_BLOCK * T_ITEMS);
  XS_TRY(ws(ctx, W_TSCAN_DESC, tiles + 1, s, &desc));
  XS_TRY(ws(ctx, W_TSCAN_FLAGS, tiles + 1, s, &tflags));
  XS_TRY(ws(ctx, W_TILE_CTR, 4, s, &tctr));
  XS_TRY(ws(ctx, W_HEADPOS, m + 1, s, &headpos));
  XS_TRY(fill_many(ctx, s, {{tflags, (unsigned long long)(tiles + 1) * sizeof(int), 0}, {tctr, sizeof(int), 0}}));
  ps_sort.end();
  ProfScope ps(ctx, ST_TRANS_SCAN, s);
  XS_LAUNCH(ctx, k_tscan, (int)tiles, XS_BLOCK, 0, s, k1, v1, m, tb, v, site_flag, headpos, desc, tflags, tctr,
            src_mask);
  XS_LAUNCH(ctx, k_tdup, grid_for(m), XS_BLOCK, 0, s, v1, headpos, k1, m, site_flag);
  return XS_OK;
}

}  // namespace xs

// ---------------------------------------------------------------------------
// transition_sites() public entry: (pair, event) list ordered per pair by
// Event.sort_key = (start, end, category, pid, tid, name, corr or -1), stable.
// ---------------------------------------------------------------------------
namespace xs {

__global__ void k_tr_count(const uint8_t* f, int64_t n, int pair_mask, int* cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cnt[i] = __popc((unsigned)(f[i] & pair_mask));
}

__global__ void k_tr_emit(const uint8_t* f, int64_t n, int pair_mask, const int* pos, int32_t* rpair, int64_t* rev) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned b = f[i] & pair_mask;
  int at = pos[i];
  for (int k = 0; k < 4; k++)
    if ((b >> k) & 1) {
      rpair[at] = k;
      rev[at] = i;
      at++;
    }
}

// mode 0: corr (sign-flipped), 1: group|name, 2: end, 3: start, 4: pair
__global__ void k_tr_key(EventView v, const int32_t* rpair, const int64_t* rev, const uint32_t* perm, int64_t m,
                         int mode, int nb, uint64_t* key) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  uint32_t r = perm[q];
  int64_t i = rev[r];
  uint64_t k;
  switch (mode) {
    case 0: k = (uint64_t)(v.ev.has_corr[i] ? v.ev.corr[i] : -1) ^ (1ull << 63); break;
    case 1: k = ((uint64_t)v.ev.tid[i] << nb) | (uint64_t)v.ev.name[i]; break;
    case 2: k = (uint64_t)(v.start[i] + v.dur[i]); break;
    case 3: k = (uint64_t)v.start[i]; break;
    default: k = (uint64_t)rpair[r]; break;
  }
  key[q] = k;
}

__global__ void k_tr_out(const int32_t* rpair, const int64_t* rev, const uint32_t* perm, int64_t m, int32_t* opair,
                         int64_t* oev) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  opair[q] = rpair[perm[q]];
  oev[q] = rev[perm[q]];
}

}  // namespace xs

using namespace xs;

extern "C" {

int xs_transition_sites(xs_ctx_t* ctx, const xs_events_t* ev, int pair_mask, int64_t* n_out, xs_stream_t stream) {
  if (!ctx || !ev || !n_out) return XS_BAD_ARGUMENT;
  if (ev->n < 0 || ev->n > ((int64_t)1 << 30)) return XS_BAD_ARGUMENT;
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  *n_out = 0;
  ctx->n_trans_out = 0;
  EventView v{*ev, ev->start, ev->dur};
  struct LsdScope {  // not a hot path: CUB radix sorts only, no overflow retries
    xs_ctx* c;
    bool prev;
    ~LsdScope() { c->force_lsd = prev; }
  } lsd{ctx, ctx->force_lsd};
  ctx->force_lsd = true;
  XS_TRY(stage_events(ctx, v, s, true, false, nullptr));
  XS_TRY(stage_ops(ctx, v, s, false));
  XS_TRY(fetch_stats(ctx, s));
  if (ctx->h_stats->n_bad) return XS_INVALID_TRACE;
  int src = 0, dst = 0;
  if (pair_mask & 1) src |= 2, dst |= 4;
  if (pair_mask & 2) src |= 2, dst |= 8;
  if (pair_mask & 4) src |= 4, dst |= 16;
  if (pair_mask & 8) src |= 8, dst |= 16;
  XS_TRY(stage_transitions(ctx, v, src, dst, s));
  const int64_t n = ev->n;
  if (n == 0) return XS_OK;
  const uint8_t* f = (const uint8_t*)ctx->ptr[W_SITE_FLAG];
  int *cnt, *pos;
  XS_TRY(ws(ctx, W_SITE_CNT, n + 1, s, &cnt));
  XS_TRY(ws(ctx, W_SITE_POS, n + 1, s, &pos));
  XS_LAUNCH(ctx, k_tr_count, grid_for(n), XS_BLOCK, 0, s, f, n, pair_mask, cnt);
  XS_TRY(scan_exclusive<int>(ctx, ArrayIn<int>{cnt}, pos, n, s));
  int lp = 0, lc = 0;
  XS_CUDA(cudaMemcpyAsync(&lp, pos + n - 1, 4, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaMemcpyAsync(&lc, cnt + n - 1, 4, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaStreamSynchronize(s));
  const int64_t m = (int64_t)lp + lc;
  int32_t *rpair, *opair;
  int64_t *rev, *oev;
  XS_TRY(ws(ctx, W_TREC_ID, m + 1, s, &rpair));
  XS_TRY(ws(ctx, W_SITE_K, m + 1, s, &rev));
  XS_TRY(ws(ctx, W_TRANS_OUT_PAIR, m + 1, s, &opair));
  XS_TRY(ws(ctx, W_TRANS_OUT_EV, m + 1, s, &oev));
  if (m > 0) {
    XS_LAUNCH(ctx, k_tr_emit, grid_for(n), XS_BLOCK, 0, s, f, n, pair_mask, pos, rpair, rev);
    uint64_t *k, *k_alt;
    uint32_t *pv, *pv_alt;
    XS_TRY(ws(ctx, W_TQ_KEY, m + 1, s, &k));
    XS_TRY(ws(ctx, W_TQ_KEY_ALT, m + 1, s, &k_alt));
    XS_TRY(ws(ctx, W_TQ_VAL, m + 1, s, &pv));
    XS_TRY(ws(ctx, W_TQ_VAL_ALT, m + 1, s, &pv_alt));
    XS_LAUNCH(ctx, k_iota_u32, grid_for(m), XS_BLOCK, 0, s, pv, m);
    const int ng = ev->n_groups;
    const int gb = bits_for((uint64_t)(ng > 0 ? ng - 1 : 0));
    const int nb = bits_for((uint64_t)(ev->n_names > 0 ? ev->n_names - 1 : 0));
    const int bits[5] = {64, gb + nb, 64, 64, 2};
    for (int mode = 0; mode < 5; mode++) {
      XS_LAUNCH(ctx, k_tr_key, grid_for(m), XS_BLOCK, 0, s, v, rpair, rev, pv, m, mode, nb, k);
      XS_TRY(sort_pairs_u64_u32(ctx, &k, &k_alt, &pv, &pv_alt, m, bits[mode], s));
    }
    XS_LAUNCH(ctx, k_tr_out, grid_for(m), XS_BLOCK, 0, s, rpair, rev, pv, m, opair, oev);
  }
  XS_CUDA(cudaStreamSynchronize(s));
  ctx->n_trans_out = m;
  *n_out = m;
  return XS_OK;
}

int xs_transition_fetch(xs_ctx_t* ctx, int32_t* pair, int64_t* event, xs_stream_t stream) {
  if (!ctx) return XS_BAD_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t m = ctx->n_trans_out;
  if (m == 0) return XS_OK;
  if (pair) XS_CUDA(cudaMemcpyAsync(pair, ctx->ptr[W_TRANS_OUT_PAIR], m * 4, cudaMemcpyDeviceToHost, s));
  if (event) XS_CUDA(cudaMemcpyAsync(event, ctx->ptr[W_TRANS_OUT_EV], m * 8, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaStreamSynchronize(s));
  return XS_OK;
}

}  // extern "C"
