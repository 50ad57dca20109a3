// xs_overlap.cu -- the boundary sweep (sweep_pid, _sweep.pyx:17-118) as a
// sort + single-pass scan + reduce-by-key.
//
// Endpoint key (64 bit):  pid | t_rel (tb bits) | code (4 bits)
//   code = cat (0..6) | close<<3.  cat 0 = OPERATION (op-count lane),
//   1..5 = resource categories, 6 = CORRELATION "tracked-only" lane.
// After the radix sort the state for [t_i, t_{i+1}) is the state after *all*
// endpoints at t_i (equivalent to the reference's remove-then-add walk), so
// only the last endpoint of each equal-(pid, t) run emits.  The per-category
// counts are a plain prefix sum over the whole sorted array: every pid opens
// and closes all of its events inside its own key range, so counts return to
// zero at pid boundaries and no segmentation is needed.  The path of the
// interval is pidpath[c-1] where c is the running count of OPERATION
// endpoints (xs_ops.cu).  Cells accumulate in a per-block shared-memory hash
// and are flushed into a dense int64 histogram [pid][path node][32 masks];
// mask 0 of path 0 holds the per-pid tracked time.
//
// CORRELATION (overlap.py:144-163, _sweep.pyx:70-79), exact decomposition:
//   * each correlated GPU event gets fp = path at its launch instant;
//   * per (pid, fp): sort fixed-event endpoints with the op segments whose
//     path == fp; where both are active the event behaves as an ordinary GPU
//     event of the current path ("own" pieces, re-injected as GPU endpoints),
//     elsewhere the union length goes to cell (fp, {GPU}) (set semantics);
//   * every fixed event also drives the tracked-only lane, so tracked time is
//     "mask != 0 or any fixed event active" as in the reference.
#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "xs_bucket.cuh"

namespace xs {

struct Cnt {
  int c[8];  // 0..4 categories 1..5, 5 tracked-only lane, 6 op endpoints
};
struct CntAdd {
  __device__ Cnt operator()(const Cnt& a, const Cnt& b) const {
    Cnt r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.c[i] = a.c[i] + b.c[i];
    return r;
  }
};

// lane update with compile-time indices only (a runtime index would put the
// state in local memory): cat 1..5 -> lanes 0..4, cat 6 -> lane 5, cat 0 ->
// op-endpoint count (lane 6, +1 for opens and closes)
__device__ __forceinline__ void apply_code(Cnt& s, uint32_t code) {
  const uint32_t cat = code & 7u;
  const int d = (code & 8u) ? -1 : 1;
#pragma unroll
  for (int i = 0; i < 6; i++) s.c[i] += (cat == (uint32_t)(i + 1)) ? d : 0;
  s.c[6] += cat == 0 ? 1 : 0;
}

// --------------------------------------------------------------------------
__global__ void __launch_bounds__(XS_BLOCK) k_keygen(EventView v, int64_t n, const int64_t* __restrict__ lo, int tb,
                                                     int corr_mode, uint64_t sentinel, uint64_t* __restrict__ keys) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t d = v.dur[i];
  uint2 out_lo, out_hi;
  uint64_t k0 = sentinel, k1 = sentinel;
  if (d > 0) {
    int p = v.ev.pid[i];
    uint32_t cat = v.ev.cat[i];
    if (corr_mode && cat == 5 && v.ev.has_corr[i]) cat = 6;
    uint64_t base = (uint64_t)p << (tb + 4);
    uint64_t s = (uint64_t)(v.start[i] - lo[p]);
    k0 = base | (s << 4) | cat;
    k1 = base | ((s + (uint64_t)d) << 4) | 8u | cat;
  }
  (void)out_lo;
  (void)out_hi;
  reinterpret_cast<ulonglong2*>(keys)[i] = make_ulonglong2(k0, k1);
}

// --------------------------------------------------------------------------
constexpr int SW_ITEMS = 16;
constexpr int SW_TILE = XS_BLOCK * SW_ITEMS;
constexpr int HT = 1024;  // shared hash slots per block

// The overlap histogram in global memory, keyed by
// idx = ((pid * n_nodes + node) * 32 + mask) (mask 0 of node 0 = tracked).
// Dense (key == nullptr): val[idx].  Hashed: an open-addressing table of
// mask + 1 slots, used when the dense [pid][node][32] layout would be too
// large (deep recursive operation scopes: hundreds of thousands of paths
// that each occur in one pid).  Its capacity is >= 2x a proven bound on the
// number of distinct cells, so probing terminates; `full` records the
// impossible case instead of dropping time.
struct GHist {
  unsigned long long* val;
  unsigned long long* key;
  unsigned long long mask;
  unsigned long long* full;
  __device__ __forceinline__ void add(unsigned long long idx, unsigned long long v) const {
    if (!key) {
      atomicAdd(&val[idx], v);
      return;
    }
    unsigned long long h = mix64(idx) & mask;
    for (unsigned long long probe = 0; probe <= mask; probe++) {
      unsigned long long k = ((volatile unsigned long long*)key)[h];
      if (k == ~0ull) {
        k = atomicCAS(&key[h], ~0ull, idx);
        if (k == ~0ull) k = idx;
      }
      if (k == idx) {
        atomicAdd(&val[h], v);
        return;
      }
      h = (h + 1) & mask;
    }
    atomicAdd(full, 1ull);
  }
};

__device__ __forceinline__ void hist_add(unsigned long long* s_key, unsigned long long* s_val,
                                         const GHist& hist, unsigned long long idx, unsigned long long v) {
  unsigned h = (unsigned)(mix64(idx) & (HT - 1));
#pragma unroll 1
  for (int probe = 0; probe < 16; probe++) {
    unsigned long long k = s_key[h];
    if (k == idx) {
      atomicAdd(&s_val[h], v);
      return;
    }
    if (k == ~0ull) {
      unsigned long long prev = atomicCAS(&s_key[h], ~0ull, idx);
      if (prev == ~0ull || prev == idx) {
        atomicAdd(&s_val[h], v);
        return;
      }
    }
    h = (h + 1) & (HT - 1);
  }
  hist.add(idx, v);
}

__global__ void __launch_bounds__(XS_BLOCK) k_sweep(const uint64_t* __restrict__ keys, int64_t nvalid, int tb,
                                                    const int* __restrict__ pidpath,
                                                    const int64_t* __restrict__ opbase, int n_nodes,
                                                    GHist hist, TileDesc<Cnt>* desc,
                                                    int* flags, int* tile_ctr) {
  __shared__ unsigned long long s_key[HT];
  __shared__ unsigned long long s_val[HT];
  for (int i = threadIdx.x; i < HT; i += XS_BLOCK) {
    s_key[i] = ~0ull;
    s_val[i] = 0;
  }
  const int tile = next_tile(tile_ctr);
  const int64_t base = (int64_t)tile * SW_TILE + (int64_t)threadIdx.x * SW_ITEMS;
  uint64_t k[SW_ITEMS + 1];
  if (base + SW_ITEMS <= nvalid) {
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(keys + base);
#pragma unroll
    for (int j = 0; j < SW_ITEMS / 2; j++) {
      ulonglong2 q = __ldcs(src + j);
      k[2 * j] = q.x;
      k[2 * j + 1] = q.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < SW_ITEMS; j++) k[j] = (base + j < nvalid) ? keys[base + j] : ~0ull;
  }
  k[SW_ITEMS] = (base + SW_ITEMS < nvalid) ? keys[base + SW_ITEMS] : ~0ull;
  Cnt agg;
#pragma unroll
  for (int i = 0; i < 8; i++) agg.c[i] = 0;
#pragma unroll
  for (int j = 0; j < SW_ITEMS; j++)
    if (base + j < nvalid) apply_code(agg, (uint32_t)(k[j] & 15u));
  Cnt zero;
#pragma unroll
  for (int i = 0; i < 8; i++) zero.c[i] = 0;
  Cnt cur = grid_exclusive(agg, CntAdd(), zero, tile, desc, flags);
  const uint64_t tmask = (1ull << tb) - 1;
  const int pshift = tb + 4;
  // running per-thread accumulators: one cell key and the pid's tracked time
  unsigned long long run_idx = ~0ull, run_len = 0;
  int tr_pid = -1;
  long long tr_len[1] = {0};
#pragma unroll
  for (int j = 0; j < SW_ITEMS; j++) {
    if (base + j >= nvalid) break;
    const uint64_t kj = k[j];
    apply_code(cur, (uint32_t)(kj & 15u));
    if (base + j + 1 >= nvalid) break;
    const uint64_t kn = k[j + 1];
    if ((kn >> 4) == (kj >> 4) || (kn >> pshift) != (kj >> pshift)) continue;
    const unsigned long long len = ((kn >> 4) & tmask) - ((kj >> 4) & tmask);
    const int p = (int)(kj >> pshift);
    unsigned mask = 0;
#pragma unroll
    for (int c = 0; c < 5; c++) mask |= (cur.c[c] > 0 ? 1u : 0u) << c;
    const unsigned long long prow = (unsigned long long)p * (unsigned long long)n_nodes;
    if (mask || cur.c[5] > 0) {
      if (p != tr_pid) {
        if (tr_pid >= 0 && tr_len[0]) hist_add(s_key, s_val, hist, (unsigned long long)tr_pid * n_nodes * 32ull,
                                               (unsigned long long)tr_len[0]);
        tr_pid = p;
        tr_len[0] = 0;
      }
      tr_len[0] += (long long)len;
    }
    if (mask) {
      const int64_t c = cur.c[6];
      const int path = c > opbase[p] ? pidpath[c - 1] : 0;
      const unsigned long long idx = (prow + (unsigned long long)path) * 32ull + mask;
      if (idx != run_idx) {
        if (run_idx != ~0ull) hist_add(s_key, s_val, hist, run_idx, run_len);
        run_idx = idx;
        run_len = 0;
      }
      run_len += len;
    }
  }
  if (run_idx != ~0ull) hist_add(s_key, s_val, hist, run_idx, run_len);
  block_keyed_flush<1>(tr_pid, tr_len, [&](int p, const long long* x) {
    if (x[0]) hist_add(s_key, s_val, hist, (unsigned long long)p * n_nodes * 32ull, (unsigned long long)x[0]);
  });
  __syncthreads();
  for (int i = threadIdx.x; i < HT; i += XS_BLOCK) {
    unsigned long long key = s_key[i];
    if (key != ~0ull) hist.add(key, s_val[i]);
  }
}

// dense histogram -> (pid, node, mask, ns) list + tracked per pid
__global__ void k_compact_cells(GHist hist, int64_t total, int n_nodes, int* cell_pid,
                                int* cell_node, int* cell_mask, int64_t* cell_ns, int64_t* tracked,
                                unsigned long long* count) {
  const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long vv = slot < total ? hist.val[slot] : 0ull;
  int p = 0, node = 0, mask = 0;
  if (vv) {
    const int64_t i = hist.key ? (int64_t)hist.key[slot] : slot;
    mask = (int)(i & 31);
    const int64_t row = i >> 5;
    p = (int)(row / n_nodes);
    node = (int)(row % n_nodes);
    if (mask == 0 && node == 0) tracked[p] = (int64_t)vv;
  }
  // one counter atomic per block: threads with a cell take consecutive slots
  const bool cell = vv && mask != 0;
  const unsigned long long at = block_reserve(count, cell ? 1u : 0u);
  if (!cell) return;
  cell_pid[at] = p;
  cell_node[at] = node;
  cell_mask[at] = mask;
  cell_ns[at] = (int64_t)vv;
}

__global__ void k_trie_count_to_stats(const int* count, Stats* st) {
  if (threadIdx.x == 0) st->pad[0] = *count;
}

// --------------------------------------------------------------------------
// CORRELATION support
// --------------------------------------------------------------------------
__device__ __forceinline__ int path_at(const uint64_t* pk, const int* pidpath, const int64_t* opbase, int p,
                                       uint64_t t_rel, int tb) {
  int64_t a = opbase[p], b = opbase[p + 1];
  const uint64_t tmask = (1ull << tb) - 1;
  int64_t lo = a, hi = b;
  while (lo < hi) {  // last index with time <= t
    int64_t mid = (lo + hi) >> 1;
    if (((pk[mid] >> 1) & tmask) <= t_rel) lo = mid + 1;
    else hi = mid;
  }
  return lo > a ? pidpath[lo - 1] : 0;
}

// FX record key: pid | path | t | code2  (code2: 0 S-, 1 S+, 2 F-, 3 F+)
__global__ void k_fx_fixed(EventView v, int64_t n, const int64_t* lo, const int64_t* launch, const uint64_t* pk,
                           const int* pidpath, const int64_t* opbase, int tb, int nodeb, uint64_t* fx,
                           unsigned long long* fx_count) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (v.ev.cat[i] != 5 || !v.ev.has_corr[i] || v.dur[i] <= 0) return;
  int p = v.ev.pid[i];
  int64_t ls = launch[i];
  int fp = path_at(pk, pidpath, opbase, p, (uint64_t)(ls - lo[p]), tb);
  uint64_t grp = (((uint64_t)p << nodeb) | (uint64_t)fp) << (tb + 2);
  uint64_t s = (uint64_t)(v.start[i] - lo[p]);
  uint64_t e = s + (uint64_t)v.dur[i];
  unsigned long long at = atomicAdd(fx_count, 2ull);
  fx[at] = grp | (s << 2) | 3u;
  fx[at + 1] = grp | (e << 2) | 2u;
}

// op segments: every pk run end opens a segment of its path until the next
// run of the pid (or +inf); the root path covers [0, first run)
__global__ void k_fx_segments(const uint64_t* pk, int64_t n2, const int* pidpath, int tb, int nodeb, uint64_t* fx,
                              unsigned long long* fx_count) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n2) return;
  const uint64_t tmask = (1ull << tb) - 1;
  uint64_t key = pk[k] >> 1;
  if (k + 1 < n2 && (pk[k + 1] >> 1) == key) return;
  uint64_t p = key >> tb;
  uint64_t t = key & tmask;
  uint64_t tn = tmask;
  if (k + 1 < n2 && (pk[k + 1] >> (tb + 1)) == p) tn = (pk[k + 1] >> 1) & tmask;
  uint64_t grp = ((p << nodeb) | (uint64_t)pidpath[k]) << (tb + 2);
  unsigned long long at = atomicAdd(fx_count, 2ull);
  fx[at] = grp | (t << 2) | 1u;
  fx[at + 1] = grp | (tn << 2) | 0u;
}

__global__ void k_fx_root(const uint64_t* pk, const int64_t* opbase, int np, int tb, int nodeb, uint64_t* fx,
                          unsigned long long* fx_count) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= np) return;
  const uint64_t tmask = (1ull << tb) - 1;
  uint64_t tn = opbase[p] < opbase[p + 1] ? ((pk[opbase[p]] >> 1) & tmask) : tmask;
  uint64_t grp = ((uint64_t)p << nodeb) << (tb + 2);
  unsigned long long at = atomicAdd(fx_count, 2ull);
  fx[at] = grp | 1u;
  fx[at + 1] = grp | (tn << 2) | 0u;
}

struct FS {
  int f, s;
};
struct FSAdd {
  __device__ FS operator()(const FS& a, const FS& b) const { return FS{a.f + b.f, a.s + b.s}; }
};

constexpr int FX_ITEMS = 4;
__global__ void __launch_bounds__(XS_BLOCK) k_fx_scan(const uint64_t* fx, int64_t nvalid, int tb, int nodeb,
                                                      int n_nodes, GHist hist, uint64_t* pieces,
                                                      unsigned long long* piece_count, TileDesc<FS>* desc, int* flags,
                                                      int* tile_ctr) {
  const int tile = next_tile(tile_ctr);
  const int64_t base = (int64_t)tile * XS_BLOCK * FX_ITEMS + (int64_t)threadIdx.x * FX_ITEMS;
  uint64_t k[FX_ITEMS + 1];
#pragma unroll
  for (int j = 0; j <= FX_ITEMS; j++) k[j] = (base + j < nvalid) ? fx[base + j] : ~0ull;
  FS agg{0, 0};
#pragma unroll
  for (int j = 0; j < FX_ITEMS; j++) {
    if (base + j >= nvalid) break;
    uint32_t c = (uint32_t)(k[j] & 3u);
    if (c & 2u) agg.f += (c & 1u) ? 1 : -1;
    else agg.s += (c & 1u) ? 1 : -1;
  }
  FS cur = grid_exclusive(agg, FSAdd(), FS{0, 0}, tile, desc, flags);
  const uint64_t tmask = (1ull << tb) - 1;
  const uint64_t nmask = (1ull << nodeb) - 1;
#pragma unroll
  for (int j = 0; j < FX_ITEMS; j++) {
    if (base + j >= nvalid) break;
    uint64_t kj = k[j];
    uint32_t c = (uint32_t)(kj & 3u);
    if (c & 2u) cur.f += (c & 1u) ? 1 : -1;
    else cur.s += (c & 1u) ? 1 : -1;
    if (base + j + 1 >= nvalid) break;
    uint64_t kn = k[j + 1];
    if ((kn >> 2) == (kj >> 2) || (kn >> (tb + 2)) != (kj >> (tb + 2))) continue;
    if (cur.f <= 0) continue;
    uint64_t t0 = (kj >> 2) & tmask, t1 = (kn >> 2) & tmask;
    uint64_t grp = kj >> (tb + 2);
    uint64_t p = grp >> nodeb, path = grp & nmask;
    if (cur.s > 0) {  // own piece: behaves as a GPU event of the current path
      unsigned long long at = atomicAdd(piece_count, 2ull);
      uint64_t pb = p << (tb + 4);
      pieces[at] = pb | (t0 << 4) | 5u;
      pieces[at + 1] = pb | (t1 << 4) | 13u;
    } else {  // foreign: (fp, {GPU}) gets the union length
      hist.add(((unsigned long long)p * n_nodes + path) * 32ull + 16ull, (unsigned long long)(t1 - t0));
    }
  }
}

// --------------------------------------------------------------------------
// Bucketed sort fused with the sweep (xs_bucket.cuh)
// --------------------------------------------------------------------------
__device__ __forceinline__ void event_keys(const EventView& v, int64_t i, const int64_t* lo, int tb, int corr_mode,
                                           uint64_t& k0, uint64_t& k1, bool& valid) {
  const int64_t d = v.dur[i];
  valid = d > 0;
  k0 = k1 = 0;
  if (!valid) return;
  const int p = v.ev.pid[i];
  uint32_t cat = v.ev.cat[i];
  if (corr_mode && cat == 5 && v.ev.has_corr[i]) cat = 6;
  const uint64_t base = (uint64_t)p << (tb + 4);
  const uint64_t st = (uint64_t)(v.start[i] - lo[p]);
  k0 = base | (st << 4) | cat;
  k1 = base | ((st + (uint64_t)d) << 4) | 8u | cat;
}

__global__ void __launch_bounds__(XS_BLOCK) k_bk_hist(EventView v, int64_t n, const int64_t* __restrict__ lo, int tb,
                                                      int corr_mode, const uint64_t* extra, int64_t n_extra,
                                                      int shift, unsigned* counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t k0 = 0, k1 = 0;
  bool v0 = false, v1 = false;
  if (i < n) {
    bool valid;
    event_keys(v, i, lo, tb, corr_mode, k0, k1, valid);
    v0 = v1 = valid;
  } else if (i - n < (n_extra + 1) / 2) {
    const int64_t q = 2 * (i - n);
    k0 = extra[q];
    v0 = true;
    v1 = q + 1 < n_extra;
    k1 = v1 ? extra[q + 1] : 0;
  }
  // warp-collective: every lane reaches both calls
  bucket_count(counts, (uint32_t)(k0 >> shift), v0);
  bucket_count(counts, (uint32_t)(k1 >> shift), v1);
}

__global__ void __launch_bounds__(XS_BLOCK) k_bk_scatter(EventView v, int64_t n, const int64_t* __restrict__ lo, int tb,
                                                         int corr_mode, const uint64_t* extra, int64_t n_extra,
                                                         int shift, unsigned* counts, const int64_t* offs,
                                                         uint64_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t k0 = 0, k1 = 0;
  bool v0 = false, v1 = false;
  if (i < n) {
    bool valid;
    event_keys(v, i, lo, tb, corr_mode, k0, k1, valid);
    v0 = v1 = valid;
  } else if (i - n < (n_extra + 1) / 2) {
    const int64_t q = 2 * (i - n);
    k0 = extra[q];
    v0 = true;
    v1 = q + 1 < n_extra;
    k1 = v1 ? extra[q + 1] : 0;
  }
  const int64_t s0 = bucket_slot(counts, offs, (uint32_t)(k0 >> shift), v0);
  if (v0) out[s0] = k0;
  const int64_t s1 = bucket_slot(counts, offs, (uint32_t)(k1 >> shift), v1);
  if (v1) out[s1] = k1;
}

struct SwState {
  int c[8];  // as Cnt
  unsigned long long last;
  int has;
  int pad;
};
struct SwOp {
  __device__ SwState operator()(const SwState& a, const SwState& b) const {
    SwState r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.c[i] = a.c[i] + b.c[i];
    r.last = b.has ? b.last : a.last;
    r.has = a.has | b.has;
    r.pad = 0;
    return r;
  }
};

// Packed endpoint counters.  Seven counters (categories 1..6 = lanes 0..5,
// OPERATION endpoints = lane 6) as 16-bit lanes of two words, summed as
// plain 64-bit integers: a sum of per-key deltas is the polynomial
// sum c_i 2^(16 i), exact as long as every true lane value fits in
// [-2^15, 2^15) -- a chunk holds <= BK_CAP keys, so chunk-local partial
// counts always do.  Decoding propagates the borrows lane by lane.
struct P2 {
  unsigned long long a, b;  // lanes 0..3 | lanes 4..6
};
struct IAdd {
  __device__ int operator()(int x, int y) const { return x + y; }
};
struct P2Add {
  __device__ P2 operator()(const P2& x, const P2& y) const { return P2{x.a + y.a, x.b + y.b}; }
};
__device__ __forceinline__ void p2_apply(P2& s, uint32_t code) {
  const uint32_t cat = code & 7u;
  const uint32_t lane = cat == 0 ? 6u : cat - 1u;
  const unsigned long long one = 1ull << (16 * (lane & 3u));
  const unsigned long long d = (cat != 0 && (code & 8u)) ? 0ull - one : one;  // (ops count both endpoints)
  if (lane < 4) s.a += d;
  else s.b += d;
}
__device__ __forceinline__ void p2_decode(P2 s, int* c /*[7]*/) {
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int v = (int)(short)(unsigned short)(s.a & 0xFFFFu);
    c[i] = v;
    s.a = (s.a - (unsigned long long)(long long)v) >> 16;
  }
#pragma unroll
  for (int i = 0; i < 3; i++) {
    const int v = (int)(short)(unsigned short)(s.b & 0xFFFFu);
    c[4 + i] = v;
    s.b = (s.b - (unsigned long long)(long long)v) >> 16;
  }
}

// Shared-memory cell table: every add is a length < 2^28 (an interval inside
// one chunk, whose relative keys span < 2^32 = 2^28 ns), split into its low
// 16 bits and the rest, each added to its own 32-bit counter without reading
// it back (fire-and-forget RED; a 64-bit shared atomicAdd is a CAS loop on
// sm_100).  A chunk makes <= BK_CAP adds per cell, so neither counter can
// wrap: value = lo + (hi << 16).
__device__ __forceinline__ void smem_add_split(unsigned* lo, unsigned* hi, unsigned v) {
  atomicAdd(lo, v & 0xFFFFu);
  if (v >> 16) atomicAdd(hi, v >> 16);
}
__device__ __forceinline__ unsigned long long split_value(unsigned lo, unsigned hi) {
  return (unsigned long long)lo + ((unsigned long long)hi << 16);
}

template <int kHT>
struct CellTableT {  // open addressing in shared memory, spill to global
  unsigned long long* key;
  unsigned* lo;
  unsigned* hi;
  __device__ __noinline__ void add(unsigned long long idx, unsigned v, const GHist& hist) {
    unsigned h = (unsigned)(mix64(idx) & (kHT - 1));
#pragma unroll 1
    for (int probe = 0; probe < 16; probe++) {
      unsigned long long k = key[h];
      if (k != idx && k == ~0ull) {
        unsigned long long prev = atomicCAS(&key[h], ~0ull, idx);
        k = prev == ~0ull ? idx : prev;
      }
      if (k == idx) {
        smem_add_split(&lo[h], &hi[h], v);
        return;
      }
      h = (h + 1) & (kHT - 1);
    }
    hist.add(idx, v);
  }
};

template <int kHT>
struct BkSmemT {
  static constexpr int NBW = 4 * kHT;     // words of local counting-sort bins: exactly the cell table's bytes
  static constexpr int NBINS = 2 * NBW;  // 16-bit bins (a count or start is <= BK_CAP)
  // chunk keys relative to the chunk base: load order, then fully sorted at
  // bk_sw(position) (one pad word per 16: a thread's 16 consecutive items are
  // conflict-free across the warp)
  uint32_t k[BK_CAP + BK_CAP / 16];
  uint32_t sorted[BK_CAP];  // keys grouped by local bin (also block-radix-sort scratch together with k[])
  union {
    struct {
      unsigned long long h_key[kHT];
      unsigned h_lo[kHT];
      unsigned h_hi[kHT];
    } t;
    unsigned bins[NBW];  // 16-bit counts, then exclusive starts (dead before the table is initialised)
  } u;
  P2 warp_p2[BK_THREADS / 32];
  uint32_t wmin[BK_THREADS / 32], wmax[BK_THREADS / 32];
  SwState tile_pre;
  SwState tile_agg;
};

// the shared cell table of the fused sweep: 1K slots (4 CTAs/SM) when a chunk's
// cells index it directly, 4K slots (2 CTAs/SM) for many-path traces whose
// cells must hash (deep recursive operations: fewer spills to the global table)
constexpr int HT_SMALL = 1024, HT_BIG = 4096;
constexpr int BK_BIN_BIG = 256;  // a local bin holding more keys sends the chunk to the block radix sort
__device__ __forceinline__ int bk_sw(int p) { return p + (p >> 4); }

__device__ __forceinline__ SwState sw_identity() {
  SwState id;
#pragma unroll
  for (int i = 0; i < 8; i++) id.c[i] = 0;
  id.last = 0;
  id.has = 0;
  id.pad = 0;
  return id;
}

// One CTA per chunk (a contiguous key range, <= BK_CAP keys, arriving grouped
// by global bucket).  The chunk is sorted in shared memory by one counting
// pass over 4*kHT local bins spanning exactly [min key, max key] of the chunk
// (so the bins adapt to how the keys cluster), then by direct comparison
// inside each bin (a few keys; one bin per distinct key when the chunk's range
// fits the bins).  The chunk aggregate (counts, max key) does not depend on
// order and is published right after the load, so the look-back chain never
// waits on a sort.  The walk keeps the six category counters as 8-bit lanes
// of one word clamped to BK_ITEMS + 1 (a thread applies at most BK_ITEMS
// endpoints, so "count > 0" is exact), the mask is a SWAR test, and every
// interval [t_prev, t) is accounted by the first endpoint of the run at t
// with the state after everything up to t_prev; across chunk boundaries
// t_prev and that state come from the look-back.
#ifndef XS_SWEEP_MINB
#define XS_SWEEP_MINB 4  // 4 CTAs per SM (64 registers): more chunks in flight
#endif
template <int kHT, int kMinB>
__global__ void __launch_bounds__(BK_THREADS, kMinB) k_bk_sweep(
    const uint64_t* __restrict__ keys, int64_t total, const int64_t* __restrict__ chunk, int shift, int tb,
    const int* __restrict__ pidpath, const int64_t* __restrict__ opbase, int n_nodes,
    GHist hist, TileDesc<SwState>* desc, int* flags, int* tile_ctr, Stats* st,
    unsigned long long* ptrace, int direct_ok, const int* trie_count) {
  using BkSmem = BkSmemT<kHT>;
  using CellTable = CellTableT<kHT>;
  constexpr int HT = kHT;
  constexpr int NB = BkSmem::NBINS;
  constexpr int NBW = BkSmem::NBW;
  constexpr int LOG_NB = kHT == 1024 ? 13 : 15;
  static_assert((1 << LOG_NB) == NB, "bins");
  constexpr int WPT = NBW / BK_THREADS;  // bin words per thread in the bin scan
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BkSmem& S = *reinterpret_cast<BkSmem*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // direct-indexed cells (path * 32 + mask) when the chunk holds one pid and
  // the paths actually interned fit the table (decided on the device: the
  // host only knows the trie's capacity without a sync)
  const int direct = direct_ok && trie_count && (int64_t)(*trie_count) * 32 <= kHT;
  // developer timing: per-phase globaltimer stamps of every CTA (XS_TRACE_SWEEP)
  unsigned long long ts0 = 0;
  if (ptrace && t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts0));
#define XS_STAMP(i)                                                  \
  if (ptrace && t == 0) {                                            \
    unsigned long long ts_;                                          \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts_));          \
    ptrace[c * 8 + (i)] = ts_;                                       \
  }
  {
    int4* b4 = reinterpret_cast<int4*>(S.u.bins);
    for (int i = t; i < NBW / 4; i += BK_THREADS) b4[i] = make_int4(0, 0, 0, 0);
  }
  const int64_t c = next_tile(tile_ctr);  // (barrier inside: also orders the bin reset)
  if (ptrace && t == 0) ptrace[c * 8] = ts0;
  XS_STAMP(1);
  const int64_t s0 = chunk[4 * c + 0];
  int cnt = s0 < 0 ? 0 : (int)(chunk[4 * c + 1] - s0);
  const int64_t b0 = chunk[4 * c + 2], b1 = chunk[4 * c + 3];
  // base aligned to 16 (keeps the 4-bit endpoint code) and to 2^shift
  const uint64_t base = ((uint64_t)b0 << shift) & ~15ull;
  const int lbits = bits_for(((uint64_t)(b1 > b0 ? b1 : b0 + 1) << shift) - 1 - base);
  if (cnt > BK_CAP || (cnt > 0 && lbits > 32)) {  // host re-runs this call through the LSD path
    if (t == 0) atomicAdd((unsigned long long*)&st->pad[3], 1ull);
    cnt = 0;
  }
  // 1. load (striped, coalesced) + the order-independent chunk aggregate
  P2 agg{0ull, 0ull};
  uint32_t kmin = 0xFFFFFFFFu, kmax = 0;
#pragma unroll
  for (int j = 0; j < BK_ITEMS; j++) {
    const int idx = j * BK_THREADS + t;
    if (idx < cnt) {
      const uint32_t kr = (uint32_t)(keys[s0 + idx] - base);
      S.k[idx] = kr;
      p2_apply(agg, kr);
      kmin = kr < kmin ? kr : kmin;
      kmax = kr > kmax ? kr : kmax;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    agg.a += __shfl_xor_sync(0xffffffffu, agg.a, o);
    agg.b += __shfl_xor_sync(0xffffffffu, agg.b, o);
  }
  kmin = __reduce_min_sync(0xffffffffu, kmin);
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  if (lane == 0) {
    S.warp_p2[warp] = agg;
    S.wmin[warp] = kmin;
    S.wmax[warp] = kmax;
  }
  __syncthreads();
#pragma unroll
  for (int w = 0; w < BK_THREADS / 32; w++) {
    kmin = S.wmin[w] < kmin ? S.wmin[w] : kmin;
    kmax = S.wmax[w] > kmax ? S.wmax[w] : kmax;
  }
  if (warp == 0) {
    SwState tile_agg = sw_identity();
    P2 ta{0ull, 0ull};
#pragma unroll
    for (int w = 0; w < BK_THREADS / 32; w++) ta = P2Add()(ta, S.warp_p2[w]);
    int cc[7];
    p2_decode(ta, cc);
#pragma unroll
    for (int i = 0; i < 7; i++) tile_agg.c[i] = cc[i];
    tile_agg.has = cnt > 0;
    tile_agg.last = cnt > 0 ? base + kmax : 0;
    if (lane == 0) {
      tile_publish_agg((int)c, tile_agg, desc, flags);
      S.tile_agg = tile_agg;  // (kept for the look-back: not live in registers through the sort)
    }
  }
  XS_STAMP(2);
  // 2. counting pass over the local bins (kr - kmin) >> s2
  const int rbits = cnt > 0 ? bits_for((uint64_t)(kmax - kmin)) : 0;
  const int s2 = rbits > LOG_NB ? rbits - LOG_NB : 0;
  uint32_t slot[BK_ITEMS / 2];  // two 16-bit slots per word (a slot is < BK_CAP)
#pragma unroll
  for (int j = 0; j < BK_ITEMS; j++) {
    const int idx = j * BK_THREADS + t;
    uint32_t sl = 0;
    if (idx < cnt) {
      const uint32_t b = (S.k[idx] - kmin) >> s2, h = 16 * (b & 1);
      sl = (atomicAdd(&S.u.bins[b >> 1], 1u << h) >> h) & 0xFFFFu;
    }
    if (j & 1) slot[j >> 1] |= sl << 16;
    else slot[j >> 1] = sl;
  }
  __syncthreads();
  bool big = false;
  {  // exclusive bin starts: 2 * WPT consecutive bins per thread + a block scan
    unsigned w[WPT];
    uint4* b4 = reinterpret_cast<uint4*>(S.u.bins + t * WPT);
#pragma unroll
    for (int q = 0; q < WPT / 4; q++) {
      const uint4 x = b4[q];
      w[4 * q] = x.x;
      w[4 * q + 1] = x.y;
      w[4 * q + 2] = x.z;
      w[4 * q + 3] = x.w;
    }
    int sum = 0;
#pragma unroll
    for (int q = 0; q < WPT; q++) {
      const unsigned lo = w[q] & 0xFFFFu, hi = w[q] >> 16;
      big |= lo > BK_BIN_BIG || hi > BK_BIN_BIG;
      w[q] = (unsigned)sum | ((unsigned)(sum + lo) << 16);  // (starts relative to this thread's first bin)
      sum += lo + hi;
    }
    int dummy;
    const int pre = block_exclusive_fast(sum, IAdd(), 0, reinterpret_cast<int*>(S.warp_p2), &dummy);
    const unsigned pp = (unsigned)pre | ((unsigned)pre << 16);
#pragma unroll
    for (int q = 0; q < WPT / 4; q++)
      b4[q] = make_uint4(w[4 * q] + pp, w[4 * q + 1] + pp, w[4 * q + 2] + pp, w[4 * q + 3] + pp);
  }
  big = __syncthreads_or(big) != 0;
  // scatter into bin order
#pragma unroll
  for (int j = 0; j < BK_ITEMS; j++) {
    const int idx = j * BK_THREADS + t;
    if (idx < cnt) {
      const uint32_t kr = S.k[idx];
      const uint32_t b = (kr - kmin) >> s2;
      S.sorted[((S.u.bins[b >> 1] >> (16 * (b & 1))) & 0xFFFFu) + ((slot[j >> 1] >> (16 * (j & 1))) & 0xFFFFu)] = kr;
    }
  }
  __syncthreads();
  XS_STAMP(3);
  if (!big) {
    // 3. order inside each bin: a bin of one key value (s2 == 0) is already
    // in place; otherwise rank by direct comparison (ties by position)
#pragma unroll 4
    for (int j = 0; j < BK_ITEMS; j++) {
      const int i = j * BK_THREADS + t;
      if (i >= cnt) break;
      const uint32_t k = S.sorted[i];
      if (s2 == 0) {
        S.k[bk_sw(i)] = k;
        continue;
      }
      const int b = (int)((k - kmin) >> s2);
      const int bs = (int)((S.u.bins[b >> 1] >> (16 * (b & 1))) & 0xFFFFu);
      const int be = b + 1 < NB ? (int)((S.u.bins[(b + 1) >> 1] >> (16 * ((b + 1) & 1))) & 0xFFFFu) : cnt;
      int r = 0;
      for (int q = bs; q < be; q++) {
        const uint32_t o = S.sorted[q];
        r += (o < k) | ((o == k) & (q < i));
      }
      S.k[bk_sw(bs + r)] = k;
    }
  } else {  // a dense bin: block radix sort of the whole chunk on lbits
    using BRS = cub::BlockRadixSort<uint32_t, BK_THREADS, BK_ITEMS, cub::NullType, 4>;
    static_assert(sizeof(typename BRS::TempStorage) <= 2 * sizeof(uint32_t) * BK_CAP, "radix scratch");
    typename BRS::TempStorage& tmp = *reinterpret_cast<typename BRS::TempStorage*>(S.k);
    uint32_t kk[BK_ITEMS];
#pragma unroll
    for (int j = 0; j < BK_ITEMS; j++) {
      const int idx = j * BK_THREADS + t;
      kk[j] = idx < cnt ? S.sorted[idx] : 0xFFFFFFFFu;
    }
    __syncthreads();
    BRS(tmp).Sort(kk, 0, lbits < 1 ? 1 : lbits);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < BK_ITEMS; j++) {
      const int idx = t * BK_ITEMS + j;  // blocked output
      if (idx < cnt) S.k[bk_sw(idx)] = kk[j];
    }
  }
  __syncthreads();
  // the cell table takes over the bins' bytes
  for (int i = t; i < HT; i += BK_THREADS) {
    S.u.t.h_key[i] = ~0ull;
    S.u.t.h_lo[i] = 0;
    S.u.t.h_hi[i] = 0;
  }
  XS_STAMP(4);
  // 4. thread prefix over this thread's sorted items + chunk prefix
  const int my0 = t * BK_ITEMS;
  const int nmine = cnt - my0 < 0 ? 0 : (cnt - my0 > BK_ITEMS ? BK_ITEMS : cnt - my0);
  const uint32_t* mine = S.k + bk_sw(my0);  // (a thread's items never straddle a pad word)
  P2 ta{0ull, 0ull};
#pragma unroll 4
  for (int j = 0; j < nmine; j++) p2_apply(ta, mine[j]);
  P2 dummy;
  const P2 excl = block_exclusive_fast(ta, P2Add(), P2{0ull, 0ull}, S.warp_p2, &dummy);
  if (warp == 0) {
    SwState pre = tile_lookback_published((int)c, S.tile_agg, desc, flags, SwOp(), sw_identity());
    if (lane == 0) S.tile_pre = pre;
  }
  __syncthreads();
  XS_STAMP(5);
  int ex[7];
  p2_decode(excl, ex);
  // six category counters as 8-bit lanes, clamped (exact for "> 0" over this
  // thread's <= BK_ITEMS endpoints); OPERATION endpoints counted exactly
  unsigned long long x = 0;
#pragma unroll
  for (int i = 0; i < 6; i++) {
    const int v = S.tile_pre.c[i] + ex[i];
    x |= (unsigned long long)(v < BK_ITEMS + 1 ? v : BK_ITEMS + 1) << (8 * i);
  }
  int64_t oc = (int64_t)S.tile_pre.c[6] + ex[6];
  // 5. the sweep over this thread's items
  const uint64_t tmask = (1ull << tb) - 1;
  const int pshift = tb + 4;
  constexpr unsigned long long L7F = 0x7F7F7F7F7F7Full, H6 = 0x808080808080ull, H5 = 0x8080808080ull;
  // lanes 0..4 of a positive-lane word -> mask bits 0..4 (bit 8i lands on 28 + i)
  auto mask_of = [](unsigned long long m5) -> unsigned { return (unsigned)((((m5 >> 7) * 0x10204081ull) >> 28) & 31u); };
  auto apply = [&](uint32_t code) {
    const uint32_t cat = code & 7u;
    if (cat == 0) {
      oc++;
    } else {
      const unsigned long long one = 1ull << (8 * (cat - 1));
      x = (code & 8u) ? x - one : x + one;
    }
  };
  // path of the op count oc is pidpath[oc - 1]; consecutive op endpoints read
  // consecutive entries, so the entry after the current one is loaded one op
  // endpoint ahead (its latency hides behind the keys in between)
  int64_t pf_oc = oc;
  int pf_cur = 0, pf_nxt = 0;
  if (pidpath && nmine > 0) {
    pf_cur = pf_oc >= 1 ? pidpath[pf_oc - 1] : 0;
    pf_nxt = pidpath[pf_oc];  // (allocated 2m + 2: in bounds even past the last endpoint)
  }
  auto path_at = [&](int64_t o) -> int {
    if (o == pf_oc) return pf_cur;
    if (o == pf_oc + 1) {
      pf_cur = pf_nxt;
    } else {
      pf_cur = o >= 1 ? pidpath[o - 1] : 0;
    }
    pf_oc = o;
    pf_nxt = pidpath[o];
    return pf_cur;
  };
  CellTable T{S.u.t.h_key, S.u.t.h_lo, S.u.t.h_hi};
  const uint64_t first_pid = (base + kmin) >> pshift;
  const bool single = cnt > 0 && first_pid == ((base + kmax) >> pshift);  // (block-uniform)
  const unsigned long long pbase = first_pid * (unsigned long long)n_nodes * 32ull;
  if (single) {
    const int p = (int)first_pid;
    const int64_t ob = opbase[p];
    // the interval from the previous chunk's last endpoint (thread 0's first
    // item) can be longer than 2^28: straight to the global histogram
    if (t == 0 && nmine > 0 && S.tile_pre.has) {
      const uint64_t prev = S.tile_pre.last, k = base + mine[0];
      if ((prev >> pshift) == (uint64_t)p && (prev >> 4) != (k >> 4)) {
        const unsigned long long pos = (x + L7F) & H6;
        if (pos) {
          const unsigned long long len = ((k >> 4) & tmask) - ((prev >> 4) & tmask);
          hist.add(pbase, len);
          const unsigned long long m5 = pos & H5;
          if (m5) hist.add(pbase + (unsigned long long)(oc > ob ? path_at(oc) : 0) * 32ull + mask_of(m5), len);
        }
      }
    }
    // everything else: 32-bit times relative to the chunk base
    uint32_t tprev = t > 0 && nmine > 0 ? S.k[bk_sw(my0 - 1)] >> 4 : 0;
    bool hp = t > 0;
    unsigned tracked = 0;
    int64_t c_oc = -1;
    unsigned c_cell = 0;
    unsigned run_k = ~0u, run_v = 0;
    auto flush_run = [&](unsigned key, unsigned v) {
      if (direct) smem_add_split(&S.u.t.h_lo[key], &S.u.t.h_hi[key], v);
      else T.add(pbase + key, v, hist);
    };
#pragma unroll 4
    for (int j = 0; j < nmine; j++) {
      const uint32_t kr = mine[j], tr = kr >> 4;
      if (hp && tr != tprev) {
        const unsigned long long pos = (x + L7F) & H6;
        if (pos) {
          const unsigned len = tr - tprev;
          tracked += len;
          const unsigned long long m5 = pos & H5;
          if (m5) {
            if (oc != c_oc) {  // the path only changes at OPERATION endpoints
              c_oc = oc;
              c_cell = (unsigned)(oc > ob ? path_at(oc) : 0) * 32u;
            }
            const unsigned key = c_cell + mask_of(m5);
            if (key == run_k) {
              run_v += len;
            } else {
              if (run_k != ~0u) flush_run(run_k, run_v);
              run_k = key;
              run_v = len;
            }
          }
        }
      }
      apply(kr);
      tprev = tr;
      hp = true;
    }
    XS_STAMP(6);
    if (run_k != ~0u) flush_run(run_k, run_v);
    // tracked time: one per chunk (cell 0 of the pid = path 0, mask 0)
#pragma unroll
    for (int o = 16; o; o >>= 1) tracked += __shfl_xor_sync(0xffffffffu, tracked, o);
    if (lane == 0 && tracked) flush_run(0u, tracked);
  } else {
    // chunks holding several pids (traces with more pids than buckets):
    // 64-bit keys, every cell through the hashed table
    uint64_t prev = 0;
    bool have_prev = false;
    if (t == 0) {
      have_prev = S.tile_pre.has;
      prev = S.tile_pre.last;
    } else if (nmine > 0) {
      have_prev = true;
      prev = base + S.k[bk_sw(my0 - 1)];
    }
    int c_pid = -1;
    int64_t c_ob = 0, c_oc = -1;
    unsigned long long c_cell = 0;
#pragma unroll 1
    for (int j = 0; j < nmine; j++) {
      const uint64_t k = base + mine[j];
      if (have_prev && (prev >> 4) != (k >> 4) && (prev >> pshift) == (k >> pshift)) {
        const unsigned long long pos = (x + L7F) & H6;
        if (pos) {
          const unsigned long long len = ((k >> 4) & tmask) - ((prev >> 4) & tmask);
          const int p = (int)(k >> pshift);
          const unsigned long long pb = (unsigned long long)p * n_nodes * 32ull;
          hist.add(pb, len);  // (rare path: no run merging)
          const unsigned long long m5 = pos & H5;
          if (m5) {
            if (p != c_pid) {
              c_pid = p;
              c_ob = opbase[p];
              c_oc = -1;
            }
            if (oc != c_oc) {
              c_oc = oc;
              c_cell = pb + (unsigned long long)(oc > c_ob ? path_at(oc) : 0) * 32ull;
            }
            hist.add(c_cell + mask_of(m5), len);
          }
        }
      }
      apply(mine[j]);
      prev = k;
      have_prev = true;
    }
    XS_STAMP(6);
  }
  __syncthreads();
  for (int i = t; i < HT; i += BK_THREADS) {
    const unsigned long long v = split_value(S.u.t.h_lo[i], S.u.t.h_hi[i]);
    if (direct) {
      if (v) hist.add(pbase + (unsigned long long)i, v);
    } else {
      const unsigned long long key = S.u.t.h_key[i];
      if (key != ~0ull) hist.add(key, v);
    }
  }
  XS_STAMP(7);
#undef XS_STAMP
}



// host driver for the bucketed endpoint sort + sweep
// phase 1: endpoint keys histogrammed, bucket offsets, chunk table, scatter
// (needs pass 1 only, so it can overlap the OPERATION stage)
static int bucket_prepare(xs_ctx* ctx, const EventView& v, const int64_t* lo, int tb, int corr_mode,
                          const uint64_t* extra, int64_t n_extra, int64_t nvalid, int key_bits, cudaStream_t s,
                          BkPlan* plan) {
  const int64_t n = v.ev.n;
  static const int max_bits = [] {
    const char* e = getenv("XS_BK_MAX_BITS");  // (tuning experiments)
    return e ? atoi(e) : 26;
  }();
  const BucketGeom g = bucket_geom(key_bits, bucket_bits_for(nvalid, key_bits, max_bits));
  unsigned* counts;
  int64_t *offs, *chunk;
  uint64_t* keys;
  XS_TRY(ws(ctx, W_BK_COUNTS, g.nbuckets + 1, s, &counts));
  XS_TRY(ws(ctx, W_BK_OFFS, g.nbuckets + 1, s, &offs));
  XS_TRY(ws(ctx, W_MKEY, nvalid + 1, s, &keys));
  // chunks never straddle pids when a pid spans whole buckets (tb + 4 >= shift)
  const int pid_shift = tb + 4;
  const bool pid_chunks = pid_shift >= g.shift && (key_bits > pid_shift);
  const int64_t pb_buckets = pid_chunks ? ((int64_t)1 << (pid_shift - g.shift)) : 0;
  const int64_t np_b = pid_chunks ? (g.nbuckets + pb_buckets - 1) / pb_buckets : 0;
  const int64_t n_chunks = (nvalid + BK_T - 1) / BK_T + np_b;
  XS_TRY(ws(ctx, W_BK_CSTART, 4 * n_chunks + 4, s, &chunk));
  XS_CUDA(cudaMemsetAsync(counts, 0, g.nbuckets * 4, s));
  const int64_t threads = n + (n_extra + 1) / 2;
  {
    ProfScope ps(ctx, ST_KEYGEN, s);
    XS_LAUNCH(ctx, k_bk_hist, grid_for(threads), XS_BLOCK, 0, s, v, n, lo, tb, corr_mode, extra, n_extra, g.shift,
              counts);
  }
  {
    ProfScope ps(ctx, ST_MAIN_SORT, s);
    // bucket offsets + offs[nb] = total, one pass
    XS_TRY(scan_exclusive<int64_t>(ctx, ArrayIn<unsigned>{counts}, offs, g.nbuckets, s, offs + g.nbuckets));
    if (pid_chunks) {
      int64_t *ccnt, *cpre;
      XS_TRY(ws(ctx, W_BK_CFIRST, 2 * np_b + 4, s, &ccnt));
      cpre = ccnt + np_b + 2;
      XS_LAUNCH(ctx, k_pid_chunk_counts, grid_for(np_b + 1), XS_BLOCK, 0, s, offs, (int64_t)g.nbuckets, pb_buckets,
                np_b, ccnt);
      XS_TRY(scan_exclusive<int64_t>(ctx, ArrayIn<int64_t>{ccnt}, cpre, np_b + 1, s));
      XS_LAUNCH(ctx, k_bucket_chunks_pid, grid_for(32 * n_chunks), XS_BLOCK, 0, s, offs, (int64_t)g.nbuckets,
                pb_buckets, np_b, cpre, n_chunks, chunk);
    } else {
      XS_LAUNCH(ctx, k_bucket_chunks, grid_for(32 * n_chunks), XS_BLOCK, 0, s, offs, g.nbuckets, n_chunks, chunk);
    }
    XS_LAUNCH(ctx, k_bk_scatter, grid_for(threads), XS_BLOCK, 0, s, v, n, lo, tb, corr_mode, extra, n_extra, g.shift,
              counts, offs, keys);
  }
  plan->ready = true;
  plan->g = g;
  plan->nvalid = nvalid;
  plan->n_chunks = n_chunks;
  plan->pid_chunks = pid_chunks;
  plan->keys = keys;
  plan->chunk = chunk;
  plan->tb = tb;
  plan->key_bits = key_bits;
  plan->start = v.start;
  plan->n = n;
  return XS_OK;
}

// phase 2: the fused per-chunk sort + sweep (needs the op paths)
static int bucket_sweep(xs_ctx* ctx, const EventView& v, const BkPlan& plan, int n_nodes, const GHist& hist,
                        cudaStream_t s) {
  OpsState& os = ctx->ops;
  Stats* st = (Stats*)ctx->ptr[W_STATS];
  const BucketGeom g = plan.g;
  const int64_t n_chunks = plan.n_chunks, nvalid = plan.nvalid;
  const bool pid_chunks = plan.pid_chunks;
  const int tb = plan.tb;
  uint64_t* keys = plan.keys;
  int64_t* chunk = plan.chunk;
  TileDesc<SwState>* desc;
  int *flags, *tctr;
  XS_TRY(ws(ctx, W_MSCAN_DESC, n_chunks + 1, s, &desc));
  XS_TRY(ws(ctx, W_MSCAN_FLAGS, n_chunks + 1, s, &flags));
  XS_TRY(ws(ctx, W_TILE_CTR, 4, s, &tctr));
  XS_TRY(fill_many(ctx, s, {{flags, (unsigned long long)(n_chunks + 1) * sizeof(int), 0}, {tctr, sizeof(int), 0}}));
  ProfScope ps(ctx, ST_SWEEP, s);
  if (!(ctx->attr_done & 1u)) {  // (per context: a context is bound to one device)
    XS_CUDA(cudaFuncSetAttribute(k_bk_sweep<HT_SMALL, XS_SWEEP_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(BkSmemT<HT_SMALL>)));
    XS_CUDA(cudaFuncSetAttribute(k_bk_sweep<HT_BIG, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(BkSmemT<HT_BIG>)));
    ctx->attr_done |= 1u;
  }
  // direct-indexed block table when every chunk holds one pid (the path-count
  // condition is checked in the kernel); the big hashed table for traces whose
  // cells go to the hashed global histogram (many deep paths)
  static const bool no_direct = getenv("XS_NO_DIRECT_CELLS") != nullptr;  // (A/B switch)
  const int direct_ok = !no_direct && (v.ev.n_pids <= 1 || pid_chunks) ? 1 : 0;
  const bool big_table = hist.key != nullptr;
  unsigned long long* ptrace = nullptr;
  if (getenv("XS_TRACE_SWEEP")) XS_CUDA(cudaMallocAsync(&ptrace, n_chunks * 64, s));
  if (!big_table)
    XS_LAUNCH(ctx, (k_bk_sweep<HT_SMALL, XS_SWEEP_MINB>), (int)n_chunks, BK_THREADS, sizeof(BkSmemT<HT_SMALL>), s,
              keys, nvalid, chunk, g.shift, tb, os.pidpath, os.opbase, n_nodes, hist, desc, flags, tctr, st, ptrace,
              direct_ok, os.trie.count);
  else
    XS_LAUNCH(ctx, (k_bk_sweep<HT_BIG, 2>), (int)n_chunks, BK_THREADS, sizeof(BkSmemT<HT_BIG>), s, keys, nvalid,
              chunk, g.shift, tb, os.pidpath, os.opbase, n_nodes, hist, desc, flags, tctr, st, ptrace, direct_ok,
              os.trie.count);
  if (getenv("XS_DEBUG_OVF") && !ctx->capturing) {  // developer diagnostics (eager runs only)
    long long f = 0;
    cudaMemcpyAsync(&f, &st->pad[3], 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "bk_sweep nvalid=%lld key_bits=%d bb=%d pid_chunks=%d overflow=%lld\n", (long long)nvalid,
            g.key_bits, g.bb, (int)pid_chunks, f);
  }
  if (ptrace) {  // developer timing: per-phase globaltimer stamps of every CTA
    std::vector<unsigned long long> h(n_chunks * 8);
    XS_CUDA(cudaMemcpyAsync(h.data(), ptrace, n_chunks * 64, cudaMemcpyDeviceToHost, s));
    XS_CUDA(cudaStreamSynchronize(s));
    cudaFreeAsync(ptrace, s);
    unsigned long long t0 = ~0ull, t1 = 0;
    double ph[7] = {0};
    for (int64_t c = 0; c < n_chunks; c++) {
      t0 = std::min(t0, h[c * 8]);
      t1 = std::max(t1, h[c * 8 + 7]);
      for (int i = 0; i < 7; i++) ph[i] += (double)(h[c * 8 + i + 1] - h[c * 8 + i]);
    }
    fprintf(stderr, "k_bk_sweep trace: chunks %lld span %.1f us; avg per CTA (us): tile %.2f load+pub %.2f bins %.2f "
            "rank %.2f scan+lookback %.2f walk %.2f flush+table %.2f\n", (long long)n_chunks, (t1 - t0) / 1e3,
            ph[0] / n_chunks / 1e3, ph[1] / n_chunks / 1e3, ph[2] / n_chunks / 1e3, ph[3] / n_chunks / 1e3,
            ph[4] / n_chunks / 1e3, ph[5] / n_chunks / 1e3, ph[6] / n_chunks / 1e3);
  }
  return XS_OK;
}

static int run_bucket_sweep(xs_ctx* ctx, const EventView& v, const int64_t* lo, int tb, int corr_mode,
                            const uint64_t* extra, int64_t n_extra, int64_t nvalid, int key_bits, int n_nodes,
                            const GHist& hist, cudaStream_t s) {
  BkPlan plan;
  XS_TRY(bucket_prepare(ctx, v, lo, tb, corr_mode, extra, n_extra, nvalid, key_bits, s, &plan));
  return bucket_sweep(ctx, v, plan, n_nodes, hist, s);
}

// INSTANT overlap, phase 1 ahead of stage_ops (concurrent branch): the plan
// is picked up by the next stage_overlap on the same events
int stage_overlap_pre(xs_ctx* ctx, const EventView& v, cudaStream_t s) {
  ctx->bk_plan.ready = false;
  const Stats& H = *ctx->h_stats;
  const int np = v.ev.n_pids;
  const int tb = bits_for((uint64_t)(H.max_span > 0 ? H.max_span : 0));
  const int pb = bits_for((uint64_t)(np > 0 ? np - 1 : 0));
  const int64_t nvalid = 2 * H.n_nonzero;
  if (ctx->force_lsd || nvalid <= 0 || pb + tb + 4 > 64) return XS_OK;
  return bucket_prepare(ctx, v, (const int64_t*)ctx->ptr[W_SPAN_LO], tb, 0, nullptr, 0, nvalid, pb + tb + 4, s,
                        &ctx->bk_plan);
}

int stage_overlap(xs_ctx* ctx, const EventView& v, int attribution, cudaStream_t s) {
  OpsState& os = ctx->ops;
  Stats* st = (Stats*)ctx->ptr[W_STATS];
  const int64_t n = v.ev.n;
  const int np = v.ev.n_pids;
  const int tb = os.tb;
  const int pb = bits_for((uint64_t)(np > 0 ? np - 1 : 0));
  if (pb + tb + 4 > 64) {
    ctx->err = "timeline too wide for 64-bit endpoint keys";
    return XS_UNSUPPORTED;
  }
  // histogram row stride: the trie's node capacity when that is small
  // (no sync), else the real node count (one sync)
  const Stats& H = *ctx->h_stats;
  int n_nodes;
  // (CORRELATION keys also carry the node bits: the trie's capacity may be
  // far above its node count after an earlier deep-path call -- use the count)
  const bool corr_wide = attribution == 1 && pb + bits_for((uint64_t)(os.trie.node_cap - 1)) + tb + 2 > 64;
  if ((int64_t)np * os.trie.node_cap * 32 <= ((int64_t)1 << 21) && !corr_wide) {
    n_nodes = os.trie.node_cap;
  } else {
    XS_LAUNCH(ctx, k_trie_count_to_stats, 1, 32, 0, s, os.trie.count, st);
    XS_TRY(fetch_stats(ctx, s));
    if (H.table_full || H.depth_overflow || H.n_bad) return XS_OK;
    n_nodes = (int)H.pad[0];
  }
  if (n_nodes < 1) n_nodes = 1;
  // dense [pid][node][32] while it is small, else a hash table sized by a
  // bound on the distinct cells: one per interval between consecutive
  // endpoints (2n), one tracked entry per pid, and in CORRELATION mode one
  // foreign cell per fixed-event endpoint interval
  const int64_t dense_n = (int64_t)np * n_nodes * 32;
  const int64_t cell_bound = 2 * H.n_nonzero + np + 64 + (attribution == 1 ? 8 * (H.n_gpu_corr + 2 * os.m + np + 1) : 0);
  GHist hist{nullptr, nullptr, 0, (unsigned long long*)&st->table_full};
  int64_t hist_n = dense_n;
  static const int dense_max_log2 = [] {  // XS_HIST_DENSE_MAX_LOG2: tests force the hashed layout
    const char* e = getenv("XS_HIST_DENSE_MAX_LOG2");
    return e ? atoi(e) : 24;
  }();
  if (dense_n > ((int64_t)1 << dense_max_log2) && (dense_n > 2 * cell_bound || dense_max_log2 < 24)) {
    int lg = 10;
    while (((int64_t)1 << lg) < cell_bound + cell_bound / 4) lg++;  // load <= 0.8 even if every interval were a cell
    hist_n = (int64_t)1 << lg;
    XS_TRY(ws(ctx, W_HIST_KEY, hist_n, s, &hist.key));
    XS_CUDA(cudaMemsetAsync(hist.key, 0xFF, hist_n * 8, s));
    hist.mask = (unsigned long long)hist_n - 1;
  }
  XS_TRY(ws(ctx, W_HIST, hist_n + 1, s, &hist.val));
  XS_CUDA(cudaMemsetAsync(hist.val, 0, (hist_n + 1) * 8, s));
  const int64_t* lo = (const int64_t*)ctx->ptr[W_SPAN_LO];

  // CORRELATION pre-pass -> own pieces + foreign cells
  int64_t n_piece_keys = 0;
  const int corr_mode = attribution == 1 && H.n_gpu_corr > 0;
  uint64_t* pieces = nullptr;
  int64_t piece_cap = 0;
  if (corr_mode) {
    ProfScope ps(ctx, ST_CORR_FX, s);
    const int nodeb = bits_for((uint64_t)(n_nodes - 1));
    if (pb + nodeb + tb + 2 > 64) {
      ctx->err = "CORRELATION keys too wide";
      return XS_UNSUPPORTED;
    }
    const int64_t n2 = 2 * os.m;
    const int64_t cap = 2 * H.n_gpu_corr + 2 * n2 + 2 * (int64_t)np + 2;
    uint64_t *fx, *fx_alt;
    unsigned long long* cnt;
    XS_TRY(ws(ctx, W_FX_KEY, cap, s, &fx));
    XS_TRY(ws(ctx, W_FX_KEY_ALT, cap, s, &fx_alt));
    XS_TRY(ws(ctx, W_FX_OWN, 4, s, &cnt));
    XS_CUDA(cudaMemsetAsync(cnt, 0, 32, s));
    XS_LAUNCH(ctx, k_fx_fixed, grid_for(n), XS_BLOCK, 0, s, v, n, lo, (const int64_t*)ctx->ptr[W_FIXED_LS], os.pk,
              os.pidpath, os.opbase, tb, nodeb, fx, cnt);
    if (n2) XS_LAUNCH(ctx, k_fx_segments, grid_for(n2), XS_BLOCK, 0, s, os.pk, n2, os.pidpath, tb, nodeb, fx, cnt);
    XS_LAUNCH(ctx, k_fx_root, grid_for(np), XS_BLOCK, 0, s, os.pk, os.opbase, np, tb, nodeb, fx, cnt);
    unsigned long long h_cnt = 0;
    XS_CUDA(cudaMemcpyAsync(&h_cnt, cnt, 8, cudaMemcpyDeviceToHost, s));
    XS_CUDA(cudaStreamSynchronize(s));
    const int64_t nfx = (int64_t)h_cnt;
    XS_TRY(sort_keys_u64(ctx, &fx, &fx_alt, nfx, pb + nodeb + tb + 2, s));
    piece_cap = 2 * nfx + 2;
    XS_TRY(ws(ctx, W_PIECE_KEY, piece_cap, s, &pieces));
    TileDesc<FS>* desc;
    int *flags, *tctr;
    const int64_t tiles = (nfx + XS_BLOCK * FX_ITEMS - 1) / (XS_BLOCK * FX_ITEMS);
    XS_TRY(ws(ctx, W_FXSCAN_DESC, tiles + 1, s, &desc));
    XS_TRY(ws(ctx, W_FXSCAN_FLAGS, tiles + 1, s, &flags));
    XS_TRY(ws(ctx, W_TILE_CTR, 4, s, &tctr));
    XS_TRY(fill_many(ctx, s, {{flags, (unsigned long long)(tiles + 1) * sizeof(int), 0}, {tctr, sizeof(int), 0},
                              {cnt + 1, 8, 0}}));
    if (tiles)
      XS_LAUNCH(ctx, k_fx_scan, (int)tiles, XS_BLOCK, 0, s, fx, nfx, tb, nodeb, n_nodes, hist, pieces, cnt + 1, desc,
                flags, tctr);
    XS_CUDA(cudaMemcpyAsync(&h_cnt, cnt + 1, 8, cudaMemcpyDeviceToHost, s));
    XS_CUDA(cudaStreamSynchronize(s));
    n_piece_keys = (int64_t)h_cnt;
  }

  // main endpoint keys
  const int key_bits = pb + tb + 4;
  const uint64_t sentinel = key_bits >= 64 ? ~0ull : ((1ull << key_bits) - 1);
  const int64_t nkeys = 2 * n + n_piece_keys;
  const int64_t nvalid_b = 2 * H.n_nonzero + n_piece_keys;
  BkPlan& pre = ctx->bk_plan;
  const bool use_pre = pre.ready && !corr_mode && pre.start == v.start && pre.n == n && pre.tb == tb &&
                       pre.key_bits == key_bits && pre.nvalid == nvalid_b;
  pre.ready = false;
  if (!ctx->force_lsd && nvalid_b > 0 && use_pre) {
    XS_TRY(bucket_sweep(ctx, v, pre, n_nodes, hist, s));
  } else if (!ctx->force_lsd && nvalid_b > 0) {
    XS_TRY(run_bucket_sweep(ctx, v, lo, tb, corr_mode, pieces, n_piece_keys, nvalid_b, key_bits, n_nodes, hist, s));
  } else {
  uint64_t *mk, *mk_alt;
  XS_TRY(ws(ctx, W_MKEY, nkeys + SW_TILE, s, &mk));
  XS_TRY(ws(ctx, W_MKEY_ALT, nkeys + SW_TILE, s, &mk_alt));
  {
    ProfScope ps(ctx, ST_KEYGEN, s);
    if (n) XS_LAUNCH(ctx, k_keygen, grid_for(n), XS_BLOCK, 0, s, v, n, lo, tb, corr_mode, sentinel, mk);
    if (n_piece_keys) XS_CUDA(cudaMemcpyAsync(mk + 2 * n, pieces, n_piece_keys * 8, cudaMemcpyDeviceToDevice, s));
  }
  {
    ProfScope ps(ctx, ST_MAIN_SORT, s);
    XS_TRY(sort_keys_u64(ctx, &mk, &mk_alt, nkeys, key_bits, s));
  }
  const int64_t nvalid = 2 * H.n_nonzero + n_piece_keys;
  if (nvalid > 0) {
    const int64_t tiles = (nvalid + SW_TILE - 1) / SW_TILE;
    TileDesc<Cnt>* desc;
    int *flags, *tctr;
    XS_TRY(ws(ctx, W_MSCAN_DESC, tiles + 1, s, &desc));
    XS_TRY(ws(ctx, W_MSCAN_FLAGS, tiles + 1, s, &flags));
    XS_TRY(ws(ctx, W_TILE_CTR, 4, s, &tctr));
    XS_TRY(fill_many(ctx, s, {{flags, (unsigned long long)(tiles + 1) * sizeof(int), 0}, {tctr, sizeof(int), 0}}));
    ProfScope ps(ctx, ST_SWEEP, s);
    XS_LAUNCH(ctx, k_sweep, (int)tiles, XS_BLOCK, 0, s, mk, nvalid, tb, os.pidpath, os.opbase, n_nodes, hist, desc,
              flags, tctr);
  }
  }  // LSD fallback
  // compact
  int *cp, *cn, *cm;
  int64_t *cns, *tracked;
  unsigned long long* ccount = (unsigned long long*)&st->pad[4];  // read at the caller's final fetch
  const int64_t cells_cap = hist_n + 1;
  XS_TRY(ws(ctx, W_CELL_PID, cells_cap, s, &cp));
  XS_TRY(ws(ctx, W_CELL_NODE, cells_cap, s, &cn));
  XS_TRY(ws(ctx, W_CELL_MASK, cells_cap, s, &cm));
  XS_TRY(ws(ctx, W_CELL_NS, cells_cap, s, &cns));
  XS_TRY(ws(ctx, W_TRACKED, np + 1, s, &tracked));
  XS_TRY(fill_many(ctx, s, {{tracked, (unsigned long long)(np + 1) * 8, 0}, {ccount, 8, 0}}));
  ProfScope ps_compact(ctx, ST_COMPACT, s);
  if (hist_n)
    XS_LAUNCH(ctx, k_compact_cells, grid_for(hist_n), XS_BLOCK, 0, s, hist, hist_n, n_nodes, cp, cn, cm, cns, tracked,
              ccount);
  XS_LAUNCH(ctx, k_trie_count_to_stats, 1, 32, 0, s, os.trie.count, st);
  ctx->res_pids = np;
  return XS_OK;  // cells count (pad[4]) and trie size (pad[0]) arrive with the caller's fetch
}

}  // namespace xs
