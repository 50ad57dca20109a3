// xs_bucket.cuh -- bucketed sort fused with its consumer.
//
// A full LSD radix sort costs one histogram read plus P read+write passes over
// the keys, and at config-2 sizes each onesweep pass is latency-bound (see
// profiles/r01_ncu_full_summary.txt).  Consumers here only need the keys in
// order *inside* contiguous key ranges, so:
//   1. histogram the keys into 2^BB fine buckets (key >> shift)   [1 read]
//   2. exclusive scan -> bucket offsets; group consecutive buckets into
//      chunks of <= CAP keys (CAP = one CTA's shared-memory tile)
//   3. scatter keys into bucket order                              [1 read, 1 write]
//   4. one CTA per chunk: load, sort in shared memory on the few low bits that
//      differ inside the chunk, and run the consumer's scan right there with
//      decoupled look-back across chunks                          [1 read]
// A bucket larger than CAP/2 sets an overflow flag; the host re-runs that call
// through the LSD path (never silently wrong).
#pragma once
#include "xs_engine.cuh"
#include "xs_prims.cuh"

namespace xs {

constexpr int BK_THREADS = 256;
#ifndef XS_BK_ITEMS
#define XS_BK_ITEMS 16
#endif
constexpr int BK_ITEMS = XS_BK_ITEMS;
constexpr int BK_CAP = BK_THREADS * BK_ITEMS;  // keys per chunk tile
constexpr int BK_T = BK_CAP / 2;                // chunk split granule (max bucket)
constexpr int BK_RANK_MAX = 64;                 // buckets up to this size are ranked by direct comparison


inline BucketGeom bucket_geom(int key_bits, int max_bb = 20) {
  BucketGeom g;
  g.key_bits = key_bits;
  g.bb = key_bits < max_bb ? key_bits : max_bb;
  g.shift = key_bits - g.bb;
  g.nbuckets = (int64_t)1 << g.bb;
  return g;
}

// warp-aggregated histogram increment (lanes that share a bucket add once)
__device__ __forceinline__ void bucket_count(unsigned* counts, uint32_t b, bool valid) {
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const unsigned peers = __match_any_sync(act, b);
  const int lane = threadIdx.x & 31;
  if (lane == __ffs(peers) - 1) atomicAdd(&counts[b], (unsigned)__popc(peers));
}

// warp-aggregated slot reservation inside a bucket.  Counts down the
// histogram itself (slots fill the bucket from its end), so the counts are
// back to zero when the scatter finishes -- no second array, no extra memset.
__device__ __forceinline__ int64_t bucket_slot(unsigned* counts, const int64_t* offs, uint32_t b, bool valid) {
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (!valid) return -1;
  const unsigned peers = __match_any_sync(act, b);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(peers) - 1;
  const unsigned k = (unsigned)__popc(peers);
  unsigned top = 0;
  if (lane == leader) top = atomicSub(&counts[b], k);  // old value: slots [top-k, top) are ours
  top = __shfl_sync(peers, top, leader);
  return offs[b] + (top - k) + __popc(peers & ((1u << lane) - 1));
}

// buckets ~ one per key over the occupied key space (SURVEY 8d key layout)
// max_bits: the record sorts stay at 2^24 buckets (their offsets scan would
// outweigh the smaller in-chunk ranks); the endpoint sort, whose per-chunk
// rank is the sweep's hot phase, goes to 2^26 (<= 768 MB of tables)
inline int bucket_bits_for(int64_t nkeys, int key_bits, int max_bits = 24, bool record_sort = false) {
  static int adj = [] {
    const char* e = getenv("XS_BK_BITS_ADJ");  // (tuning experiments)
    return e ? atoi(e) : 1;  // ~2 buckets per key (adj 0: +2% at config 2 but config 5 overflows to LSD)
  }();
  static int adj_rec = [] {
    const char* e = getenv("XS_BK_BITS_ADJ_REC");  // (tuning experiments: record sorts)
    // ~1 record per bucket: the chunk sort adapts its own bins to the keys,
    // so fewer global buckets only shrink the offset scan (config 2 -3%)
    return e ? atoi(e) : -1;
  }();
  int b = 1;
  while (b < 62 && ((int64_t)1 << b) < nkeys) b++;
  b += record_sort ? adj_rec : adj;
  if (b < 10) b = 10;
  if (b > max_bits) b = max_bits;
  return b < key_bits ? b : key_bits;
}

// Chunk c = the buckets whose exclusive offset lies in [c*T, (c+1)*T); its
// first bucket is lower_bound(offs, c*T) when that bucket's offset is still in
// range, otherwise chunk c is empty (a bucket spanning several granules).  A
// chunk holds < 2T = CAP keys whenever no bucket exceeds T (the consumer
// flags overflow otherwise).
__device__ __forceinline__ int64_t upper_bound_i64(const int64_t* a, int64_t lo, int64_t hi, int64_t x) {
  while (lo < hi) {  // first index with a[i] > x
    int64_t m = (lo + hi) >> 1;
    if (a[m] <= x) lo = m + 1;
    else hi = m;
  }
  return lo;
}

__device__ __forceinline__ int64_t lower_bound_i64(const int64_t* a, int64_t lo, int64_t hi, int64_t x) {
  while (lo < hi) {  // first index with a[i] >= x
    int64_t m = (lo + hi) >> 1;
    if (a[m] < x) lo = m + 1;
    else hi = m;
  }
  return lo;
}

// offs[nb] = number of keys, from the device counts: the host's figure is
// only an upper bound when the pass was launched speculatively (xs_analyze)
static __global__ void k_bk_total(int64_t* offs, const unsigned* counts, int64_t nb) {
  if (threadIdx.x == 0) offs[nb] = nb ? offs[nb - 1] + counts[nb - 1] : 0;
}

// Warp-cooperative searches: 32 probes per step shrink the range 32x, so a
// search over millions of bucket offsets takes ~5 dependent loads, not ~22.
template <bool kUpper>  // kUpper: first index with a[i] > x, else a[i] >= x
__device__ __forceinline__ int64_t warp_search_i64(const int64_t* a, int64_t lo, int64_t hi, int64_t x) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t q = lo + lane * step;
    const bool in = q < hi;
    const int64_t av = in ? a[q] : 0;
    const bool pred = in && (kUpper ? av > x : av >= x);
    const unsigned bal = __ballot_sync(0xffffffffu, pred);
    if (bal == 0) {
      const unsigned inb = __ballot_sync(0xffffffffu, in);
      const int last = 31 - __clz(inb);
      lo = lo + last * step + 1;
    } else {
      const int f = __ffs(bal) - 1;
      if (f == 0) return lo;
      const int64_t nhi = lo + f * step;
      lo = lo + (f - 1) * step + 1;
      hi = nhi;
    }
  }
  const int64_t q = lo + lane;
  const bool pred = q < hi && (kUpper ? a[q] > x : a[q] >= x);
  const unsigned bal = __ballot_sync(0xffffffffu, pred);
  return bal ? lo + (__ffs(bal) - 1) : hi;
}

// 16-lane search: lanes [16h, 16h+16) of a warp search `a` together (two
// independent searches per warp run side by side).
template <bool kUpper>  // kUpper: first index with a[i] > x, else a[i] >= x
__device__ __forceinline__ int64_t half_search_i64(const int64_t* a, int64_t lo, int64_t hi, int64_t x) {
  // all 32 lanes keep calling the ballots until both halves are done
  const int hl = threadIdx.x & 15;
  const int sh = threadIdx.x & 16;
  const unsigned hm = 0xFFFFu << sh;
  while (__any_sync(0xffffffffu, hi - lo > 16)) {
    const bool act = hi - lo > 16;
    const int64_t step = act ? (hi - lo + 15) / 16 : 1;
    const int64_t q = lo + hl * step;
    const bool in = act && q < hi;
    const int64_t av = in ? a[q] : 0;
    const bool pred = in && (kUpper ? av > x : av >= x);
    const unsigned bal = (__ballot_sync(0xffffffffu, pred) & hm) >> sh;
    const unsigned inb = (__ballot_sync(0xffffffffu, in) & hm) >> sh;
    if (act) {
      if (bal == 0) {
        lo = lo + (31 - __clz(inb)) * step + 1;
      } else {
        const int f = __ffs(bal) - 1;
        if (f == 0) {
          hi = lo;  // a[lo] qualifies
        } else {
          const int64_t nhi = lo + f * step;
          lo = lo + (f - 1) * step + 1;
          hi = nhi;
        }
      }
    }
  }
  const int64_t q = lo + hl;
  const bool pred = q < hi && (kUpper ? a[q] > x : a[q] >= x);
  const unsigned bal = (__ballot_sync(0xffffffffu, pred) & hm) >> sh;
  return bal ? lo + (__ffs(bal) - 1) : hi;
}

// One warp per chunk, all chunks in parallel: key range [start, end) and
// the tight bucket range [b0, b1) (first / last nonempty bucket) so each
// consumer CTA starts with four loads instead of serial searches.
// offs has nb+1 entries (offs[nb] = total).  The two half-warps search the
// chunk's two granule boundaries at once, then its first / last buckets.
static __global__ void k_bucket_chunks(const int64_t* offs, int64_t nb, int64_t n_chunks, int64_t* chunk) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= n_chunks) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const bool h1 = lane >= 16;
  const int64_t total = offs[nb];
  // half 0: b = first bucket with offs >= c*T; half 1: bn = first with offs >= (c+1)*T
  const int64_t r = half_search_i64<false>(offs, 0, nb, (c + (h1 ? 1 : 0)) * BK_T);
  const int64_t b = __shfl_sync(0xffffffffu, r, 0), bn = __shfl_sync(0xffffffffu, r, 16);
  int64_t s = -1, e = -1, b0 = 0, b1 = 0;
  const bool live = b < nb && offs[b] < total && offs[b] / BK_T == c;  // (warp-uniform)
  if (live) {
    s = offs[b];
    e = bn < nb ? offs[bn] : total;
    // half 0: bucket holding key s; half 1: bucket holding key e-1, plus one
    // both lie in [b, bn]: offs[bn] >= e (or bn = nb, offs[nb] = total = e)
    const int64_t hi = (bn < nb ? bn : nb) + 1;
    const int64_t r2 = h1 ? half_search_i64<true>(offs, b, hi, e - 1)
                          : half_search_i64<true>(offs, b, hi, s) - 1;
    b0 = __shfl_sync(0xffffffffu, r2, 0);
    b1 = __shfl_sync(0xffffffffu, r2, 16);
  }
  if (lane == 0) {
    chunk[4 * c + 0] = s;
    chunk[4 * c + 1] = e;
    chunk[4 * c + 2] = b0;
    chunk[4 * c + 3] = b1;
  }
}

// Pid-aligned chunking for the endpoint sort (keys = pid | t | code): a chunk
// never straddles two pids, so its relative key range stays within one pid's
// timeline (the fused sweep keeps 32-bit relative keys; across a pid boundary
// the gap up to the next pid's range would not fit).  Pid p owns buckets
// [p*PB, (p+1)*PB) and gets ceil(keys_p / BK_T) chunks; cpre[p] is the
// exclusive prefix of those counts (cpre[np_b] = total chunks).
static __global__ void k_pid_chunk_counts(const int64_t* offs, int64_t nb, int64_t pb_buckets, int64_t np_b,
                                          int64_t* cnt) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p > np_b) return;
  if (p == np_b) {  // the scan's last input: cpre[np_b] becomes the total
    cnt[p] = 0;
    return;
  }
  const int64_t b0 = p * pb_buckets, b1 = (p + 1) * pb_buckets < nb ? (p + 1) * pb_buckets : nb;
  const int64_t k = offs[b1] - offs[b0];
  cnt[p] = (k + BK_T - 1) / BK_T;
}

static __global__ void k_bucket_chunks_pid(const int64_t* offs, int64_t nb, int64_t pb_buckets, int64_t np_b,
                                           const int64_t* cpre, int64_t n_chunks, int64_t* chunk) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= n_chunks) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  int64_t s = -1, e = -1, b0 = 0, b1 = 0;
  if (c < cpre[np_b]) {
    const int64_t p = warp_search_i64<true>(cpre, 0, np_b + 1, c) - 1;  // last pid with cpre[p] <= c
    const int64_t j = c - cpre[p];
    const int64_t pb0 = p * pb_buckets;
    const int64_t pb1 = (p + 1) * pb_buckets < nb ? (p + 1) * pb_buckets : nb;
    const int64_t kend = offs[pb1];
    const int64_t g0 = offs[pb0] + j * BK_T, g1 = g0 + BK_T;
    const int64_t b = warp_search_i64<false>(offs, pb0, pb1, g0);
    if (b < pb1 && offs[b] < kend && offs[b] < g1) {
      s = offs[b];
      const int64_t bn = warp_search_i64<false>(offs, b, pb1, g1);
      e = offs[bn];  // bn <= pb1 and offs[pb1] = kend
      b0 = warp_search_i64<true>(offs, b, pb1 + 1, s) - 1;   // bucket holding key s
      b1 = warp_search_i64<true>(offs, b0, pb1 + 1, e - 1);  // bucket holding key e-1, plus one
    }
  }
  if (lane == 0) {
    chunk[4 * c + 0] = s;
    chunk[4 * c + 1] = e;
    chunk[4 * c + 2] = b0;
    chunk[4 * c + 3] = b1;
  }
}

}  // namespace xs
