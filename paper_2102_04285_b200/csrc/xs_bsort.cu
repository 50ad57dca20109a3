// xs_bsort.cu -- bucketed (key, value) sort for the pipeline's record sorts.
//
// The op-endpoint, transition-record and site sorts hold 0.1-2 M keys of
// 35-45 bits: CUB's onesweep needs 5-6 latency-bound passes for them.  Their
// keys are (group, time, code) with time spread over the trace span, so the
// bucket scheme of xs_bucket.cuh sorts them in one scatter plus one
// shared-memory pass:
//   1. histogram of key >> shift into ~2 buckets per key       [read keys]
//   2. exclusive scan -> bucket offsets, chunk table
//   3. scatter (key, value) into bucket order                   [read, write]
//   4. one CTA per chunk (<= BK_CAP records): a counting pass over local
//      bins spanning the chunk's key range, then direct comparison inside
//      each bin (a block radix sort when some bin is dense); the chunk is
//      written back in order                                     [read, write]
// Keys >= 2^key_bits (the callers' "unused slot" sentinels) go to the tail,
// after every real key, in any order.  The order among equal keys is
// unspecified: every caller breaks ties with its own total order afterwards
// (k_op_tiefix, k_trec_tiefix, k_tie_fix).  A chunk that cannot be sorted in
// shared memory raises Stats.pad[3]; the host then re-runs the call with
// CUB's radix sort (never silently wrong).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "xs_bucket.cuh"

namespace xs {


__global__ void __launch_bounds__(XS_BLOCK) k_bs_hist(const uint64_t* __restrict__ keys, int64_t n, int key_bits,
                                                      int shift, unsigned* counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t k = i < n ? keys[i] : 0;
  const bool valid = i < n && (key_bits >= 64 || (k >> key_bits) == 0);
  bucket_count(counts, (uint32_t)(k >> shift), valid);
}

__global__ void __launch_bounds__(XS_BLOCK) k_bs_scatter(const uint64_t* __restrict__ keys,
                                                         const uint32_t* __restrict__ vals, int64_t n, int key_bits,
                                                         int shift, unsigned* counts, const int64_t* offs, int64_t nb,
                                                         unsigned long long* tail, uint64_t* okeys, uint32_t* ovals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = i < n;
  const uint64_t k = in ? keys[i] : 0;
  const bool valid = in && (key_bits >= 64 || (k >> key_bits) == 0);
  const int64_t slot = bucket_slot(counts, offs, (uint32_t)(k >> shift), valid);
  if (valid) {
    okeys[slot] = k;
    if (vals) ovals[slot] = vals[i];
  } else if (in) {  // sentinel: after all real keys
    const int64_t at = offs[nb] + (int64_t)atomicAdd(tail, 1ull);
    okeys[at] = k;
    if (vals) ovals[at] = vals[i];
  }
}

// the sentinel tail [offs[nb], n) unchanged from the scatter buffer
__global__ void k_bs_tail(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t n,
                          const int64_t* total, uint64_t* okeys, uint32_t* ovals) {
  for (int64_t i = *total + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    okeys[i] = keys[i];
    if (vals) ovals[i] = vals[i];
  }
}

constexpr int BS_NBW = 4096;                     // words of local counting-sort bins per chunk
constexpr int BS_NB = 2 * BS_NBW, BS_LOG_NB = 13;  // 16-bit bins (a count or start is <= BK_CAP)
constexpr int BS_BIN_BIG = 256;                // a bin holding more records sends the chunk to the block radix sort

struct BsSmem {
  uint64_t sk[BK_CAP];  // keys relative to the chunk base, grouped by local bin; radix scratch with sv[]
  uint32_t sv[BK_CAP];
  unsigned bins[BS_NBW];  // 16-bit counts, then exclusive starts
  uint64_t wmin[BK_THREADS / 32], wmax[BK_THREADS / 32];
  int scan[32];
};

struct BsIAdd {
  __device__ int operator()(int x, int y) const { return x + y; }
};

// One CTA per chunk (a contiguous key range of <= BK_CAP records).  The
// keys stay in registers from the load to the bin scatter; sorted by one
// counting pass over BS_NB bins spanning exactly the chunk's [min key, max
// key] (the bins follow how the keys cluster), then by direct comparison
// inside each bin -- a handful of records, none when a bin holds one key
// value -- and written straight to their final slot (every write lands in the
// chunk's own window of the output).  Two shared arrays + the bins (~64 KB):
// 3 CTAs per SM.  A bin denser than BS_BIN_BIG sends the chunk to a block
// radix sort on the chunk's key bits.
__global__ void __launch_bounds__(BK_THREADS, 3) k_bs_local(const uint64_t* __restrict__ keys,
                                                           const uint32_t* __restrict__ vals,
                                                           const int64_t* __restrict__ chunk, int shift,
                                                           uint64_t* okeys, uint32_t* ovals, Stats* st) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BsSmem& S = *reinterpret_cast<BsSmem*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t c = blockIdx.x;
  const int64_t s0 = chunk[4 * c + 0];
  if (s0 < 0) return;
  const int cnt = (int)(chunk[4 * c + 1] - s0);
  const int64_t b0 = chunk[4 * c + 2], b1 = chunk[4 * c + 3];
  const uint64_t base = (uint64_t)b0 << shift;
  const int lbits = bits_for(((uint64_t)(b1 > b0 ? b1 : b0 + 1) << shift) - 1 - base);
  if (cnt > BK_CAP) {  // a bucket larger than BK_T: the host re-runs the call through CUB
    if (t == 0) atomicAdd((unsigned long long*)&st->pad[3], 1ull);
    return;
  }
  {
    int4* b4 = reinterpret_cast<int4*>(S.bins);
    for (int i = t; i < BS_NBW / 4; i += BK_THREADS) b4[i] = make_int4(0, 0, 0, 0);
  }
  uint64_t kr[BK_ITEMS];
  uint64_t kmin = ~0ull, kmax = 0;
#pragma unroll
  for (int j = 0; j < BK_ITEMS; j++) {
    const int idx = j * BK_THREADS + t;
    kr[j] = 0;
    if (idx < cnt) {
      kr[j] = keys[s0 + idx] - base;
      kmin = kr[j] < kmin ? kr[j] : kmin;
      kmax = kr[j] > kmax ? kr[j] : kmax;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, kmin, o), b = __shfl_xor_sync(0xffffffffu, kmax, o);
    kmin = a < kmin ? a : kmin;
    kmax = b > kmax ? b : kmax;
  }
  if (lane == 0) {
    S.wmin[warp] = kmin;
    S.wmax[warp] = kmax;
  }
  __syncthreads();
#pragma unroll
  for (int w = 0; w < BK_THREADS / 32; w++) {
    kmin = S.wmin[w] < kmin ? S.wmin[w] : kmin;
    kmax = S.wmax[w] > kmax ? S.wmax[w] : kmax;
  }
  const int rbits = cnt > 0 ? bits_for(kmax - kmin) : 0;
  const int s2 = rbits > BS_LOG_NB ? rbits - BS_LOG_NB : 0;
  uint32_t slot[BK_ITEMS / 2];  // two 16-bit slots per word
#pragma unroll
  for (int j = 0; j < BK_ITEMS; j++) {
    const int idx = j * BK_THREADS + t;
    uint32_t sl = 0;
    if (idx < cnt) {
      const uint32_t b = (uint32_t)((kr[j] - kmin) >> s2), h = 16 * (b & 1);
      sl = (atomicAdd(&S.bins[b >> 1], 1u << h) >> h) & 0xFFFFu;
    }
    if (j & 1) slot[j >> 1] |= sl << 16;
    else slot[j >> 1] = sl;
  }
  __syncthreads();
  bool big = false;
  {  // exclusive bin starts: 2 * WPT consecutive bins per thread + a block scan
    constexpr int WPT = BS_NBW / BK_THREADS;
    unsigned w[WPT];
    uint4* b4 = reinterpret_cast<uint4*>(S.bins + t * WPT);
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
      big |= lo > BS_BIN_BIG || hi > BS_BIN_BIG;
      w[q] = (unsigned)sum | ((unsigned)(sum + lo) << 16);
      sum += lo + hi;
    }
    int dummy;
    const int pre = block_exclusive_fast(sum, BsIAdd(), 0, S.scan, &dummy);
    const unsigned pp = (unsigned)pre | ((unsigned)pre << 16);
#pragma unroll
    for (int q = 0; q < WPT / 4; q++)
      b4[q] = make_uint4(w[4 * q] + pp, w[4 * q + 1] + pp, w[4 * q + 2] + pp, w[4 * q + 3] + pp);
  }
  big = __syncthreads_or(big) != 0;
  // values are read only now (coalesced, like the keys): they never occupy
  // registers through the bin pass
#pragma unroll
  for (int j = 0; j < BK_ITEMS; j++) {
    const int idx = j * BK_THREADS + t;
    if (idx < cnt) {
      const uint32_t b = (uint32_t)((kr[j] - kmin) >> s2);
      const int at = (int)((S.bins[b >> 1] >> (16 * (b & 1))) & 0xFFFFu) + (int)((slot[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
      S.sk[at] = kr[j];
      S.sv[at] = vals ? vals[s0 + idx] : 0u;
    }
  }
  __syncthreads();
  if (!big) {
#pragma unroll 4
    for (int j = 0; j < BK_ITEMS; j++) {
      const int i = j * BK_THREADS + t;
      if (i >= cnt) break;
      const uint64_t k = S.sk[i];
      int at = i;
      if (s2 > 0) {
        const int b = (int)((k - kmin) >> s2);
        const int bs = (int)((S.bins[b >> 1] >> (16 * (b & 1))) & 0xFFFFu);
        const int be = b + 1 < BS_NB ? (int)((S.bins[(b + 1) >> 1] >> (16 * ((b + 1) & 1))) & 0xFFFFu) : cnt;
        int r = 0;
        for (int q = bs; q < be; q++) {
          const uint64_t o = S.sk[q];
          r += (o < k) | ((o == k) & (q < i));
        }
        at = bs + r;
      }
      okeys[s0 + at] = base + k;
      if (ovals) ovals[s0 + at] = S.sv[i];
    }
    return;
  }
  // a dense bin: block radix sort of the whole chunk on lbits
  using BRS = cub::BlockRadixSort<uint64_t, BK_THREADS, BK_ITEMS, uint32_t, 4>;
  static_assert(sizeof(typename BRS::TempStorage) <= sizeof(S.sk) + sizeof(S.sv) + sizeof(S.bins), "radix scratch");
  uint64_t kk[BK_ITEMS];
  uint32_t vv[BK_ITEMS];
#pragma unroll
  for (int j = 0; j < BK_ITEMS; j++) {
    const int idx = t * BK_ITEMS + j;  // blocked
    kk[j] = idx < cnt ? S.sk[idx] : ~0ull;
    vv[j] = idx < cnt ? S.sv[idx] : 0u;
  }
  __syncthreads();
  typename BRS::TempStorage& tmp = *reinterpret_cast<typename BRS::TempStorage*>(S.sk);
  // padding (~0, blocked at the end) stays after equal real keys: the sort is stable
  BRS(tmp).Sort(kk, vv, 0, lbits < 1 ? 1 : lbits);
#pragma unroll
  for (int j = 0; j < BK_ITEMS; j++) {
    const int idx = t * BK_ITEMS + j;
    if (idx < cnt) {
      okeys[s0 + idx] = base + kk[j];
      if (ovals) ovals[s0 + idx] = vv[j];
    }
  }
}

static int bucket_sort_pairs_impl(xs_ctx* ctx, uint64_t** keys, uint64_t** keys_alt, uint32_t** vals,
                                  uint32_t** vals_alt, int64_t n, int key_bits, cudaStream_t s);

// XS_CHECK_BSORT=1 (debugging, eager only): compare against a host sort
int bucket_sort_pairs(xs_ctx* ctx, uint64_t** keys, uint64_t** keys_alt, uint32_t** vals, uint32_t** vals_alt,
                      int64_t n, int key_bits, cudaStream_t s) {
  static const bool check = getenv("XS_CHECK_BSORT") != nullptr;
  if (!check || !*vals) return bucket_sort_pairs_impl(ctx, keys, keys_alt, vals, vals_alt, n, key_bits, s);
  std::vector<uint64_t> in(n), out(n);
  std::vector<uint32_t> vin(n), vout(n);
  XS_CUDA(cudaMemcpyAsync(in.data(), *keys, n * 8, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaMemcpyAsync(vin.data(), *vals, n * 4, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaStreamSynchronize(s));
  XS_TRY(bucket_sort_pairs_impl(ctx, keys, keys_alt, vals, vals_alt, n, key_bits, s));
  XS_CUDA(cudaMemcpyAsync(out.data(), *keys, n * 8, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaMemcpyAsync(vout.data(), *vals, n * 4, cudaMemcpyDeviceToHost, s));
  XS_CUDA(cudaStreamSynchronize(s));
  {  // same (key, value) multiset?
    std::vector<std::pair<uint64_t, uint32_t>> a(n), b(n);
    for (int64_t i = 0; i < n; i++) a[i] = {in[i], vin[i]}, b[i] = {out[i], vout[i]};
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    fprintf(stderr, "bsort pairs %s\n", a == b ? "same" : "DIFFER");
  }
  const uint64_t lim = key_bits >= 64 ? ~0ull : (1ull << key_bits);
  std::vector<uint64_t> ref(in);
  std::stable_sort(ref.begin(), ref.end(), [&](uint64_t a, uint64_t b) {
    const bool va = a < lim, vb = b < lim;
    if (va != vb) return va;
    return va && a < b;
  });
  int64_t bad = -1, nsent = 0;
  for (int64_t i = 0; i < n; i++) {
    if (ref[i] >= lim) nsent++;
    if (bad < 0 && ref[i] < lim && ref[i] != out[i]) bad = i;
  }
  fprintf(stderr, "bsort check n=%lld bits=%d sentinels=%lld first_mismatch=%lld\n", (long long)n, key_bits,
          (long long)nsent, (long long)bad);
  if (bad >= 0)
    fprintf(stderr, "  ref %llx got %llx\n", (unsigned long long)ref[bad], (unsigned long long)out[bad]);
  return XS_OK;
}

static int bucket_sort_pairs_impl(xs_ctx* ctx, uint64_t** keys, uint64_t** keys_alt, uint32_t** vals,
                                  uint32_t** vals_alt, int64_t n, int key_bits, cudaStream_t s) {
  Stats* st = (Stats*)ctx->ptr[W_STATS];
  const BucketGeom g = bucket_geom(key_bits, bucket_bits_for(n, key_bits, 24, true));
  unsigned* counts;
  int64_t *offs, *chunk;
  unsigned long long* tail;
  XS_TRY(ws(ctx, W_BS_COUNTS, g.nbuckets + 1, s, &counts));
  XS_TRY(ws(ctx, W_BS_OFFS, g.nbuckets + 1, s, &offs));
  XS_TRY(ws(ctx, W_BS_TAIL, 1, s, &tail));
  const int64_t n_chunks = (n + BK_T - 1) / BK_T;
  XS_TRY(ws(ctx, W_BS_CHUNK, 4 * n_chunks + 4, s, &chunk));
  XS_TRY(fill_many(ctx, s, {{counts, (unsigned long long)g.nbuckets * 4, 0}, {tail, 8, 0}}));
  XS_LAUNCH(ctx, k_bs_hist, grid_for(n), XS_BLOCK, 0, s, *keys, n, key_bits, g.shift, counts);
  // bucket offsets + offs[nb] = total, one pass
  XS_TRY(scan_exclusive<int64_t>(ctx, ArrayIn<unsigned>{counts}, offs, g.nbuckets, s, offs + g.nbuckets));
  XS_LAUNCH(ctx, k_bucket_chunks, grid_for(32 * n_chunks), XS_BLOCK, 0, s, offs, g.nbuckets, n_chunks, chunk);
  XS_LAUNCH(ctx, k_bs_scatter, grid_for(n), XS_BLOCK, 0, s, *keys, *vals, n, key_bits, g.shift, counts, offs,
            g.nbuckets, tail, *keys_alt, *vals_alt);
  if (!(ctx->attr_done & 2u)) {  // (per context: a context is bound to one device)
    XS_CUDA(cudaFuncSetAttribute(k_bs_local, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BsSmem)));
    ctx->attr_done |= 2u;
  }
  // chunks sort from the alt buffers back into the primary ones; the sentinel
  // tail is copied over unchanged
  XS_LAUNCH(ctx, k_bs_local, (int)n_chunks, BK_THREADS, sizeof(BsSmem), s, *keys_alt, *vals_alt, chunk, g.shift, *keys,
            *vals, st);
  XS_LAUNCH(ctx, k_bs_tail, 148, XS_BLOCK, 0, s, *keys_alt, *vals_alt, n, offs + g.nbuckets, *keys, *vals);
  if (getenv("XS_DEBUG_OVF") && !ctx->capturing) {  // developer diagnostics (eager runs only)
    long long f = 0;
    cudaMemcpyAsync(&f, &st->pad[3], 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "bsort n=%lld key_bits=%d bb=%d overflow=%lld\n", (long long)n, key_bits, g.bb, f);
  }
  return XS_OK;
}

}  // namespace xs
