// xs_prims.cuh -- device-wide primitives of the pipeline (own kernels, one
// pass each with decoupled look-back; they replace the library scan / select
// launches between the stages):
//   scan_exclusive   out[i] = sum_{j<i} f(i)       (+ optional total)
//   select_indices   stable compaction of the indices i < n with pred(i)
// The input is a functor of the index, so counts, 0/1 flags and transformed
// columns scan without a materialised input array.
#pragma once
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <type_traits>

#include "xs_engine.cuh"

namespace xs {

constexpr int PS_ITEMS = 16;  // items per thread (4096 per tile)

// input functor over an array
template <class T>
struct ArrayIn {
  const T* p;
  __device__ __forceinline__ T operator()(int64_t i) const { return p[i]; }
};
// f(p[i])
template <class F, class T>
struct MapIn {
  const T* p;
  F f;
  __device__ __forceinline__ int operator()(int64_t i) const { return f(p[i]); }
};
template <class F, class T>
MapIn<F, T> map_in(const T* p, F f) { return MapIn<F, T>{p, f}; }

template <class T>
struct is_array_in : std::false_type {};
template <class T>
struct is_array_in<ArrayIn<T>> : std::true_type {};

// thread t of a tile starting at t0 reads items [t0 + t*ITEMS, +ITEMS)
// (blocked: a warp covers one contiguous 64-item-per-lane span); full tiles
// of 4-byte array inputs use 128-bit loads
template <class Out, class In>
__device__ __forceinline__ void load_blocked(const In& in, int64_t i0, int64_t end, Out (&v)[PS_ITEMS]) {
  if constexpr (is_array_in<In>::value) {
    using T = std::remove_cv_t<std::remove_pointer_t<decltype(in.p)>>;
    if constexpr (sizeof(T) == 4) {
      if (i0 + PS_ITEMS <= end && ((reinterpret_cast<uintptr_t>(in.p + i0) & 15) == 0)) {
        const uint4* q = reinterpret_cast<const uint4*>(in.p + i0);
#pragma unroll
        for (int k = 0; k < PS_ITEMS / 4; k++) {
          const uint4 w = q[k];
          v[4 * k + 0] = (Out)(T)w.x;
          v[4 * k + 1] = (Out)(T)w.y;
          v[4 * k + 2] = (Out)(T)w.z;
          v[4 * k + 3] = (Out)(T)w.w;
        }
        return;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < PS_ITEMS; j++) v[j] = i0 + j < end ? (Out)in(i0 + j) : (Out)0;
}

template <class Out>
__device__ __forceinline__ void store_blocked(Out* out, int64_t i0, int64_t end, const Out (&v)[PS_ITEMS]) {
  if constexpr (sizeof(Out) == 8) {
    if (i0 + PS_ITEMS <= end && ((reinterpret_cast<uintptr_t>(out + i0) & 15) == 0)) {
      longlong2* q = reinterpret_cast<longlong2*>(out + i0);
#pragma unroll
      for (int k = 0; k < PS_ITEMS / 2; k++) q[k] = make_longlong2((long long)v[2 * k], (long long)v[2 * k + 1]);
      return;
    }
  } else {
    if (i0 + PS_ITEMS <= end && ((reinterpret_cast<uintptr_t>(out + i0) & 15) == 0)) {
      int4* q = reinterpret_cast<int4*>(out + i0);
#pragma unroll
      for (int k = 0; k < PS_ITEMS / 4; k++)
        q[k] = make_int4((int)v[4 * k], (int)v[4 * k + 1], (int)v[4 * k + 2], (int)v[4 * k + 3]);
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < PS_ITEMS; j++)
    if (i0 + j < end) out[i0 + j] = v[j];
}


template <class Out, class In, bool kIncl>
__global__ void __launch_bounds__(XS_BLOCK) k_scan_excl(In in, Out* out, int64_t n, Out* total,
                                                       TileDesc<Out>* desc, int* flags, int* tile_ctr) {
  const int tile = next_tile(tile_ctr);
  const int64_t i0 = (int64_t)tile * XS_BLOCK * PS_ITEMS + (int64_t)threadIdx.x * PS_ITEMS;
  Out v[PS_ITEMS];
  load_blocked(in, i0, n, v);
  Out sum = 0;
#pragma unroll
  for (int j = 0; j < PS_ITEMS; j++) sum += v[j];
  struct Plus {
    __device__ Out operator()(const Out& a, const Out& b) const { return a + b; }
  };
  Out run = grid_exclusive(sum, Plus(), (Out)0, tile, desc, flags);
#pragma unroll
  for (int j = 0; j < PS_ITEMS; j++) {
    const Out x = v[j];
    v[j] = kIncl ? run + x : run;
    run += x;
  }
  store_blocked(out, i0, n, v);
  if (total && i0 < n && i0 + PS_ITEMS >= n) *total = run;  // the thread holding the last item
}

// Large inputs: reduce-then-scan over a persistent grid (RTS_GRID CTAs, each
// owning one contiguous range): range sums, one spine scan, then each CTA
// scans its range tile by tile with a running carry.  Two reads + one write,
// no inter-CTA waiting -- at memory speed, where a single-pass look-back
// over tens of thousands of small tiles is latency-bound.
constexpr int RTS_GRID = 148 * 4;
constexpr int RTS_TILE = XS_BLOCK * PS_ITEMS;
constexpr int64_t RTS_MIN_N = (int64_t)16 * RTS_TILE;  // below: one single-pass look-back kernel

template <class Out, class F>
__global__ void __launch_bounds__(XS_BLOCK) k_rts_reduce(F f, int64_t n, int64_t per, Out* sums) {
  const int64_t a = (int64_t)blockIdx.x * per, b = min(n, a + per);
  Out acc = 0;
  for (int64_t t0 = a; t0 < b; t0 += RTS_TILE) {
    Out v[PS_ITEMS];
    load_blocked(f, t0 + (int64_t)threadIdx.x * PS_ITEMS, b, v);
#pragma unroll
    for (int j = 0; j < PS_ITEMS; j++) acc += v[j];
  }
  using BR = cub::BlockReduce<Out, XS_BLOCK>;
  __shared__ typename BR::TempStorage tmp;
  const Out tot = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <class Out>
__global__ void __launch_bounds__(1024) k_rts_spine(Out* sums, int g, Out* total) {
  using BS = cub::BlockScan<Out, 1024>;
  __shared__ typename BS::TempStorage tmp;
  const Out v = threadIdx.x < g ? sums[threadIdx.x] : (Out)0;
  Out ex, agg;
  BS(tmp).ExclusiveSum(v, ex, agg);
  if (threadIdx.x < g) sums[threadIdx.x] = ex;
  if (total && threadIdx.x == 0) *total = agg;
}

template <class Out, class In, bool kIncl>
__global__ void __launch_bounds__(XS_BLOCK) k_rts_scan(In in, Out* out, int64_t n, int64_t per, const Out* sums) {
  const int64_t a = (int64_t)blockIdx.x * per, b = min(n, a + per);
  using BS = cub::BlockScan<Out, XS_BLOCK>;
  __shared__ typename BS::TempStorage tmp;
  Out carry = sums[blockIdx.x];
  for (int64_t t0 = a; t0 < b; t0 += RTS_TILE) {
    const int64_t i0 = t0 + (int64_t)threadIdx.x * PS_ITEMS;
    Out v[PS_ITEMS];
    load_blocked(in, i0, b, v);
    Out sum = 0;
#pragma unroll
    for (int j = 0; j < PS_ITEMS; j++) sum += v[j];
    Out ex, agg;
    BS(tmp).ExclusiveSum(sum, ex, agg);
    Out run = carry + ex;
#pragma unroll
    for (int j = 0; j < PS_ITEMS; j++) {
      const Out x = v[j];
      v[j] = kIncl ? run + x : run;
      run += x;
    }
    store_blocked(out, i0, b, v);
    carry += agg;
    __syncthreads();
  }
}

// exclusive prefix sum of in(0 .. n-1) into out[0 .. n-1]; *total (device)
// receives the sum when given.  bank: the caller's scratch bank (branches).
template <class Out, class In, bool kIncl = false>
int scan_exclusive(xs_ctx* ctx, In in, Out* out, int64_t n, cudaStream_t s, Out* total = nullptr) {
  if (n <= 0) {
    if (total) XS_CUDA(cudaMemsetAsync(total, 0, sizeof(Out), s));
    return XS_OK;
  }
  if (n >= RTS_MIN_N) {
    const int64_t per = ((n + RTS_GRID - 1) / RTS_GRID + RTS_TILE - 1) / RTS_TILE * RTS_TILE;  // (>= 1 tile)
    const int g = (int)((n + per - 1) / per);
    Out* sums;
    XS_TRY(ws(ctx, W_PSCAN_DESC, (size_t)RTS_GRID + 1, s, &sums));
    XS_LAUNCH(ctx, (k_rts_reduce<Out, In>), g, XS_BLOCK, 0, s, in, n, per, sums);
    XS_LAUNCH(ctx, k_rts_spine<Out>, 1, 1024, 0, s, sums, g, total);
    XS_LAUNCH(ctx, (k_rts_scan<Out, In, kIncl>), g, XS_BLOCK, 0, s, in, out, n, per, sums);
    return XS_OK;
  }
  const int64_t tiles = (n + XS_BLOCK * PS_ITEMS - 1) / (XS_BLOCK * PS_ITEMS);
  TileDesc<Out>* desc;
  int *flags, *ctr;
  XS_TRY(ws(ctx, W_PSCAN_DESC, (size_t)tiles + 1, s, &desc));
  XS_TRY(ws(ctx, W_PSCAN_FLAGS, (size_t)tiles + 1, s, &flags));
  XS_TRY(ws(ctx, W_PSCAN_CTR, 4, s, &ctr));
  XS_TRY(fill_many(ctx, s, {{flags, (unsigned long long)(tiles + 1) * sizeof(int), 0}, {ctr, sizeof(int), 0}}));
  XS_LAUNCH(ctx, (k_scan_excl<Out, In, kIncl>), (int)tiles, XS_BLOCK, 0, s, in, out, n, total, desc, flags, ctr);
  return XS_OK;
}

template <class Out, class In>
int scan_inclusive(xs_ctx* ctx, In in, Out* out, int64_t n, cudaStream_t s) {
  return scan_exclusive<Out, In, true>(ctx, in, out, n, s, nullptr);
}

// stable compaction: out[k] = the k-th index i (ascending) with pred(i); *count
// (device int) receives the number selected
template <class Pred>
__global__ void __launch_bounds__(XS_BLOCK) k_select(Pred pred, int64_t n, int* out, int* count,
                                                    TileDesc<int>* desc, int* flags, int* tile_ctr) {
  const int tile = next_tile(tile_ctr);
  const int64_t t0 = (int64_t)tile * XS_BLOCK * PS_ITEMS;
  // blocked items per thread: thread t owns [t0 + t*ITEMS, +ITEMS)
  unsigned bits = 0;
  int c = 0;
#pragma unroll
  for (int j = 0; j < PS_ITEMS; j++) {
    const int64_t i = t0 + (int64_t)threadIdx.x * PS_ITEMS + j;
    const bool f = i < n && pred(i);
    bits |= (unsigned)f << j;
    c += f;
  }
  struct Plus {
    __device__ int operator()(const int& a, const int& b) const { return a + b; }
  };
  int at = grid_exclusive(c, Plus(), 0, tile, desc, flags);
#pragma unroll
  for (int j = 0; j < PS_ITEMS; j++)
    if (bits >> j & 1u) out[at++] = (int)(t0 + (int64_t)threadIdx.x * PS_ITEMS + j);
  if (t0 + XS_BLOCK * PS_ITEMS >= n && threadIdx.x == XS_BLOCK - 1) *count = at;  // last tile
}

template <class Pred>
struct PredCount {
  Pred p;
  __device__ __forceinline__ int operator()(int64_t i) const { return p(i) ? 1 : 0; }
};

// the write phase of the reduce-then-scan select: each CTA compacts its range
// tile by tile (block scan of per-thread counts + running carry)
template <class Pred>
__global__ void __launch_bounds__(XS_BLOCK) k_rts_select(Pred pred, int64_t n, int64_t per, const int* sums,
                                                        int* out) {
  const int64_t a = (int64_t)blockIdx.x * per, b = min(n, a + per);
  using BS = cub::BlockScan<int, XS_BLOCK>;
  __shared__ typename BS::TempStorage tmp;
  int carry = sums[blockIdx.x];
  for (int64_t t0 = a; t0 < b; t0 += RTS_TILE) {
    unsigned bits = 0;
    int c = 0;
#pragma unroll
    for (int j = 0; j < PS_ITEMS; j++) {
      const int64_t i = t0 + (int64_t)threadIdx.x * PS_ITEMS + j;
      const bool f = i < b && pred(i);
      bits |= (unsigned)f << j;
      c += f;
    }
    int ex, agg;
    BS(tmp).ExclusiveSum(c, ex, agg);
    int at = carry + ex;
#pragma unroll
    for (int j = 0; j < PS_ITEMS; j++)
      if (bits >> j & 1u) out[at++] = (int)(t0 + (int64_t)threadIdx.x * PS_ITEMS + j);
    carry += agg;
    __syncthreads();
  }
}

template <class Pred>
int select_indices(xs_ctx* ctx, Pred pred, int64_t n, int* out, int* count, cudaStream_t s) {
  if (n <= 0) {
    XS_CUDA(cudaMemsetAsync(count, 0, sizeof(int), s));
    return XS_OK;
  }
  if (n >= RTS_MIN_N) {
    const int64_t per = ((n + RTS_GRID - 1) / RTS_GRID + RTS_TILE - 1) / RTS_TILE * RTS_TILE;  // (>= 1 tile)
    const int g = (int)((n + per - 1) / per);
    int* sums;
    XS_TRY(ws(ctx, W_PSCAN_DESC, (size_t)RTS_GRID + 1, s, &sums));
    XS_LAUNCH(ctx, (k_rts_reduce<int, PredCount<Pred>>), g, XS_BLOCK, 0, s, PredCount<Pred>{pred}, n, per, sums);
    XS_LAUNCH(ctx, k_rts_spine<int>, 1, 1024, 0, s, sums, g, count);
    XS_LAUNCH(ctx, k_rts_select<Pred>, g, XS_BLOCK, 0, s, pred, n, per, sums, out);
    return XS_OK;
  }
  const int64_t tiles = (n + XS_BLOCK * PS_ITEMS - 1) / (XS_BLOCK * PS_ITEMS);
  TileDesc<int>* desc;
  int *flags, *ctr;
  XS_TRY(ws(ctx, W_PSCAN_DESC, (size_t)tiles + 1, s, &desc));
  XS_TRY(ws(ctx, W_PSCAN_FLAGS, (size_t)tiles + 1, s, &flags));
  XS_TRY(ws(ctx, W_PSCAN_CTR, 4, s, &ctr));
  XS_TRY(fill_many(ctx, s, {{flags, (unsigned long long)(tiles + 1) * sizeof(int), 0}, {ctr, sizeof(int), 0}}));
  XS_LAUNCH(ctx, k_select<Pred>, (int)tiles, XS_BLOCK, 0, s, pred, n, out, count, desc, flags, ctr);
  return XS_OK;
}

}  // namespace xs
