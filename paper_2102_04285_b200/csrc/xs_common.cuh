// xs_common.cuh -- shared device helpers for the xstrace-b200 kernels (sm_100a).
//
// Everything here is integer-only: the path is HBM/latency bound (sorts,
// scans, reductions), there is nothing to contract, so no tensor cores.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cuda/atomic>

#include "../../include/xstrace_b200.h"

#define XS_BLOCK 256

namespace xs {

constexpr int64_t kNegInf = INT64_MIN / 4;  // -inf for (max,+) scans; survives + of any real ns

__host__ __device__ inline int bits_for(uint64_t v) {  // bits needed to hold values 0..v
#ifdef __CUDA_ARCH__
  return 64 - __clzll((long long)v);
#else
  return v ? 64 - __builtin_clzll(v) : 0;
#endif
}

__device__ __forceinline__ int64_t ld_cg(const int64_t* p) { return __ldcg(reinterpret_cast<const long long*>(p)); }

// ---------------------------------------------------------------------------
// Decoupled look-back tile prefix (single-pass scans).
//
// Each tile publishes its aggregate (flag 1) and, once known, its inclusive
// prefix (flag 2).  Tiles take ids from an atomic counter in launch order, so
// a tile only ever waits on tiles that are already resident: forward progress
// holds without grid sync.  Op may be non-commutative (segmented scans): the
// walk prepends older aggregates.
// ---------------------------------------------------------------------------
template <class T>
struct TileDesc {
  T agg;
  T incl;
};

__device__ __forceinline__ int flag_load(int* f) {
  cuda::atomic_ref<int, cuda::thread_scope_device> r(*f);
  return r.load(cuda::memory_order_acquire);
}
__device__ __forceinline__ void flag_store(int* f, int v) {
  cuda::atomic_ref<int, cuda::thread_scope_device> r(*f);
  r.store(v, cuda::memory_order_release);
}

template <class T>
__device__ __forceinline__ T ld_volatile_T(const T* p) {
  T out;
  const volatile int* src = reinterpret_cast<const volatile int*>(p);
  int* dst = reinterpret_cast<int*>(&out);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); i++) dst[i] = src[i];
  return out;
}

template <class T>
__device__ __forceinline__ void st_volatile_T(T* p, const T& v) {
  volatile int* dst = reinterpret_cast<volatile int*>(p);
  const int* src = reinterpret_cast<const int*>(&v);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); i++) dst[i] = src[i];
}

// shuffle any 4-byte-multiple POD
template <class T>
__device__ __forceinline__ T shfl_up_T(const T& v, int d) {
  T out;
  const int* s = reinterpret_cast<const int*>(&v);
  int* o = reinterpret_cast<int*>(&out);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); i++) o[i] = __shfl_up_sync(0xffffffffu, s[i], d);
  return out;
}
template <class T>
__device__ __forceinline__ T shfl_down_T(const T& v, int d) {
  T out;
  const int* s = reinterpret_cast<const int*>(&v);
  int* o = reinterpret_cast<int*>(&out);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); i++) o[i] = __shfl_down_sync(0xffffffffu, s[i], d);
  return out;
}
template <class T>
__device__ __forceinline__ T shfl_idx_T(const T& v, int src) {
  T out;
  const int* s = reinterpret_cast<const int*>(&v);
  int* o = reinterpret_cast<int*>(&out);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); i++) o[i] = __shfl_sync(0xffffffffu, s[i], src);
  return out;
}

// Warp-parallel look-back (called by all 32 lanes of warp 0).  Lane k looks
// at tile (pred - k); the window stops at the nearest inclusive prefix and the
// aggregates in between are folded oldest-first (op may be non-commutative).
template <class T, class Op>
__device__ T lookback_warp(int tile, const T& agg, TileDesc<T>* desc, int* flags, Op op, const T& identity) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) {
      st_volatile_T(&desc[0].incl, agg);
      __threadfence();
      flag_store(&flags[0], 2);
    }
    return identity;
  }
  if (lane == 0) {
    st_volatile_T(&desc[tile].agg, agg);
    __threadfence();
    flag_store(&flags[tile], 1);
  }
  T excl = identity;
  int pred = tile - 1;
  while (true) {
    const int idx = pred - lane;
    int f = 2;
    if (idx >= 0) {
      int spins = 0;
      while ((f = flag_load(&flags[idx])) == 0) {
        if (++spins > 32) __nanosleep(20);
      }
    }
    const unsigned m2 = __ballot_sync(0xffffffffu, f == 2);
    const int stop = m2 ? (__ffs(m2) - 1) : 32;
    T v = identity;
    if (idx >= 0 && lane <= stop) v = (lane == stop) ? ld_volatile_T(&desc[idx].incl) : ld_volatile_T(&desc[idx].agg);
    // ordered reduction: result = v[31] . v[30] . ... . v[0]  (older on the left)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T other = shfl_down_T(v, o);
      if ((lane & (2 * o - 1)) == 0) v = op(other, v);
    }
    v = shfl_idx_T(v, 0);
    excl = op(v, excl);
    if (m2) break;
    pred -= 32;
  }
  if (lane == 0) {
    T incl = op(excl, agg);
    st_volatile_T(&desc[tile].incl, incl);
    __threadfence();
    flag_store(&flags[tile], 2);
  }
  return excl;
}

// Split look-back for tiles whose aggregate is known before their own
// per-thread prefixes (order-independent aggregates): publish early, walk
// later.  Both are called by lane(s) of warp 0 only.
template <class T>
__device__ __forceinline__ void tile_publish_agg(int tile, const T& agg, TileDesc<T>* desc, int* flags) {
  if (tile == 0) {
    st_volatile_T(&desc[0].incl, agg);
    __threadfence();
    flag_store(&flags[0], 2);
  } else {
    st_volatile_T(&desc[tile].agg, agg);
    __threadfence();
    flag_store(&flags[tile], 1);
  }
}

template <class T, class Op>
__device__ T tile_lookback_published(int tile, const T& agg, TileDesc<T>* desc, int* flags, Op op,
                                     const T& identity) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) return identity;
  T excl = identity;
  int pred = tile - 1;
  while (true) {
    const int idx = pred - lane;
    int f = 2;
    if (idx >= 0) {
      int spins = 0;
      while ((f = flag_load(&flags[idx])) == 0) {
        if (++spins > 32) __nanosleep(20);
      }
    }
    const unsigned m2 = __ballot_sync(0xffffffffu, f == 2);
    const int stop = m2 ? (__ffs(m2) - 1) : 32;
    T v = identity;
    if (idx >= 0 && lane <= stop) v = (lane == stop) ? ld_volatile_T(&desc[idx].incl) : ld_volatile_T(&desc[idx].agg);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T other = shfl_down_T(v, o);
      if ((lane & (2 * o - 1)) == 0) v = op(other, v);
    }
    v = shfl_idx_T(v, 0);
    excl = op(v, excl);
    if (m2) break;
    pred -= 32;
  }
  if (lane == 0) {
    T incl = op(excl, agg);
    st_volatile_T(&desc[tile].incl, incl);
    __threadfence();
    flag_store(&flags[tile], 2);
  }
  return excl;
}

// Block-wide exclusive scan with warp shuffles (2 barriers).
template <class T, class Op>
__device__ T block_exclusive_fast(T v, Op op, const T& identity, T* s_warp /*[32]*/, T* agg_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = XS_BLOCK / 32;
  T incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T other = shfl_up_T(incl, o);
    if (lane >= o) incl = op(other, incl);
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T w = lane < NW ? s_warp[lane] : identity;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      T other = shfl_up_T(w, o);
      if (lane >= o) w = op(other, w);
    }
    if (lane < NW) s_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  T warp_pre = warp ? s_warp[warp - 1] : identity;
  *agg_out = s_warp[NW - 1];
  T excl_in_warp = shfl_up_T(incl, 1);
  if (lane == 0) excl_in_warp = identity;
  return op(warp_pre, excl_in_warp);
}

// Called by thread 0 only.  Returns the exclusive prefix of `tile`.
template <class T, class Op>
__device__ T lookback(int tile, const T& agg, TileDesc<T>* desc, int* flags, Op op, const T& identity) {
  if (tile == 0) {
    st_volatile_T(&desc[0].incl, agg);
    __threadfence();
    flag_store(&flags[0], 2);
    return identity;
  }
  st_volatile_T(&desc[tile].agg, agg);
  __threadfence();
  flag_store(&flags[tile], 1);
  T excl = identity;
  int pred = tile - 1;
  while (true) {
    int f;
    int spins = 0;
    while ((f = flag_load(&flags[pred])) == 0) {
      if (++spins > 64) __nanosleep(32);
    }
    if (f == 2) {
      T v = ld_volatile_T(&desc[pred].incl);
      excl = op(v, excl);
      break;
    }
    T v = ld_volatile_T(&desc[pred].agg);
    excl = op(v, excl);
    pred--;
  }
  T incl = op(excl, agg);
  st_volatile_T(&desc[tile].incl, incl);
  __threadfence();
  flag_store(&flags[tile], 2);
  return excl;
}

// Block-wide exclusive scan over XS_BLOCK thread values (shared-memory
// Hillis-Steele; T may be any POD).  Returns the exclusive value, writes the
// block aggregate to *agg_out for every thread.
template <class T, class Op>
__device__ T block_exclusive(T v, Op op, const T& identity, T* s, T* agg_out) {
  const int t = threadIdx.x;
  s[t] = v;
  __syncthreads();
#pragma unroll 1
  for (int off = 1; off < XS_BLOCK; off <<= 1) {
    T o = identity;
    if (t >= off) o = s[t - off];
    __syncthreads();
    if (t >= off) s[t] = op(o, s[t]);
    __syncthreads();
  }
  T excl = t ? s[t - 1] : identity;
  *agg_out = s[XS_BLOCK - 1];
  __syncthreads();
  return excl;
}

// Full single-pass tile prefix: block scan + look-back.  Every thread gets
// the exclusive prefix of its own value across the whole grid.
template <class T, class Op>
__device__ T grid_exclusive(T v, Op op, const T& identity, int tile, TileDesc<T>* desc, int* flags) {
  __shared__ __align__(16) unsigned char s_raw[32 * sizeof(T)];
  __shared__ __align__(16) unsigned char s_pref_raw[sizeof(T)];
  T* s = reinterpret_cast<T*>(s_raw);
  T* s_pref = reinterpret_cast<T*>(s_pref_raw);
  T agg;
  T excl = block_exclusive_fast(v, op, identity, s, &agg);
  if (threadIdx.x < 32) {
    T pre = lookback_warp(tile, agg, desc, flags, op, identity);
    if (threadIdx.x == 0) *s_pref = pre;
  }
  __syncthreads();
  T pre = *s_pref;
  __syncthreads();
  return op(pre, excl);
}

// Warp-aggregated atomicAdd on one counter (all 32 lanes must call; lanes
// with nothing to write pass k = 0).  Returns this lane's first slot.
__device__ __forceinline__ unsigned long long warp_reserve(unsigned long long* counter, unsigned k) {
  const int lane = threadIdx.x & 31;
  unsigned x = k;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  unsigned long long base = 0;
  if (lane == 31 && x) base = atomicAdd(counter, (unsigned long long)x);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + (x - k);
}

// Block-aggregated reservation: ONE atomicAdd per block on the counter (a
// per-warp atomic on one address serialises at the L2: ~1M of them cost
// ~0.9 ms for 30M events).  All threads of the block must call.
__device__ __forceinline__ unsigned long long block_reserve(unsigned long long* counter, unsigned k) {
  constexpr int NW = XS_BLOCK / 32;
  __shared__ unsigned s_w[NW];
  __shared__ unsigned long long s_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = k;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned acc = 0;
    for (int w = 0; w < NW; w++) {
      const unsigned t = s_w[w];
      s_w[w] = acc;
      acc += t;
    }
    s_base = acc ? atomicAdd(counter, (unsigned long long)acc) : 0ull;
  }
  __syncthreads();
  return s_base + s_w[warp] + (x - k);
}

// Keyed block reduction for per-pid totals: every thread passes its running
// (key, v[NV]) (key < 0 = nothing).  Warps that agree on one key reduce with
// shuffles and thread 0 merges equal keys across warps, so a block emits one
// update per distinct key instead of one per thread.  All threads must call.
template <int NV, class Emit>
__device__ __forceinline__ void block_keyed_flush(int key, long long (&v)[NV], Emit emit) {
  constexpr int NW = XS_BLOCK / 32;
  __shared__ int s_key[NW];
  __shared__ long long s_v[NW][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k0 = __shfl_sync(0xffffffffu, key, 0);
  if (__all_sync(0xffffffffu, key == k0)) {
#pragma unroll
    for (int i = 0; i < NV; i++) {
#pragma unroll
      for (int o = 16; o; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
    }
    if (lane == 0) {
      s_key[warp] = k0;
#pragma unroll
      for (int i = 0; i < NV; i++) s_v[warp][i] = v[i];
    }
  } else {
    if (key >= 0) emit(key, v);
    if (lane == 0) s_key[warp] = -1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int ck = -1;
    long long acc[NV];
    for (int w = 0; w < NW; w++) {
      if (s_key[w] < 0) continue;
      if (s_key[w] != ck) {
        if (ck >= 0) emit(ck, acc);
        ck = s_key[w];
#pragma unroll
        for (int i = 0; i < NV; i++) acc[i] = 0;
      }
#pragma unroll
      for (int i = 0; i < NV; i++) acc[i] += s_v[w][i];
    }
    if (ck >= 0) emit(ck, acc);
  }
  __syncthreads();
}

// Sum `v` over the warp for lanes whose key equals lane 0's key when the
// whole warp agrees (returns true and the sum on lane 0); otherwise false.
__device__ __forceinline__ bool warp_uniform_sum(int key, long long& v) {
  const int k0 = __shfl_sync(0xffffffffu, key, 0);
  if (!__all_sync(0xffffffffu, key == k0)) return false;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return true;
}

__device__ __forceinline__ int next_tile(int* counter) {
  __shared__ int s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1);
  __syncthreads();
  int t = s_tile;
  __syncthreads();
  return t;
}

// ---------------------------------------------------------------------------
// Segmented helpers
// ---------------------------------------------------------------------------
struct SegI128 {  // segmented int128 sum: head flag + value
  __int128 v;
  int head;
  int pad[3];
};
struct SegI128Op {
  __device__ SegI128 operator()(const SegI128& a, const SegI128& b) const {
    SegI128 r;
    r.head = a.head | b.head;
    r.v = b.head ? b.v : (a.v + b.v);
    r.pad[0] = r.pad[1] = r.pad[2] = 0;
    return r;
  }
};

__device__ __forceinline__ int64_t floor_div(__int128 a, int64_t d) {
  __int128 q = a / d;
  if ((a % d != 0) && ((a < 0) != (d < 0))) q -= 1;
  return (int64_t)q;
}

// int64 atomic helpers
__device__ __forceinline__ void atomic_add_i64(int64_t* p, int64_t v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}
__device__ __forceinline__ void atomic_min_i64(int64_t* p, int64_t v) {
  atomicMin(reinterpret_cast<long long*>(p), (long long)v);
}
__device__ __forceinline__ void atomic_max_i64(int64_t* p, int64_t v) {
  atomicMax(reinterpret_cast<long long*>(p), (long long)v);
}

inline int grid_for(int64_t n, int per_block = XS_BLOCK) {
  int64_t g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace xs
