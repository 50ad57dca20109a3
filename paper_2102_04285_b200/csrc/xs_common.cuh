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
  int b = 0;
  while (b < 64 && (v >> b) != 0) b++;
  return b;
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
  __shared__ __align__(16) unsigned char s_raw[XS_BLOCK * sizeof(T)];
  __shared__ __align__(16) unsigned char s_pref_raw[sizeof(T)];
  T* s = reinterpret_cast<T*>(s_raw);
  T* s_pref = reinterpret_cast<T*>(s_pref_raw);
  T agg;
  T excl = block_exclusive(v, op, identity, s, &agg);
  if (threadIdx.x == 0) *s_pref = lookback(tile, agg, desc, flags, op, identity);
  __syncthreads();
  T pre = *s_pref;
  __syncthreads();
  return op(pre, excl);
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
