// xs_ops.cu -- OPERATION machinery: ranks, nesting validation, path interning.
//
// Reference semantics:
//   rank order  = (start, -end, tid, name), stable     overlap.py:96-99
//   path at t   = dedupe(names of active ops in rank order)   _sweep_py.py:16-26
//   nesting     = per (pid, tid) no partial overlap         model.py:137-156
// Device formulation (all integer, parallel, exact):
//   1-2. open/close endpoints of the nonzero ops sorted once by
//      (group, t, close<open); the only unordered runs are endpoints at one
//      instant, which a local tie pass puts outer-first for opens and
//      inner-first for closes using the rank order (start, -end, name, index)
//      => a balanced parenthesisation in the reference's rank order.  The
//      prefix sum of +-1 is the depth; an op is properly nested iff its depth
//      after close == depth after open - 1 (equivalent to the reference stack
//      check).
//   3. parent(op) = last open at depth-1 before it (binary search in the
//      depth-sorted opens);  node(op) = trie child of node(parent) (dedupe of
//      equal adjacent names), interned in a lock-free (parent,name) table by a
//      dependency-ordered work queue (parents are always dequeued first).
//   4. the path of every op segment (the state after all op endpoints at one
//      instant of a pid) is node(innermost) when one tid carries ops, or the
//      rank-merge of every tid's chain (interned root-down) otherwise.
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "xs_engine.cuh"
#include "xs_prims.cuh"

namespace xs {

struct OpPred {
  const uint8_t* cat;
  const int64_t* dur;
  __device__ bool operator()(const int& i) const { return cat[i] == 0 && dur[i] > 0; }
};

// endpoint stream: slot m+j = open of op j, slot j = close of op j (op j =
// j-th nonzero OPERATION in event order).  Key = group | t | open.
// (pid, tid) groups are renumbered densely over the groups that carry
// operations (opg, order-preserving): the sort key then spends bits on the
// few op groups, not on every GPU stream of the trace (config 5: 16k groups,
// 256 with ops), which keeps the bucket sort's buckets fine.
__global__ void k_op_groups(const int* group_ops, int ng, int* opg, int* opg_inv) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int has = group_ops[g] > 0;
  if (has) opg_inv[opg[g]] = g;
  if (g == ng - 1) opg[ng] = opg[g] + has;  // (per-pid op-group ranges: opg[first group of p .. of p+1])
}

struct HasOps {
  __device__ int operator()(const int& c) const { return c > 0 ? 1 : 0; }
};

__global__ void k_endpoints(const int* op_ev, int64_t m, EventView v, const int64_t* lo, int tb, const int* opg,
                            int zero_sentinel, uint64_t* keys, uint32_t* vals) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  int i = op_ev[j];
  if (zero_sentinel && v.dur[i] == 0) {  // shrunk to zero length: out of every path (tail of the sort)
    keys[m + j] = ~0ull;
    keys[j] = ~0ull;
    vals[m + j] = (uint32_t)j;
    vals[j] = (uint32_t)j;
    return;
  }
  int p = v.ev.pid[i];
  uint64_t g = (uint64_t)opg[v.ev.tid[i]];
  uint64_t s = (uint64_t)(v.start[i] - lo[p]);
  uint64_t e = (uint64_t)(v.start[i] + v.dur[i] - lo[p]);
  keys[m + j] = (g << (tb + 1)) | (s << 1) | 1ull;
  vals[m + j] = (uint32_t)j;
  keys[j] = (g << (tb + 1)) | (e << 1);
  vals[j] = (uint32_t)j;
}

// Rank order inside a (pid, tid) group is (start, -end, name, index)
// (overlap.py:96-99).  After the (group, t, open) sort, only runs of equal
// keys are unordered: opens at one instant go outer-first (rank order),
// closes at one instant inner-first (reverse rank order).  Runs are tiny, so
// one thread per run insertion-sorts it.
__device__ __forceinline__ bool rank_less(const EventView& v, const int* op_ev, uint32_t a, uint32_t b) {
  const int ia = op_ev[a], ib = op_ev[b];
  const int64_t sa = v.start[ia], sb = v.start[ib];
  if (sa != sb) return sa < sb;
  const int64_t ea = sa + v.dur[ia], eb = sb + v.dur[ib];
  if (ea != eb) return ea > eb;
  const int na = v.ev.name[ia], nb = v.ev.name[ib];
  if (na != nb) return na < nb;
  return ia < ib;
}

__global__ void k_op_tiefix(const uint64_t* keys, uint32_t* vals, int64_t n2, const int* op_ev, EventView v) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n2) return;
  const uint64_t k = keys[q];
  if (k == ~0ull) return;  // sentinel tail
  if (q > 0 && keys[q - 1] == k) return;
  if (q + 1 >= n2 || keys[q + 1] != k) return;
  int64_t e = q + 1;
  while (e < n2 && keys[e] == k) e++;
  const bool open = k & 1ull;
  for (int64_t a = q + 1; a < e; a++) {
    const uint32_t x = vals[a];
    int64_t b = a - 1;
    while (b >= q) {
      const uint32_t y = vals[b];
      const bool out_of_order = open ? rank_less(v, op_ev, x, y) : rank_less(v, op_ev, y, x);
      if (!out_of_order) break;
      vals[b + 1] = y;
      b--;
    }
    vals[b + 1] = x;
  }
}

struct DepthDelta {
  __device__ int operator()(const uint64_t& k) const { return (k & 1ull) ? 1 : -1; }
};

__global__ void k_depth_scatter(const uint64_t* keys, const uint32_t* vals, const int* depth, int64_t n2,
                                int* d_open, int* pos_open, int* d_close) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n2) return;
  uint32_t r = vals[j];
  if (keys[j] == ~0ull) {  // sentinel op (zero length): consistent, never referenced
    d_open[r] = 1;
    d_close[r] = 0;
    pos_open[r] = (int)j;
  } else if (keys[j] & 1ull) {
    d_open[r] = depth[j];
    pos_open[r] = (int)j;
  } else {
    d_close[r] = depth[j];
  }
}

__global__ void k_depth_check(const int* d_open, const int* d_close, int64_t m, Stats* st) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int bad = 0, mx = 0;
  if (r < m) {
    bad = d_close[r] != d_open[r] - 1;
    mx = d_open[r];
  }
  bad = __reduce_add_sync(0xffffffffu, bad);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd((unsigned long long*)&st->n_bad, (unsigned long long)bad);
    if (mx) atomicMax(&st->max_depth, (long long)mx);
  }
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t lo, int64_t hi, uint64_t x) {
  while (lo < hi) {
    int64_t m = (lo + hi) >> 1;
    if (a[m] < x) lo = m + 1;
    else hi = m;
  }
  return lo;
}

// Parents and trie nodes in one pass over the endpoint stream, in stream
// order (a dynamic work queue, so every dependency points at an earlier,
// already-dequeued position).  For an open at j with depth d >= 2 the parent
// is the op opened at the nearest previous position whose depth is d-1: if
// j-1 is an open that is it; if j-1 closes a sibling y, skip y's subtree
// (jump to pos_open[y]-1).  After 32 hops the sibling's own parent (already
// resolved or being resolved earlier in the queue) is copied instead, so a
// wide fan-out costs O(fan-out / 32) waits.  node(o) = child(node(parent),
// name) with adjacent-name dedupe (trie_intern).
__global__ void k_parent_nodes(const uint64_t* __restrict__ sk, const uint32_t* __restrict__ sv, int64_t n2,
                               const int* __restrict__ depth, const int* __restrict__ pos_open,
                               const int* __restrict__ op_ev, const int32_t* __restrict__ name, int tb, int* parent,
                               int* node, int* pready, int* nready, int* counter, TrieView t,
                               const long long* guard_a, const long long* guard_b) {
  const int lane = threadIdx.x & 31;
  // speculative pass (xs_analyze): the op set was taken from the original
  // trace; if an op shrank to zero length the stream is not a valid nesting,
  // nothing may wait on it, and the pass's result is discarded
  if (guard_a && *guard_a != *guard_b) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n2; j += (int64_t)gridDim.x * blockDim.x) {
      if (sk[j] & 1ull) {
        parent[sv[j]] = -1;
        node[sv[j]] = 0;
      }
    }
    return;
  }
  while (true) {
    int base = 0;
    if (lane == 0) base = atomicAdd(counter, 32);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= n2) return;
    const int64_t j = base + lane;
    if (j < n2 && sk[j] == ~0ull) {  // sentinel op (zero length, speculative pass): no path
      parent[sv[j]] = -1;
      node[sv[j]] = 0;
      __threadfence();
      atomicExch(&pready[sv[j]], 1);
      atomicExch(&nready[sv[j]], 1);
    }
    bool done = j >= n2 || !(sk[j] & 1ull) || sk[j] == ~0ull;  // closes need no work
    int o = -1, p = -2, nm = 0, wait_on = -1;
    if (!done) {
      o = (int)sv[j];
      nm = name[op_ev[o]];
      const int d = depth[j];
      if (d <= 1) {
        p = -1;
      } else {
        const uint64_t g = sk[j] >> (tb + 1);
        int64_t q = j - 1;
        for (int hop = 0;; hop++) {
          if (q < 0 || (sk[q] >> (tb + 1)) != g) {  // only on invalid nesting
            p = -1;
            break;
          }
          const uint32_t y = sv[q];
          if (sk[q] & 1ull) {
            p = (int)y;
            break;
          }
          if (hop >= 32) {  // copy the sibling's parent once it is published
            wait_on = (int)y;
            break;
          }
          q = (int64_t)pos_open[y] - 1;
        }
      }
    }
    int pn = -1;  // parent's node, -1 = not yet known
    while (!__all_sync(0xffffffffu, done)) {
      if (!done) {
        if (p == -2) {
          if (((volatile int*)pready)[wait_on]) {
            __threadfence();
            p = ((volatile int*)parent)[wait_on];
          }
        }
        if (p != -2) {
          if (p >= 0 && pn < 0) {
            if (((volatile int*)nready)[p]) {
              __threadfence();
              pn = ((volatile int*)node)[p];
            }
          }
          if (p < 0 || pn >= 0) {
            parent[o] = p;
            node[o] = trie_intern(p < 0 ? 0 : pn, nm, t);
            __threadfence();
            atomicExch(&pready[o], 1);
            atomicExch(&nready[o], 1);
            done = true;
          }
        }
      }
    }
  }
}

__device__ __forceinline__ int ctx_node_at(const uint64_t* skeys, const uint32_t* svals, int64_t j, const int* parent,
                                           const int* node) {
  uint32_t r = svals[j];
  if (skeys[j] & 1ull) return node[r];
  int p = parent[r];
  return p >= 0 ? node[p] : 0;
}

// single-tid-per-pid case: pid order == group order
__global__ void k_pidpath_simple(const uint64_t* skeys, const uint32_t* svals, int64_t n2, const int* parent,
                                 const int* node, int* pidpath) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n2) return;
  pidpath[j] = ctx_node_at(skeys, svals, j, parent, node);
}

__global__ void k_pid_keys(const uint64_t* skeys, int64_t n2, const int32_t* group_pid, const int* opg_inv, int tb,
                           uint64_t* pk) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n2) return;
  uint64_t k = skeys[j];
  if (k == ~0ull) {
    pk[j] = ~0ull;
    return;
  }
  uint64_t g = (uint64_t)opg_inv[k >> (tb + 1)];
  uint64_t low = k & ((2ull << tb) - 1);
  pk[j] = ((uint64_t)group_pid[g] << (tb + 1)) | low;
}

constexpr int MAXD = 256;

// innermost op of group g active just after time tt (its chain to the root
// is the group's active stack), or -1
__device__ __forceinline__ int group_ctx(int g, const int* group_ops, const int64_t* gs_off, const uint64_t* skeys,
                                         const uint32_t* svals, const int* parent, uint64_t tt, uint64_t tmask) {
  const int cnt = group_ops[g];
  if (!cnt) return -1;
  int64_t a = gs_off[g], b = a + 2 * (int64_t)cnt;
  // last j in [a,b) with time <= tt
  int64_t lo = a, hi = b;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (((skeys[mid] >> 1) & tmask) <= tt) lo = mid + 1;
    else hi = mid;
  }
  if (lo == a) return -1;
  const int64_t j = lo - 1;
  const uint32_t r = svals[j];
  return (skeys[j] & 1ull) ? (int)r : parent[r];
}

// merge the rank-ordered chains (ops[cs[c] .. end of chain c], leaf first,
// head[c] = its root end) root-down in rank order (start, -end, group, name,
// index -- overlap.py:96-99), interning the adjacent-deduplicated name path
// (path_of, _sweep_py.py:16-26) in the trie as we go
__device__ __forceinline__ int kway_merge(const int* ops, const int* cs, int* head, int nctx, int n,
                                          const int* rank_ev, const EventView& v, TrieView t) {
  int cur = 0;
  for (int done = 0; done < n; done++) {
    int best = -1;
    int64_t bs = 0, be = 0;
    int bg = 0, bn = 0, bi = 0;
    for (int c = 0; c < nctx; c++) {
      if (head[c] < cs[c]) continue;
      const int ix = rank_ev[ops[head[c]]];
      const int64_t xs_ = v.start[ix], xe = v.start[ix] + v.dur[ix];
      const int xg = v.ev.tid[ix], xn = v.ev.name[ix];
      const bool less = best < 0 || (xs_ != bs ? xs_ < bs : xe != be ? xe > be : xg != bg ? xg < bg
                                                                  : xn != bn ? xn < bn : ix < bi);
      if (less) {
        best = c;
        bs = xs_;
        be = xe;
        bg = xg;
        bn = xn;
        bi = ix;
      }
    }
    head[best]--;
    cur = trie_intern(cur, bn, t);
  }
  return cur;
}

// general case: rank-merge of every tid's chain at each run end of the pid
// order.  Endpoints whose merged stack exceeds the register-sized arrays
// (more than 64 op tids active, or more than MAXD ops) go to an overflow
// list served by k_pidpath_deep from a global scratch of deep_cap ints per
// thread; when deep_cap is too small the need is recorded (Stats pad[7]) and
// the host re-runs the attempt with a scratch that fits -- no depth limit.
__global__ void k_pidpath_general(const uint64_t* pk, int64_t n2, int tb, const int* pid_group0, const int* opg,
                                  const int* opg_inv, const int* group_ops,
                                  const int64_t* gs_off, const uint64_t* skeys, const uint32_t* svals,
                                  const int* parent, const int* node, const int* rank_ev, EventView v,
                                  int* pidpath, TrieView t, Stats* st, int* ovf_list, int* ovf_count,
                                  long long deep_cap) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n2) return;
  if (pk[k] == ~0ull) {  // sentinel tail
    pidpath[k] = 0;
    return;
  }
  uint64_t key = pk[k] >> 1;
  if (k + 1 < n2 && (pk[k + 1] >> 1) == key) {
    pidpath[k] = 0;  // not a run end: never looked up
    return;
  }
  const uint64_t tmask = (1ull << tb) - 1;
  int p = (int)(key >> tb);
  uint64_t tt = key & tmask;
  int ctxs[64];
  int nctx = 0;
  bool over = false;
  // only the pid's op-carrying groups (dense numbering): a pid with hundreds
  // of GPU-stream tids has a handful of op tids
  const int x0 = opg[pid_group0[p]], x1 = opg[pid_group0[p + 1]];
  for (int x = x0; x < x1 && !over; x++) {
    const int o = group_ctx(opg_inv[x], group_ops, gs_off, skeys, svals, parent, tt, tmask);
    if (o < 0) continue;
    if (nctx == 64) over = true;
    else ctxs[nctx++] = o;
  }
  if (!over && nctx == 0) {
    pidpath[k] = 0;
    return;
  }
  if (!over && nctx == 1) {
    pidpath[k] = node[ctxs[0]];
    return;
  }
  int ops[MAXD];
  int cs[64], head[64];
  int n = 0;
  for (int c = 0; c < nctx && !over; c++) {
    cs[c] = n;
    for (int o = ctxs[c]; o >= 0 && !over; o = parent[o]) {
      if (n == MAXD) over = true;
      else ops[n++] = o;
    }
    head[c] = n - 1;  // root end of chain c (chain c is ops[cs[c] .. n), leaf first)
  }
  if (over) {  // needs 3 ints per active op tid + one per stacked op
    long long need = 0;
    for (int x = x0; x < x1; x++) {
      int o = group_ctx(opg_inv[x], group_ops, gs_off, skeys, svals, parent, tt, tmask);
      if (o < 0) continue;
      need += 3;
      for (; o >= 0; o = parent[o]) need++;
    }
    pidpath[k] = 0;
    if (need <= deep_cap) {
      ovf_list[atomicAdd(ovf_count, 1)] = (int)k;
    } else {
      atomicMax((unsigned long long*)&st->pad[7], (unsigned long long)need);
      atomicAdd((unsigned long long*)&st->depth_overflow, 1ull);
    }
    return;
  }
  pidpath[k] = kway_merge(ops, cs, head, nctx, n, rank_ev, v, t);
}

// the overflow endpoints of k_pidpath_general, each with deep_cap ints of
// global scratch: [ctx | cs | head] (nctx each) then the stacked ops
__global__ void k_pidpath_deep(const uint64_t* pk, int tb, const int* pid_group0, const int* opg, const int* opg_inv,
                               const int* group_ops, const int64_t* gs_off, const uint64_t* skeys,
                               const uint32_t* svals, const int* parent, const int* rank_ev, EventView v,
                               int* pidpath, TrieView t, const int* ovf_list, const int* ovf_count, int* scratch,
                               long long deep_cap) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int* mem = scratch + tid * deep_cap;
  const uint64_t tmask = (1ull << tb) - 1;
  const int total = *ovf_count;
  for (int64_t i = tid; i < total; i += stride) {
    const int64_t k = ovf_list[i];
    const uint64_t key = pk[k] >> 1;
    const int p = (int)(key >> tb);
    const uint64_t tt = key & tmask;
    const int x0 = opg[pid_group0[p]], x1 = opg[pid_group0[p + 1]];
    int nctx = 0;
    for (int x = x0; x < x1; x++)
      nctx += group_ctx(opg_inv[x], group_ops, gs_off, skeys, svals, parent, tt, tmask) >= 0;
    int* ctxs = mem;
    int* cs = mem + nctx;
    int* head = mem + 2 * nctx;
    int* ops = mem + 3 * nctx;
    int c = 0;
    for (int x = x0; x < x1; x++) {
      const int o = group_ctx(opg_inv[x], group_ops, gs_off, skeys, svals, parent, tt, tmask);
      if (o >= 0) ctxs[c++] = o;
    }
    int n = 0;
    for (c = 0; c < nctx; c++) {
      cs[c] = n;
      for (int o = ctxs[c]; o >= 0; o = parent[o]) ops[n++] = o;
      head[c] = n - 1;
    }
    pidpath[k] = kway_merge(ops, cs, head, nctx, n, rank_ev, v, t);
  }
}

__global__ void k_trie_init(uint64_t* keys, int* vals, int64_t cap, int* parent, int* name, int* count) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cap) {
    keys[i] = ~0ull;
    vals[i] = -1;
  }
  if (i == 0) {
    parent[0] = -1;
    name[0] = -1;
    *count = 1;
  }
}

__global__ void k_opbase(const int* pid_ops, int np, int64_t* opbase) {
  // tiny serial scan (np is the number of processes)
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t acc = 0;
    for (int p = 0; p < np; p++) {
      opbase[p] = acc;
      acc += 2 * (int64_t)pid_ops[p];
    }
    opbase[np] = acc;
  }
}

// exclusive offsets of 2*group_ops (one block; a serial loop over ~16k
// groups cost ~0.9 ms on config 5)
__global__ void __launch_bounds__(1024) k_gs_off(const int* group_ops, int ng, int64_t* gs_off) {
  typedef cub::BlockScan<long long, 1024> BS;
  __shared__ typename BS::TempStorage tmp;
  const int per = (ng + 1023) / 1024;
  const int a = threadIdx.x * per, b = a + per < ng ? a + per : ng;
  long long sum = 0;
  for (int g = a; g < b; g++) sum += 2LL * group_ops[g];
  long long excl;
  BS(tmp).ExclusiveSum(sum, excl);
  for (int g = a; g < b; g++) {
    gs_off[g] = excl;
    excl += 2LL * group_ops[g];
  }
  if (threadIdx.x == 1023) gs_off[ng] = excl;
}

__global__ void k_iota_u32(uint32_t* v, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
}

int trie_setup(xs_ctx* ctx, cudaStream_t s, TrieView* t) {
  int64_t cap = (int64_t)1 << ctx->trie_cap_log2;
  uint64_t* keys;
  int *vals, *parent, *name, *count;
  XS_TRY(ws(ctx, W_TRIE_KEYS, cap, s, &keys));
  XS_TRY(ws(ctx, W_TRIE_VALS, cap, s, &vals));
  XS_TRY(ws(ctx, W_TRIE_PARENT, cap, s, &parent));
  XS_TRY(ws(ctx, W_TRIE_NAME, cap, s, &name));
  XS_TRY(ws(ctx, W_TRIE_COUNT, 4, s, &count));
  XS_LAUNCH(ctx, k_trie_init, grid_for(cap), XS_BLOCK, 0, s, keys, vals, cap, parent, name, count);
  t->keys = keys;
  t->vals = vals;
  t->parent = parent;
  t->name = name;
  t->count = count;
  t->mask = (uint64_t)cap - 1;
  t->node_cap = (int)(cap / 2);
  t->st = (Stats*)ctx->ptr[W_STATS];
  return XS_OK;
}

int stage_ops(xs_ctx* ctx, const EventView& v, cudaStream_t s, bool build_paths) {
  ProfScope ps(ctx, ST_OPS, s);
  if (!ctx->skip_ops_reset) {  // retry-able flags start clear on every attempt
    Stats* stp = (Stats*)ctx->ptr[W_STATS];
    XS_TRY(fill_many(ctx, s, {{&stp->table_full, sizeof(long long), 0}, {&stp->depth_overflow, sizeof(long long), 0},
                              {&stp->pad[3], sizeof(long long), 0}, {&stp->pad[7], sizeof(long long), 0}}));
  }
  const Stats& H = *ctx->h_stats;
  const int64_t m = H.n_ops_nz;
  const int np = v.ev.n_pids, ng = v.ev.n_groups;
  OpsState& os = ctx_ops(ctx);
  os.m = m;
  os.tb = bits_for((uint64_t)(H.max_span > 0 ? H.max_span : 0));
  int64_t *lo = (int64_t*)ctx->ptr[W_SPAN_LO];
  int* pid_ops = (int*)ctx->ptr[W_PID_OPS];
  int* group_ops = (int*)ctx->ptr[W_GROUP_OPS];
  // positions in the sorted stream count only the ops that kept a nonzero
  // length: in the speculative sentinel mode those are the corrected pass 1's
  int* pid_ops_pos = ctx->spec_zero_sentinel ? (int*)ctx->ptr[W_PID_OPS_ALT] : pid_ops;
  int* group_ops_pos = ctx->spec_zero_sentinel ? (int*)ctx->ptr[W_GROUP_OPS_ALT] : group_ops;
  Stats* st = (Stats*)ctx->ptr[W_STATS];
  const int tb = os.tb;
  const int gb = bits_for((uint64_t)(ng > 0 ? ng - 1 : 0));
  const int pb = bits_for((uint64_t)(np > 0 ? np - 1 : 0));
  const int nb = bits_for((uint64_t)(v.ev.n_names > 0 ? v.ev.n_names - 1 : 0));
  int64_t* opbase;
  XS_TRY(ws(ctx, W_OPBASE, np + 1, s, &opbase));
  XS_LAUNCH(ctx, k_opbase, 1, 32, 0, s, pid_ops_pos, np, opbase);
  os.opbase = opbase;
  os.pidpath = nullptr;
  os.pk = nullptr;
  if (m == 0) {
    if (build_paths) XS_TRY(trie_setup(ctx, s, &os.trie));
    return XS_OK;
  }
  if (gb + tb + 1 > 64 || pb + tb + 1 > 64) {  // (op-group keys use <= gb bits)
    ctx->err = "timeline too wide for 64-bit endpoint keys";
    return XS_UNSUPPORTED;
  }
  // 1. compact nonzero OPERATION rows (index order)
  int* op_ev;
  XS_TRY(ws(ctx, W_OP_EV, m + 1, s, &op_ev));
  {
    int* nsel;
    XS_TRY(ws(ctx, W_SEL_COUNT, 4, s, &nsel));
    OpPred pred{v.ev.cat, ctx->spec_select_dur ? ctx->spec_select_dur : v.dur};
    XS_TRY(select_indices(ctx, pred, v.ev.n, op_ev, nsel, s));
  }
  // 2. endpoint stream per (pid, tid) group: one sort + local tie order
  uint64_t *sk, *sk_alt;
  uint32_t *sv, *sv_alt;
  XS_TRY(ws(ctx, W_SKEY, 2 * m + 2, s, &sk));
  XS_TRY(ws(ctx, W_SKEY_ALT, 2 * m + 2, s, &sk_alt));
  XS_TRY(ws(ctx, W_SVAL, 2 * m + 2, s, &sv));
  XS_TRY(ws(ctx, W_SVAL_ALT, 2 * m + 2, s, &sv_alt));
  // dense numbering of the op-carrying groups (order-preserving)
  int *opg, *opg_inv;
  const int64_t nog = H.pad[5] > 0 ? H.pad[5] : 1;
  const int gbo = bits_for((uint64_t)(nog - 1));
  XS_TRY(ws(ctx, W_OPG, ng + 1, s, &opg));
  XS_TRY(ws(ctx, W_OPG_INV, nog + 1, s, &opg_inv));
  {
    XS_TRY(scan_exclusive<int>(ctx, map_in(group_ops, HasOps()), opg, ng, s));
  }
  XS_LAUNCH(ctx, k_op_groups, grid_for(ng), XS_BLOCK, 0, s, group_ops, ng, opg, opg_inv);
  XS_LAUNCH(ctx, k_endpoints, grid_for(m), XS_BLOCK, 0, s, op_ev, m, v, lo, tb, opg, ctx->spec_zero_sentinel ? 1 : 0,
            sk, sv);
  XS_TRY(sort_pairs_u64_u32(ctx, &sk, &sk_alt, &sv, &sv_alt, 2 * m, gbo + tb + 1, s));
  XS_LAUNCH(ctx, k_op_tiefix, grid_for(2 * m), XS_BLOCK, 0, s, sk, sv, 2 * m, op_ev, v);
  const int* rank_ev = op_ev;  // op ids index every per-op array
  os.skeys = sk;
  os.svals = sv;
  os.rank_ev = rank_ev;
  // 4. depth = prefix sum of +-1
  int *depth, *d_open, *pos_open, *d_close, *parent;
  XS_TRY(ws(ctx, W_DEPTH_SCAN_DESC, 2 * m + 2, s, &depth));
  XS_TRY(ws(ctx, W_DOPEN, m + 1, s, &d_open));
  XS_TRY(ws(ctx, W_POPEN, m + 1, s, &pos_open));
  XS_TRY(ws(ctx, W_DCLOSE, m + 1, s, &d_close));
  XS_TRY(ws(ctx, W_PARENT, m + 1, s, &parent));
  {
    XS_TRY(scan_inclusive<int>(ctx, map_in((const uint64_t*)sk, DepthDelta()), depth, 2 * m, s));
  }
  XS_LAUNCH(ctx, k_depth_scatter, grid_for(2 * m), XS_BLOCK, 0, s, sk, sv, depth, 2 * m, d_open, pos_open, d_close);
  XS_LAUNCH(ctx, k_depth_check, grid_for(m), XS_BLOCK, 0, s, d_open, d_close, m, st);
  if (!build_paths) return XS_OK;  // nesting verdict is read at the caller's next sync
  return stage_ops_paths(ctx, v, s);
}

// The path half of the operation stage, from the sorted endpoint stream and
// depths the first half left in the workspace (it may run on another stream
// later, e.g. concurrently with the correction when analyze reuses the
// original trace's paths).
int stage_ops_paths(xs_ctx* ctx, const EventView& v, cudaStream_t s) {
  const Stats& H = *ctx->h_stats;  // (the original trace's pass 1)
  OpsState& os = ctx_ops(ctx);
  const int64_t m = os.m;
  if (m == 0) {
    XS_TRY(trie_setup(ctx, s, &os.trie));
    return XS_OK;
  }
  const int np = v.ev.n_pids, ng = v.ev.n_groups;
  const int tb = os.tb;
  const int pb = bits_for((uint64_t)(np > 0 ? np - 1 : 0));
  int* group_ops_pos = ctx->spec_zero_sentinel ? (int*)ctx->ptr[W_GROUP_OPS_ALT] : (int*)ctx->ptr[W_GROUP_OPS];
  Stats* st = (Stats*)ctx->ptr[W_STATS];
  uint64_t* sk = const_cast<uint64_t*>(os.skeys);
  uint32_t* sv = const_cast<uint32_t*>(os.svals);
  const int* op_ev = os.rank_ev;
  int* depth = (int*)ctx->ptr[W_DEPTH_SCAN_DESC];
  int* pos_open = (int*)ctx->ptr[W_POPEN];
  int* parent = (int*)ctx->ptr[W_PARENT];
  int* opg = (int*)ctx->ptr[W_OPG];
  int* opg_inv = (int*)ctx->ptr[W_OPG_INV];
  const int* rank_ev = op_ev;
  // 3-5. parents + node(op) in one dependency-ordered pass over the stream
  XS_TRY(trie_setup(ctx, s, &os.trie));
  int *node, *pready, *nready, *ctr;
  XS_TRY(ws(ctx, W_NODE, m + 1, s, &node));
  XS_TRY(ws(ctx, W_READY, 2 * m + 2, s, &pready));
  nready = pready + (m + 1);
  XS_TRY(ws(ctx, W_TILE_CTR, 4, s, &ctr));
  XS_TRY(fill_many(ctx, s, {{pready, (unsigned long long)(2 * m + 2) * sizeof(int), 0}, {ctr, sizeof(int), 0}}));
  {
    int blocks = (int)std::min<int64_t>((2 * m + 255) / 256, 148 * 8);
    XS_LAUNCH(ctx, k_parent_nodes, blocks, XS_BLOCK, 0, s, sk, sv, 2 * m, depth, pos_open, op_ev, v.ev.name, tb,
              parent, node, pready, nready, ctr, os.trie, ctx->spec_guard_a, ctx->spec_guard_b);
  }
  os.parent = parent;
  os.node = node;
  // 6. path of every op segment, indexed in (pid, t) order
  int* pidpath;
  XS_TRY(ws(ctx, W_PIDPATH, 2 * m + 2, s, &pidpath));
  XS_CUDA(cudaMemsetAsync(pidpath + 2 * m, 0, 2 * sizeof(int), s));  // (the sweep prefetches one past the last)
  os.pidpath = pidpath;
  uint64_t *pk, *pk_alt;
  XS_TRY(ws(ctx, W_PK, 2 * m + 2, s, &pk));
  XS_TRY(ws(ctx, W_PK_ALT, 2 * m + 2, s, &pk_alt));
  // op endpoints relabelled group -> pid (monotone, so order is kept)
  XS_LAUNCH(ctx, k_pid_keys, grid_for(2 * m), XS_BLOCK, 0, s, sk, 2 * m, v.ev.group_pid, opg_inv, tb, pk);
  if (H.multi_op_pids == 0) {
    // one op tid per pid: pid order == group order
    XS_LAUNCH(ctx, k_pidpath_simple, grid_for(2 * m), XS_BLOCK, 0, s, sk, sv, 2 * m, parent, node, pidpath);
    os.pk = pk;
  } else {
    int64_t* gs_off;
    XS_TRY(ws(ctx, W_GS_OFF, ng + 1, s, &gs_off));
    XS_LAUNCH(ctx, k_gs_off, 1, 1024, 0, s, group_ops_pos, ng, gs_off);
    XS_TRY(sort_keys_u64(ctx, &pk, &pk_alt, 2 * m, pb + tb + 1, s));
    int* ovf;  // [count | list of overflow endpoints]
    XS_TRY(ws(ctx, W_DEEP_OVF, 2 * m + 4, s, &ovf));
    XS_CUDA(cudaMemsetAsync(ovf, 0, sizeof(int), s));
    XS_LAUNCH(ctx, k_pidpath_general, grid_for(2 * m, 128), 128, 0, s, pk, 2 * m, tb, (int*)ctx->ptr[W_PID_GROUP0],
              opg, opg_inv, group_ops_pos, gs_off, sk, sv, parent, node, rank_ev, v, pidpath, os.trie, st, ovf + 1,
              ovf, ctx->deep_cap);
    if (ctx->deep_cap > 0) {  // a previous attempt overflowed: serve the deep stacks
      const int threads = (int)std::max<long long>(32, std::min<long long>(148 * 128, (1ll << 28) / ctx->deep_cap));
      int* scratch;
      XS_TRY(ws(ctx, W_DEEP_SCRATCH, (int64_t)threads * ctx->deep_cap, s, &scratch));
      XS_LAUNCH(ctx, k_pidpath_deep, (threads + 127) / 128, 128, 0, s, pk, tb, (int*)ctx->ptr[W_PID_GROUP0], opg,
                opg_inv, group_ops_pos, gs_off, sk, sv, parent, rank_ev, v, pidpath, os.trie, ovf + 1, ovf, scratch,
                ctx->deep_cap);
    }
    os.pk = pk;
  }
  return XS_OK;
}

}  // namespace xs
