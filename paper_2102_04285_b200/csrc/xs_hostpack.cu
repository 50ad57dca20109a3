// Host-side builder of the packed upload format (xs_packed_t, see
// include/xstrace_b200.h): the columns of a host trace, in the engine's
// dtypes, narrowed into one staging block (normally page-locked) that then
// goes to the device in ONE DMA and is widened there by xs_unpack.
//
// Two passes over the rows, each split across host threads by 256-row
// blocks: xs_pack_plan reads every column once (index maxima, the 32-bit fit
// of start-offset / dur / corr, per-thread exception counts) and fixes the
// layout; xs_pack_fill writes the block.  The bytes equal the numpy builder
// columnar._pack_layout + PackedLayout.fill (tests/test_pack.py compares them)
// with every padding byte zeroed.  This replaces the per-column host -> device
// copies of the reference's in-process Trace (model.py:78-88): the input of
// every analysis call is staged here.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <unistd.h>
#if defined(__x86_64__) || defined(_M_X64)
#include <immintrin.h>
#define XS_NT_STORES 1
#endif

#include "xstrace_b200.h"

namespace {

constexpr int64_t kRows = 256;          // rows per start base (columnar.PACK_ROWS)
constexpr uint32_t kExc = 0xFFFFFFFFu;  // slot whose value is in the exception table

enum { S_START, S_BASE, S_DUR, S_CORR, S_PID, S_TID, S_NAME, S_CATF, S_GPID, S_META, S_EROW, S_EVAL, S_ECOL };

inline bool fits32(int64_t v) { return v >= 0 && v < (int64_t)kExc; }

inline int64_t off_of(int64_t s, int64_t base) {  // s - base with int64 wrap (numpy)
  return (int64_t)((uint64_t)s - (uint64_t)base);
}

inline int index_width(int64_t hi) { return hi < (1 << 8) ? 1 : hi < (1 << 16) ? 2 : 4; }

// Copy into the staging block with non-temporal stores: the block is DMA'd
// to the device right after, and a block left dirty in the CPU caches is
// read by the DMA at ~20 GB/s instead of the link's ~55 (every line is
// snooped); streaming stores also skip the read-for-ownership of each line.
// dst is 16-byte aligned at every 256-row segment (sections are 16-aligned,
// segments start at multiples of 256 rows).
inline void nt_copy(uint8_t* dst, const void* src_v, int64_t n) {
  const uint8_t* src = (const uint8_t*)src_v;
#ifdef XS_NT_STORES
  int64_t i = 0;
  if (((uintptr_t)dst & 15) == 0) {
    for (; i + 16 <= n; i += 16)
      _mm_stream_si128((__m128i*)(dst + i), _mm_loadu_si128((const __m128i*)(src + i)));
  }
  if (i < n) memcpy(dst + i, src + i, n - i);
#else
  memcpy(dst, src, n);
#endif
}

struct Part {
  int64_t r0, r1;
  int64_t max_pid = 0, max_tid = 0, max_name = 0;
  int cat_max = 0, hc_max = 0;
  int64_t bad_s = 0, bad_d = 0, bad_c = 0;
};

int threads_for(int64_t n, int n_threads) {
  int hw = (int)std::thread::hardware_concurrency();
  int t = n_threads > 0 ? n_threads : std::max(hw, 1);
  int64_t by_size = (n + 65535) / 65536;  // >= 64K rows per thread
  t = (int)std::min<int64_t>({(int64_t)t, std::max<int64_t>(by_size, 1), (int64_t)XS_PACK_MAX_THREADS});
  return std::max(t, 1);
}

// A persistent worker pool: spawning ~15 threads per pass cost more than the
// pass itself at 1M rows.  Workers are detached and park on a condition
// variable between jobs; a forked child (no threads) starts a new pool.
class Pool {
 public:
  void run(int T, const std::function<void(int)>& f) {
    // one job at a time: concurrent callers (the pipelined analysis packs
    // from several host threads) would overwrite job_ / pending_ mid-job
    std::lock_guard<std::mutex> one(run_m_);
    std::unique_lock<std::mutex> lk(m_);
    if (owner_ != getpid()) {  // first use, or a fork: the threads are gone
      owner_ = getpid();
      nthreads_ = 0;
      gen_ = 0;
    }
    while (nthreads_ < T - 1) {
      std::thread(&Pool::worker, this, gen_).detach();
      ++nthreads_;
    }
    job_ = &f;
    ntask_ = T;
    next_ = 1;
    pending_ = T - 1;
    ++gen_;
    lk.unlock();
    cv_.notify_all();
    f(0);
    lk.lock();
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void worker(unsigned long long seen) {
    std::unique_lock<std::mutex> lk(m_);
    const pid_t me = owner_;
    for (;;) {
      cv_.wait(lk, [&] { return gen_ != seen; });
      if (owner_ != me) return;  // (a forked child's pool: not ours)
      seen = gen_;
      while (next_ < ntask_) {
        const int t = next_++;
        const std::function<void(int)>* job = job_;
        lk.unlock();
        (*job)(t);
        lk.lock();
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::mutex m_, run_m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  unsigned long long gen_ = 0;
  int ntask_ = 0, next_ = 0, pending_ = 0, nthreads_ = 0;
  pid_t owner_ = 0;
};

Pool& pool() {
  static Pool* p = new Pool();  // (never destroyed: detached workers may still park on it at exit)
  return *p;
}

template <class F>
void run_parts(int T, F&& f) {
  if (T == 1) {
    f(0);
    return;
  }
  const std::function<void(int)> fn = f;  // (Pool::run admits one pass at a time)
  pool().run(T, fn);
}

void part_range(int64_t n, int T, int t, int64_t* r0, int64_t* r1) {
  int64_t blocks = (n + kRows - 1) / kRows;
  int64_t per = (blocks + T - 1) / T;
  *r0 = std::min(n, (int64_t)t * per * kRows);
  *r1 = std::min(n, (int64_t)(t + 1) * per * kRows);
}

void scan_part(const xs_events_t* ev, Part* p) {
  const int64_t* s = ev->start;
  const int64_t* d = ev->dur;
  const int64_t* c = ev->corr;
  int64_t mp = 0, mt = 0, mn = 0, bs = 0, bd = 0, bc = 0;
  int cm = 0, hm = 0;
  for (int64_t b0 = p->r0; b0 < p->r1; b0 += kRows) {
    int64_t b1 = std::min(p->r1, b0 + kRows);
    int64_t base = s[b0];
    for (int64_t i = b0 + 1; i < b1; ++i) base = std::min(base, s[i]);
    for (int64_t i = b0; i < b1; ++i) {
      bs += !fits32(off_of(s[i], base));
      bd += !fits32(d[i]);
      bc += !fits32(c[i]);
      mp = std::max<int64_t>(mp, ev->pid[i]);
      mt = std::max<int64_t>(mt, ev->tid[i]);
      mn = std::max<int64_t>(mn, ev->name[i]);
      cm = std::max<int>(cm, ev->cat[i]);
      hm = std::max<int>(hm, ev->has_corr[i]);
    }
  }
  p->max_pid = mp, p->max_tid = mt, p->max_name = mn, p->cat_max = cm, p->hc_max = hm;
  p->bad_s = bs, p->bad_d = bd, p->bad_c = bc;
}

// rows [b0, b1) of a 64-bit column as 32-bit values (v - base), misfits as
// kExc; returns whether any row misfit
inline bool narrow32(uint32_t* dst, const int64_t* src, int64_t b0, int64_t b1, int64_t base) {
  uint32_t any = 0;
  for (int64_t i = b0; i < b1; ++i) {
    int64_t o = off_of(src[i], base);
    uint32_t ok = fits32(o);
    dst[i] = ok ? (uint32_t)o : kExc;
    any |= ok ^ 1u;
  }
  return any != 0;
}

template <class T>
inline void put_w(uint8_t* dst, const int32_t* src, int64_t b0, int64_t b1) {
  T* o = (T*)dst;
  for (int64_t i = b0; i < b1; ++i) o[i] = (T)src[i];
}

inline void put_index(uint8_t* dst, const int32_t* src, int64_t b0, int64_t b1, int w) {
  if (w == 1) put_w<uint8_t>(dst, src, b0, b1);
  else if (w == 2) put_w<uint16_t>(dst, src, b0, b1);
  else put_w<int32_t>(dst, src, b0, b1);
}

}  // namespace

extern "C" int xs_pack_plan(const xs_events_t* ev, int n_threads, xs_pack_layout_t* lay) {
  if (!ev || !lay || ev->n < 0) return XS_BAD_ARGUMENT;
  const int64_t n = ev->n;
  memset(lay, 0, sizeof(*lay));
  const int T = threads_for(n, n_threads);
  std::vector<Part> parts(T);
  for (int t = 0; t < T; ++t) part_range(n, T, t, &parts[t].r0, &parts[t].r1);
  run_parts(T, [&](int t) { scan_part(ev, &parts[t]); });
  int64_t mp = 0, mt = 0, mn = 0, bs = 0, bd = 0, bc = 0;
  int cm = 0, hm = 0;
  for (auto& p : parts) {
    mp = std::max(mp, p.max_pid), mt = std::max(mt, p.max_tid), mn = std::max(mn, p.max_name);
    cm = std::max(cm, p.cat_max), hm = std::max(hm, p.hc_max);
    bs += p.bad_s, bd += p.bad_d, bc += p.bad_c;
  }
  if (cm >= 128 || hm > 1) return XS_UNSUPPORTED;  // not losslessly packable (columnar._pack_layout)
  const int64_t n_max = n / 16;
  lay->n = n;
  lay->start_w = (n > 0 && bs <= n_max) ? 4 : 8;
  lay->dur_w = bd <= n_max ? 4 : 8;
  lay->corr_w = bc <= n_max ? 4 : 8;
  lay->pid_w = index_width(mp), lay->tid_w = index_width(mt), lay->name_w = index_width(mn);
  lay->n_threads = T;
  int64_t acc = 0;
  for (int t = 0; t < T; ++t) {
    const Part& p = parts[t];
    lay->thread_exc[t] = acc;
    acc += (lay->start_w == 4 ? p.bad_s : 0) + (lay->dur_w == 4 ? p.bad_d : 0) + (lay->corr_w == 4 ? p.bad_c : 0);
  }
  lay->n_exc = acc;
  int64_t nb[13] = {n * lay->start_w,
                    lay->start_w == 4 ? (n + kRows - 1) / kRows * 8 : 8,
                    n * lay->dur_w,
                    n * lay->corr_w,
                    n * lay->pid_w,
                    n * lay->tid_w,
                    n * lay->name_w,
                    n,
                    (int64_t)ev->n_groups * 4,
                    (int64_t)ev->n_pids,
                    acc * 8,
                    acc * 8,
                    acc};
  int64_t off = 0;
  for (int k = 0; k < 13; ++k) {
    lay->offset[k] = off;
    lay->nbytes[k] = nb[k];
    off += (nb[k] + 15) / 16 * 16;
  }
  lay->total = off;
  return XS_OK;
}

extern "C" int xs_pack_fill(const xs_events_t* ev, const xs_pack_layout_t* lay, void* block_v, int64_t block_bytes) {
  if (!ev || !lay || !block_v || ev->n != lay->n || block_bytes < lay->total) return XS_BAD_ARGUMENT;
  uint8_t* blk = (uint8_t*)block_v;
  const int64_t n = lay->n;
  const int T = lay->n_threads;
  uint8_t* sec[13];
  for (int k = 0; k < 13; ++k) sec[k] = blk + lay->offset[k];
  const bool s4 = lay->start_w == 4, d4 = lay->dur_w == 4, c4 = lay->corr_w == 4;
  run_parts(T, [&](int t) {
    int64_t r0, r1;
    part_range(n, T, t, &r0, &r1);
    int64_t e = lay->thread_exc[t];
    int64_t* erow = (int64_t*)sec[S_EROW];
    int64_t* eval = (int64_t*)sec[S_EVAL];
    uint8_t* ecol = sec[S_ECOL];
    const int64_t* s = ev->start;
    const int64_t* d = ev->dur;
    const int64_t* c = ev->corr;
    for (int64_t b0 = r0; b0 < r1; b0 += kRows) {
      const int64_t b1 = std::min(r1, b0 + kRows);
      // column by column over the 256-row block (branch-free, vectorisable);
      // the rare block with a misfit gets a row-ordered exception pass
      // each column segment is built in a local buffer (cache-resident),
      // then streamed into the block
      alignas(16) uint8_t seg[kRows * 8];
      const int64_t m = b1 - b0;
      bool bad = false;
      int64_t base = 0;
      if (s4) {
        base = s[b0];
        for (int64_t i = b0 + 1; i < b1; ++i) base = std::min(base, s[i]);
        ((int64_t*)sec[S_BASE])[b0 / kRows] = base;
        bad |= narrow32((uint32_t*)seg - b0, s, b0, b1, base);
        nt_copy(sec[S_START] + b0 * 4, seg, m * 4);
      } else {
        nt_copy(sec[S_START] + b0 * 8, s + b0, m * 8);
      }
      if (d4) {
        bad |= narrow32((uint32_t*)seg - b0, d, b0, b1, 0);
        nt_copy(sec[S_DUR] + b0 * 4, seg, m * 4);
      } else {
        nt_copy(sec[S_DUR] + b0 * 8, d + b0, m * 8);
      }
      if (c4) {
        bad |= narrow32((uint32_t*)seg - b0, c, b0, b1, 0);
        nt_copy(sec[S_CORR] + b0 * 4, seg, m * 4);
      } else {
        nt_copy(sec[S_CORR] + b0 * 8, c + b0, m * 8);
      }
      put_index(seg - b0 * lay->pid_w, ev->pid, b0, b1, lay->pid_w);
      nt_copy(sec[S_PID] + b0 * lay->pid_w, seg, m * lay->pid_w);
      put_index(seg - b0 * lay->tid_w, ev->tid, b0, b1, lay->tid_w);
      nt_copy(sec[S_TID] + b0 * lay->tid_w, seg, m * lay->tid_w);
      put_index(seg - b0 * lay->name_w, ev->name, b0, b1, lay->name_w);
      nt_copy(sec[S_NAME] + b0 * lay->name_w, seg, m * lay->name_w);
      for (int64_t i = b0; i < b1; ++i) seg[i - b0] = (uint8_t)(ev->cat[i] | (ev->has_corr[i] << 7));
      nt_copy(sec[S_CATF] + b0, seg, m);
      if (!bad) continue;
      for (int64_t i = b0; i < b1; ++i) {  // exceptions: row order, then column 0 / 1 / 2
        if (s4 && !fits32(off_of(s[i], base))) erow[e] = i, eval[e] = s[i], ecol[e] = 0, ++e;
        if (d4 && !fits32(d[i])) erow[e] = i, eval[e] = d[i], ecol[e] = 1, ++e;
        if (c4 && !fits32(c[i])) erow[e] = i, eval[e] = c[i], ecol[e] = 2, ++e;
      }
    }
#ifdef XS_NT_STORES
    _mm_sfence();  // streaming stores visible before the caller's DMA
#endif
  });
  if (!s4) memset(sec[S_BASE], 0, 8);
  if (lay->nbytes[S_GPID]) memcpy(sec[S_GPID], ev->group_pid, lay->nbytes[S_GPID]);
  if (lay->nbytes[S_META]) memcpy(sec[S_META], ev->pid_has_meta, lay->nbytes[S_META]);
  for (int k = 0; k < 13; ++k) {  // zero the alignment padding of every section
    int64_t end = lay->offset[k] + lay->nbytes[k];
    int64_t next = k + 1 < 13 ? lay->offset[k + 1] : lay->total;
    if (next > end) memset(blk + end, 0, next - end);
  }
  if (block_bytes > lay->total) memset(blk + lay->total, 0, std::min<int64_t>(block_bytes - lay->total, 16));
  return XS_OK;
}
