/*
 * xs_oracle.c -- CPU restatement of the reference hot path (TEST ORACLE).
 *
 * This file is test infrastructure: tests/, __graft_entry__.smoke() and the
 * bench's cpu_baseline / --impl reference legs load it as the *checker*.  The
 * product (paper_2102_04285_b200) never imports, links or executes it.
 *
 * It restates, sequentially and per pid exactly as the reference does:
 *   validate_trace event rules ........ pkg/src/xstrace/model.py:159-228
 *   _check_operation_nesting .......... model.py:137-156
 *   compute_overlap ................... overlap.py:106-188
 *   _op_rank_order .................... overlap.py:96-99
 *   sweep_pid / path_of ............... _sweep_py.py:16-115 (= _sweep.pyx:17-118)
 *   transition_sites .................. overlap.py:220-289
 *   collect_sites ..................... correction.py:79-112
 *   correct_trace ..................... correction.py:115-186
 *   quantize_amounts / RemovalMap ..... _timeline.py:57-67, 84-117
 *   map_events ........................ _timeline.py:120-132
 *
 * Rational amounts (fractions.Fraction in the reference) are carried exactly
 * as integers over one common denominator L (scaled by the host), with the
 * running sum in __int128 -- floor(cum) is then floor(cum_scaled / L), which
 * is the identical value.
 */
#include "xs_oracle.h"

#include <stdlib.h>
#include <string.h>

#define MAX_TS INT64_MAX

/* ------------------------------------------------------------------------ */
/* stable merge sort of int64 index arrays                                  */
/* ------------------------------------------------------------------------ */
typedef int (*cmp_fn)(int64_t a, int64_t b, const void* ctx);

static void msort_rec(int64_t* a, int64_t* tmp, int64_t n, cmp_fn cmp, const void* ctx) {
  if (n < 2) return;
  if (n <= 16) {
    for (int64_t i = 1; i < n; i++) {
      int64_t v = a[i];
      int64_t j = i - 1;
      while (j >= 0 && cmp(a[j], v, ctx) > 0) {
        a[j + 1] = a[j];
        j--;
      }
      a[j + 1] = v;
    }
    return;
  }
  int64_t m = n / 2;
  msort_rec(a, tmp, m, cmp, ctx);
  msort_rec(a + m, tmp, n - m, cmp, ctx);
  if (cmp(a[m - 1], a[m], ctx) <= 0) return;
  int64_t i = 0, j = m, k = 0;
  while (i < m && j < n) {
    if (cmp(a[j], a[i], ctx) < 0) tmp[k++] = a[j++];
    else tmp[k++] = a[i++];
  }
  while (i < m) tmp[k++] = a[i++];
  while (j < n) tmp[k++] = a[j++];
  memcpy(a, tmp, (size_t)n * sizeof(int64_t));
}

static int stable_sort(int64_t* a, int64_t n, cmp_fn cmp, const void* ctx) {
  if (n < 2) return 0;
  int64_t* tmp = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  if (!tmp) return -1;
  msort_rec(a, tmp, n, cmp, ctx);
  free(tmp);
  return 0;
}

#define CMP(x, y) (((x) > (y)) - ((x) < (y)))

/* ------------------------------------------------------------------------ */
/* int64 -> int64 open-addressing map                                        */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t cap, count;
  int64_t* keys;
  int64_t* vals;
  uint8_t* used;
} map_t;

static uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

static int map_init(map_t* m, int64_t cap) {
  int64_t c = 16;
  while (c < cap * 2) c <<= 1;
  m->cap = c;
  m->count = 0;
  m->keys = (int64_t*)malloc((size_t)c * sizeof(int64_t));
  m->vals = (int64_t*)malloc((size_t)c * sizeof(int64_t));
  m->used = (uint8_t*)calloc((size_t)c, 1);
  return (m->keys && m->vals && m->used) ? 0 : -1;
}

static void map_free(map_t* m) {
  free(m->keys);
  free(m->vals);
  free(m->used);
  memset(m, 0, sizeof(*m));
}

static int map_grow(map_t* m);

/* returns slot index; *found set when key existed */
static int64_t map_slot(map_t* m, int64_t key, int* found) {
  if ((m->count + 1) * 2 > m->cap) {
    if (map_grow(m)) return -1;
  }
  uint64_t h = mix64((uint64_t)key) & (uint64_t)(m->cap - 1);
  while (m->used[h]) {
    if (m->keys[h] == key) {
      *found = 1;
      return (int64_t)h;
    }
    h = (h + 1) & (uint64_t)(m->cap - 1);
  }
  *found = 0;
  m->used[h] = 1;
  m->keys[h] = key;
  m->vals[h] = 0;
  m->count++;
  return (int64_t)h;
}

static int map_grow(map_t* m) {
  map_t n2;
  if (map_init(&n2, m->cap)) return -1;
  for (int64_t i = 0; i < m->cap; i++) {
    if (!m->used[i]) continue;
    int f;
    int64_t s = map_slot(&n2, m->keys[i], &f);
    n2.vals[s] = m->vals[i];
  }
  map_free(m);
  *m = n2;
  return 0;
}

static int map_get(const map_t* m, int64_t key, int64_t* val) {
  if (m->cap == 0) return 0;
  uint64_t h = mix64((uint64_t)key) & (uint64_t)(m->cap - 1);
  while (m->used[h]) {
    if (m->keys[h] == key) {
      *val = m->vals[h];
      return 1;
    }
    h = (h + 1) & (uint64_t)(m->cap - 1);
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* path table (overlap.py:80-93) as a trie: tuple <-> node is a bijection    */
/* ------------------------------------------------------------------------ */
typedef struct {
  map_t index; /* (parent<<32 | name) -> node */
  int32_t n, cap;
  int32_t* parent;
  int32_t* name;
} trie_t;

static int trie_init(trie_t* t) {
  if (map_init(&t->index, 64)) return -1;
  t->cap = 64;
  t->n = 1;
  t->parent = (int32_t*)malloc(64 * sizeof(int32_t));
  t->name = (int32_t*)malloc(64 * sizeof(int32_t));
  if (!t->parent || !t->name) return -1;
  t->parent[0] = -1;
  t->name[0] = -1;
  return 0;
}

static void trie_free(trie_t* t) {
  map_free(&t->index);
  free(t->parent);
  free(t->name);
}

static int32_t trie_child(trie_t* t, int32_t parent, int32_t name) {
  int64_t key = ((int64_t)parent << 32) | (uint32_t)name;
  int found;
  int64_t s = map_slot(&t->index, key, &found);
  if (s < 0) return -1;
  if (found) return (int32_t)t->index.vals[s];
  if (t->n == t->cap) {
    t->cap *= 2;
    t->parent = (int32_t*)realloc(t->parent, (size_t)t->cap * sizeof(int32_t));
    t->name = (int32_t*)realloc(t->name, (size_t)t->cap * sizeof(int32_t));
    if (!t->parent || !t->name) return -1;
  }
  int32_t id = t->n++;
  t->parent[id] = parent;
  t->name[id] = name;
  t->index.vals[s] = id;
  return id;
}

/* path_of (_sweep_py.py:16-26): adjacent equal names collapse, then intern */
static int32_t intern_names(trie_t* t, const int32_t* names, int64_t k) {
  int32_t node = 0;
  int32_t last = -1;
  int have = 0;
  for (int64_t i = 0; i < k; i++) {
    if (have && names[i] == last) continue;
    node = trie_child(t, node, names[i]);
    if (node < 0) return -1;
    last = names[i];
    have = 1;
  }
  return node;
}

/* ------------------------------------------------------------------------ */
/* helpers                                                                   */
/* ------------------------------------------------------------------------ */
typedef struct {
  const xo_events_t* ev;
} ectx;

static inline int64_t ev_end(const xo_events_t* ev, int64_t i) {
  return (int64_t)((uint64_t)ev->start[i] + (uint64_t)ev->dur[i]);
}

/* pid grouping: stable counting sort (trace order within each pid) */
static int group_by_pid(const xo_events_t* ev, int64_t** off_out, int64_t** idx_out) {
  int64_t* off = (int64_t*)calloc((size_t)ev->n_pids + 1, sizeof(int64_t));
  int64_t* idx = (int64_t*)malloc((size_t)(ev->n ? ev->n : 1) * sizeof(int64_t));
  if (!off || !idx) return -1;
  for (int64_t i = 0; i < ev->n; i++) off[ev->pid[i] + 1]++;
  for (int32_t p = 0; p < ev->n_pids; p++) off[p + 1] += off[p];
  int64_t* cur = (int64_t*)malloc(((size_t)ev->n_pids + 1) * sizeof(int64_t));
  if (!cur) return -1;
  memcpy(cur, off, ((size_t)ev->n_pids + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < ev->n; i++) idx[cur[ev->pid[i]]++] = i;
  free(cur);
  *off_out = off;
  *idx_out = idx;
  return 0;
}

/* Event.sort_key (model.py:61-63): (start, end, category, pid, tid, name, corr or -1) */
static int cmp_sort_key(int64_t a, int64_t b, const void* c) {
  const xo_events_t* ev = ((const ectx*)c)->ev;
  int r;
  if ((r = CMP(ev->start[a], ev->start[b]))) return r;
  if ((r = CMP(ev_end(ev, a), ev_end(ev, b)))) return r;
  if ((r = CMP(ev->cat[a], ev->cat[b]))) return r;
  if ((r = CMP(ev->pid[a], ev->pid[b]))) return r;
  if ((r = CMP(ev->tid[a], ev->tid[b]))) return r;
  if ((r = CMP(ev->name[a], ev->name[b]))) return r;
  int64_t ca = ev->has_corr[a] ? ev->corr[a] : -1;
  int64_t cb = ev->has_corr[b] ? ev->corr[b] : -1;
  return CMP(ca, cb);
}

/* ------------------------------------------------------------------------ */
/* validation (model.py:137-228), event rules; meta rules live on the host   */
/* ------------------------------------------------------------------------ */
static int cmp_nesting(int64_t a, int64_t b, const void* c) {
  /* (start, -end, idx) within one (pid, tid); model.py:140 */
  const xo_events_t* ev = ((const ectx*)c)->ev;
  int r;
  if ((r = CMP(ev->tid[a], ev->tid[b]))) return r;
  if ((r = CMP(ev->start[a], ev->start[b]))) return r;
  if ((r = CMP(ev_end(ev, b), ev_end(ev, a)))) return r;
  return CMP(a, b);
}

typedef struct {
  int64_t pid, corr;
} pc_t;

static int cmp_pc(const void* x, const void* y) {
  const pc_t* a = (const pc_t*)x;
  const pc_t* b = (const pc_t*)y;
  int r = CMP(a->pid, b->pid);
  return r ? r : CMP(a->corr, b->corr);
}

int64_t xo_validate_count(const xo_events_t* ev) {
  int64_t bad = 0;
  /* api correlations per pid (model.py:186-189): sorted (pid, corr) set */
  int64_t n_api = 0, n_ops = 0;
  for (int64_t i = 0; i < ev->n; i++) {
    n_api += ev->cat[i] == 4 && ev->has_corr[i];
    n_ops += ev->cat[i] == 0;
  }
  pc_t* api = (pc_t*)malloc((size_t)(n_api + 1) * sizeof(pc_t));
  int64_t k = 0;
  for (int64_t i = 0; i < ev->n; i++)
    if (ev->cat[i] == 4 && ev->has_corr[i]) {
      api[k].pid = ev->pid[i];
      api[k].corr = ev->corr[i];
      k++;
    }
  qsort(api, (size_t)n_api, sizeof(pc_t), cmp_pc);
  int64_t* ops = (int64_t*)malloc((size_t)(n_ops ? n_ops : 1) * sizeof(int64_t));
  k = 0;
  for (int64_t i = 0; i < ev->n; i++) {
    int64_t s = ev->start[i], d = ev->dur[i];
    if (d < 0) bad++;
    if (s < 0) bad++;
    int64_t dd = d > 0 ? d : 0;
    if (s > 0 && dd > MAX_TS - s) bad++;
    if (!ev->pid_has_meta[ev->pid[i]]) bad++;
    if (ev->cat[i] == 0) {
      ops[k++] = i;
    } else if (ev->cat[i] == 5 && ev->has_corr[i]) {
      pc_t key = {ev->pid[i], ev->corr[i]};
      if (!bsearch(&key, api, (size_t)n_api, sizeof(pc_t), cmp_pc)) bad++;
    }
  }
  free(api);
  /* nesting per (pid, tid): groups are dense (pid,tid) so sort by (tid, start, -end, idx) */
  ectx c = {ev};
  stable_sort(ops, n_ops, cmp_nesting, &c);
  int64_t* stack = (int64_t*)malloc((size_t)(n_ops ? n_ops : 1) * sizeof(int64_t));
  int64_t i = 0;
  while (i < n_ops) {
    int64_t j = i;
    while (j < n_ops && ev->tid[ops[j]] == ev->tid[ops[i]]) j++;
    int64_t sp = 0;
    for (int64_t q = i; q < j; q++) {
      int64_t e = ops[q];
      while (sp && ev_end(ev, stack[sp - 1]) <= ev->start[e]) sp--;
      if (sp && ev_end(ev, e) > ev_end(ev, stack[sp - 1])) {
        bad++;
        continue;
      }
      stack[sp++] = e;
    }
    i = j;
  }
  free(stack);
  free(ops);
  return bad;
}

/* ------------------------------------------------------------------------ */
/* compute_overlap (overlap.py:106-188) + sweep_pid (_sweep_py.py:29-115)    */
/* ------------------------------------------------------------------------ */
typedef struct {
  const xo_events_t* ev;
  const int64_t* idx; /* local -> global */
} lctx;

static int cmp_rank(int64_t a, int64_t b, const void* c) {
  /* (start, -end, tid, name); stable => ties by position (overlap.py:99) */
  const lctx* l = (const lctx*)c;
  const xo_events_t* ev = l->ev;
  int64_t ga = l->idx[a], gb = l->idx[b];
  int r;
  if ((r = CMP(ev->start[ga], ev->start[gb]))) return r;
  if ((r = CMP(ev_end(ev, gb), ev_end(ev, ga)))) return r;
  if ((r = CMP(ev->tid[ga], ev->tid[gb]))) return r;
  return CMP(ev->name[ga], ev->name[gb]);
}

static int cmp_local_sort_key(int64_t a, int64_t b, const void* c) {
  const lctx* l = (const lctx*)c;
  ectx e = {l->ev};
  return cmp_sort_key(l->idx[a], l->idx[b], &e);
}

static int cmp_by_start(int64_t a, int64_t b, const void* c) {
  const lctx* l = (const lctx*)c;
  return CMP(l->ev->start[l->idx[a]], l->ev->start[l->idx[b]]);
}

static int cmp_by_end(int64_t a, int64_t b, const void* c) {
  const lctx* l = (const lctx*)c;
  return CMP(ev_end(l->ev, l->idx[a]), ev_end(l->ev, l->idx[b]));
}

static void cells_add(map_t* cells, int64_t key, int64_t len) {
  int f;
  int64_t s = map_slot(cells, key, &f);
  cells->vals[s] += len;
}

int xo_overlap(const xo_events_t* ev, int attribution, xo_overlap_t* out) {
  memset(out, 0, sizeof(*out));
  if (xo_validate_count(ev) != 0) return XO_INVALID;
  int64_t *off, *gidx;
  if (group_by_pid(ev, &off, &gidx)) return XO_NOMEM;
  int32_t P = ev->n_pids;
  out->span_lo = (int64_t*)calloc((size_t)P + 1, sizeof(int64_t));
  out->span_hi = (int64_t*)calloc((size_t)P + 1, sizeof(int64_t));
  out->tracked = (int64_t*)calloc((size_t)P + 1, sizeof(int64_t));
  out->has_events = (uint8_t*)calloc((size_t)P + 1, 1);
  trie_t trie;
  trie_init(&trie);
  int64_t cells_cap = 64, n_cells = 0;
  out->cell_pid = (int32_t*)malloc(cells_cap * sizeof(int32_t));
  out->cell_node = (int32_t*)malloc(cells_cap * sizeof(int32_t));
  out->cell_mask = (int32_t*)malloc(cells_cap * sizeof(int32_t));
  out->cell_ns = (int64_t*)malloc(cells_cap * sizeof(int64_t));

  for (int32_t p = 0; p < P; p++) {
    int64_t n = off[p + 1] - off[p];
    if (n == 0) continue;
    const int64_t* E = gidx + off[p];
    lctx L = {ev, E};
    /* pid_spans (model.py:125-134) */
    int64_t lo = ev->start[E[0]], hi = ev_end(ev, E[0]);
    for (int64_t i = 1; i < n; i++) {
      if (ev->start[E[i]] < lo) lo = ev->start[E[i]];
      if (ev_end(ev, E[i]) > hi) hi = ev_end(ev, E[i]);
    }
    out->span_lo[p] = lo;
    out->span_hi[p] = hi;
    out->has_events[p] = 1;

    /* op ranks (overlap.py:130-142) */
    int64_t n_ops = 0;
    for (int64_t i = 0; i < n; i++) n_ops += ev->cat[E[i]] == 0;
    int64_t* ranked = (int64_t*)malloc((size_t)(n_ops + 1) * sizeof(int64_t));
    int64_t k = 0;
    for (int64_t i = 0; i < n; i++)
      if (ev->cat[E[i]] == 0) ranked[k++] = i;
    stable_sort(ranked, n_ops, cmp_rank, &L);
    int64_t* ranks = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
    int32_t* rank_name = (int32_t*)malloc((size_t)(n_ops + 1) * sizeof(int32_t));
    for (int64_t r = 0; r < n_ops; r++) {
      ranks[ranked[r]] = r;
      rank_name[r] = ev->name[E[ranked[r]]];
    }
    int32_t* scratch = (int32_t*)malloc((size_t)(n_ops + 1) * sizeof(int32_t));

    /* CORRELATION fixed paths (overlap.py:144-163) */
    int64_t* fixed = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) fixed[i] = -1;
    if (attribution == 1) {
      int64_t* order = (int64_t*)malloc((size_t)n * sizeof(int64_t));
      for (int64_t i = 0; i < n; i++) order[i] = i;
      stable_sort(order, n, cmp_local_sort_key, &L);
      map_t api;
      map_init(&api, 64);
      for (int64_t q = 0; q < n; q++) {
        int64_t g = E[order[q]];
        if (ev->cat[g] == 4 && ev->has_corr[g]) {
          int f;
          int64_t s = map_slot(&api, ev->corr[g], &f);
          if (!f) api.vals[s] = ev->start[g]; /* setdefault: earliest in sort_key order */
        }
      }
      for (int64_t i = 0; i < n; i++) {
        int64_t g = E[i];
        if (ev->cat[g] != 5 || !ev->has_corr[g]) continue;
        int64_t ls = 0;
        if (!map_get(&api, ev->corr[g], &ls)) return XO_INVALID;
        int64_t m = 0;
        for (int64_t r = 0; r < n_ops; r++) {
          int64_t go = E[ranked[r]];
          if (ev->start[go] <= ls && ls < ev_end(ev, go)) scratch[m++] = ev->name[go];
        }
        fixed[i] = intern_names(&trie, scratch, m);
      }
      map_free(&api);
      free(order);
    }

    /* endpoint orders over nonzero-duration events (overlap.py:165-170) */
    int64_t nn = 0;
    for (int64_t i = 0; i < n; i++) nn += ev->dur[E[i]] > 0;
    int64_t* add = (int64_t*)malloc((size_t)(nn + 1) * sizeof(int64_t));
    int64_t* rem = (int64_t*)malloc((size_t)(nn + 1) * sizeof(int64_t));
    k = 0;
    for (int64_t i = 0; i < n; i++)
      if (ev->dur[E[i]] > 0) add[k++] = i;
    memcpy(rem, add, (size_t)nn * sizeof(int64_t));
    stable_sort(add, nn, cmp_by_start, &L);
    stable_sort(rem, nn, cmp_by_end, &L);

    /* sweep_pid (_sweep_py.py:29-115) */
    map_t cells;
    map_init(&cells, 64);
    int64_t tracked = 0;
    int64_t cat_count[6] = {0, 0, 0, 0, 0, 0};
    int64_t* fc_path = (int64_t*)malloc((size_t)(nn + 1) * sizeof(int64_t));
    int64_t* fc_cnt = (int64_t*)malloc((size_t)(nn + 1) * sizeof(int64_t));
    int64_t n_fc = 0;
    int64_t* active = (int64_t*)malloc((size_t)(n_ops + 1) * sizeof(int64_t));
    int64_t n_active = 0;
    int64_t cur_path = 0; /* path_table.get_id(()) */
    int ops_changed = 0, have_prev = 0;
    int64_t prev_t = 0;
    int64_t ia = 0, ir = 0;
    while (ir < nn) {
      int64_t t = ev_end(ev, E[rem[ir]]);
      if (ia < nn) {
        int64_t ta = ev->start[E[add[ia]]];
        if (ta < t) t = ta;
      }
      if (have_prev && t > prev_t) {
        int64_t len = t - prev_t;
        if (ops_changed) {
          for (int64_t a = 0; a < n_active; a++) scratch[a] = rank_name[active[a]];
          cur_path = intern_names(&trie, scratch, n_active);
          ops_changed = 0;
        }
        int64_t mask = 0;
        for (int c = 1; c <= 5; c++)
          if (cat_count[c] > 0) mask |= 1LL << (c - 1);
        if (n_fc) {
          int in_f = 0;
          for (int64_t f = 0; f < n_fc; f++) in_f |= fc_path[f] == cur_path;
          int64_t m = in_f ? (mask | 16) : mask;
          if (m) cells_add(&cells, (cur_path << 6) | m, len);
          for (int64_t f = 0; f < n_fc; f++)
            if (fc_path[f] != cur_path) cells_add(&cells, (fc_path[f] << 6) | 16, len);
          tracked += len;
        } else if (mask) {
          cells_add(&cells, (cur_path << 6) | mask, len);
          tracked += len;
        }
      }
      while (ir < nn && ev_end(ev, E[rem[ir]]) == t) {
        int64_t i = rem[ir++];
        int c = ev->cat[E[i]];
        if (c == 0) {
          int64_t r = ranks[i], a = 0;
          while (active[a] != r) a++;
          memmove(active + a, active + a + 1, (size_t)(n_active - a - 1) * sizeof(int64_t));
          n_active--;
          ops_changed = 1;
        } else if (fixed[i] >= 0) {
          int64_t f = 0;
          while (fc_path[f] != fixed[i]) f++;
          if (--fc_cnt[f] == 0) {
            fc_path[f] = fc_path[n_fc - 1];
            fc_cnt[f] = fc_cnt[n_fc - 1];
            n_fc--;
          }
        } else {
          cat_count[c]--;
        }
      }
      while (ia < nn && ev->start[E[add[ia]]] == t) {
        int64_t i = add[ia++];
        int c = ev->cat[E[i]];
        if (c == 0) {
          int64_t r = ranks[i], a = n_active; /* insort */
          while (a > 0 && active[a - 1] > r) a--;
          memmove(active + a + 1, active + a, (size_t)(n_active - a) * sizeof(int64_t));
          active[a] = r;
          n_active++;
          ops_changed = 1;
        } else if (fixed[i] >= 0) {
          int64_t f = 0;
          while (f < n_fc && fc_path[f] != fixed[i]) f++;
          if (f == n_fc) {
            fc_path[n_fc] = fixed[i];
            fc_cnt[n_fc++] = 0;
          }
          fc_cnt[f]++;
        } else {
          cat_count[c]++;
        }
      }
      prev_t = t;
      have_prev = 1;
    }
    out->tracked[p] = tracked;
    for (int64_t s = 0; s < cells.cap; s++) {
      if (!cells.used[s]) continue;
      if (n_cells == cells_cap) {
        cells_cap *= 2;
        out->cell_pid = (int32_t*)realloc(out->cell_pid, cells_cap * sizeof(int32_t));
        out->cell_node = (int32_t*)realloc(out->cell_node, cells_cap * sizeof(int32_t));
        out->cell_mask = (int32_t*)realloc(out->cell_mask, cells_cap * sizeof(int32_t));
        out->cell_ns = (int64_t*)realloc(out->cell_ns, cells_cap * sizeof(int64_t));
      }
      out->cell_pid[n_cells] = p;
      out->cell_node[n_cells] = (int32_t)(cells.keys[s] >> 6);
      out->cell_mask[n_cells] = (int32_t)(cells.keys[s] & 63);
      out->cell_ns[n_cells] = cells.vals[s];
      n_cells++;
    }
    map_free(&cells);
    free(fc_path);
    free(fc_cnt);
    free(active);
    free(add);
    free(rem);
    free(fixed);
    free(scratch);
    free(rank_name);
    free(ranks);
    free(ranked);
  }
  out->n_cells = n_cells;
  out->n_nodes = trie.n;
  out->node_parent = trie.parent;
  out->node_name = trie.name;
  trie.parent = NULL;
  trie.name = NULL;
  trie_free(&trie);
  free(off);
  free(gidx);
  return XO_OK;
}

void xo_free_overlap(xo_overlap_t* o) {
  free(o->cell_pid);
  free(o->cell_node);
  free(o->cell_mask);
  free(o->cell_ns);
  free(o->node_parent);
  free(o->node_name);
  free(o->span_lo);
  free(o->span_hi);
  free(o->tracked);
  free(o->has_events);
  memset(o, 0, sizeof(*o));
}

/* ------------------------------------------------------------------------ */
/* transition_sites (overlap.py:220-289)                                     */
/* ------------------------------------------------------------------------ */
static const int PAIR_SRC[4] = {1, 1, 2, 3};
static const int PAIR_DST[4] = {2, 3, 4, 4};

static int cmp_start_negend(int64_t a, int64_t b, const void* c) {
  const xo_events_t* ev = ((const ectx*)c)->ev;
  int r;
  if ((r = CMP(ev->start[a], ev->start[b]))) return r;
  return CMP(ev_end(ev, b), ev_end(ev, a));
}

static int cmp_start_end(int64_t a, int64_t b, const void* c) {
  const xo_events_t* ev = ((const ectx*)c)->ev;
  int r;
  if ((r = CMP(ev->start[a], ev->start[b]))) return r;
  return CMP(ev_end(ev, a), ev_end(ev, b));
}

/* _maximal_events (220-243): in-place filter of a sorted copy; returns count */
static int64_t maximal_events(const xo_events_t* ev, int64_t* lst, int64_t n, int64_t* out) {
  ectx c = {ev};
  stable_sort(lst, n, cmp_start_negend, &c);
  int64_t m = 0;
  int have_before = 0, have_group = 0;
  int64_t max_end_before = 0, group_start = 0, group_max_end = 0;
  for (int64_t q = 0; q < n; q++) {
    int64_t e = lst[q];
    int64_t s = ev->start[e], en = ev_end(ev, e);
    int contained;
    if (!have_group || s != group_start) {
      if (have_group) {
        max_end_before = !have_before ? group_max_end
                                      : (group_max_end > max_end_before ? group_max_end : max_end_before);
        have_before = 1;
      }
      group_start = s;
      group_max_end = en;
      have_group = 1;
      contained = have_before && max_end_before >= en;
    } else {
      contained = (group_max_end > en) || (have_before && max_end_before >= en);
    }
    if (!contained) out[m++] = e;
  }
  return m;
}

/* _union_intervals (246-255) */
static int64_t union_intervals(const xo_events_t* ev, int64_t* lst, int64_t n, int64_t* ulo, int64_t* uhi) {
  ectx c = {ev};
  stable_sort(lst, n, cmp_start_end, &c);
  int64_t m = 0;
  for (int64_t q = 0; q < n; q++) {
    int64_t e = lst[q];
    if (ev->dur[e] <= 0) continue;
    if (m && ev->start[e] <= uhi[m - 1]) {
      if (ev_end(ev, e) > uhi[m - 1]) uhi[m - 1] = ev_end(ev, e);
    } else {
      ulo[m] = ev->start[e];
      uhi[m] = ev_end(ev, e);
      m++;
    }
  }
  return m;
}

/* _covered (258-260) */
static int covered(const int64_t* ulo, const int64_t* uhi, int64_t m, int64_t x) {
  int64_t lo = 0, hi = m; /* bisect_right on lo <= x */
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (ulo[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  int64_t i = lo - 1;
  return i >= 0 && ulo[i] <= x && x < uhi[i];
}

int xo_transition_sites(const xo_events_t* ev, int pair_mask, int64_t* n_out, int32_t* out_pair,
                        int64_t* out_event) {
  *n_out = 0;
  if (xo_validate_count(ev) != 0) return XO_INVALID;
  int32_t G = ev->n_groups;
  /* by_key (pid, tid, cat) in trace order; groups are dense sorted (pid, tid) */
  int64_t* off = (int64_t*)calloc((size_t)G * 6 + 1, sizeof(int64_t));
  uint8_t* seen = (uint8_t*)calloc((size_t)G + 1, 1);
  for (int64_t i = 0; i < ev->n; i++) {
    seen[ev->tid[i]] = 1;
    off[(int64_t)ev->tid[i] * 6 + ev->cat[i] + 1]++;
  }
  for (int64_t q = 0; q < (int64_t)G * 6; q++) off[q + 1] += off[q];
  int64_t* lst = (int64_t*)malloc((size_t)(ev->n + 1) * sizeof(int64_t));
  int64_t* cur = (int64_t*)malloc(((size_t)G * 6 + 1) * sizeof(int64_t));
  memcpy(cur, off, ((size_t)G * 6 + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < ev->n; i++) lst[cur[(int64_t)ev->tid[i] * 6 + ev->cat[i]]++] = i;
  free(cur);
  int64_t* tmp = (int64_t*)malloc((size_t)(ev->n + 1) * sizeof(int64_t));
  int64_t* mx = (int64_t*)malloc((size_t)(ev->n + 1) * sizeof(int64_t));
  int64_t* ulo[4];
  int64_t* uhi[4];
  int64_t um[4];
  for (int c = 0; c < 4; c++) {
    ulo[c] = (int64_t*)malloc((size_t)(ev->n + 1) * sizeof(int64_t));
    uhi[c] = (int64_t*)malloc((size_t)(ev->n + 1) * sizeof(int64_t));
  }
  int64_t* pair_cnt = (int64_t*)calloc(4, sizeof(int64_t));
  int64_t total = 0;
  int64_t* plist[4];
  for (int k = 0; k < 4; k++) plist[k] = (int64_t*)malloc((size_t)(ev->n + 1) * sizeof(int64_t));
  for (int32_t g = 0; g < G; g++) {
    if (!seen[g]) continue;
    for (int c = 1; c <= 3; c++) {
      int64_t b = off[(int64_t)g * 6 + c], e = off[(int64_t)g * 6 + c + 1];
      memcpy(tmp, lst + b, (size_t)(e - b) * sizeof(int64_t));
      um[c] = union_intervals(ev, tmp, e - b, ulo[c], uhi[c]);
    }
    for (int k = 0; k < 4; k++) {
      if (!((pair_mask >> k) & 1)) continue;
      int src = PAIR_SRC[k], dst = PAIR_DST[k];
      if (um[src] == 0) continue;
      int64_t b = off[(int64_t)g * 6 + dst], e = off[(int64_t)g * 6 + dst + 1];
      memcpy(tmp, lst + b, (size_t)(e - b) * sizeof(int64_t));
      int64_t m = maximal_events(ev, tmp, e - b, mx);
      for (int64_t q = 0; q < m; q++)
        if (covered(ulo[src], uhi[src], um[src], ev->start[mx[q]])) plist[k][pair_cnt[k]++] = mx[q];
    }
  }
  ectx c = {ev};
  for (int k = 0; k < 4; k++) {
    stable_sort(plist[k], pair_cnt[k], cmp_sort_key, &c);
    for (int64_t q = 0; q < pair_cnt[k]; q++) {
      out_pair[total] = k;
      out_event[total] = plist[k][q];
      total++;
    }
    free(plist[k]);
  }
  *n_out = total;
  for (int q = 0; q < 4; q++) {
    free(ulo[q]);
    free(uhi[q]);
  }
  free(pair_cnt);
  free(mx);
  free(tmp);
  free(lst);
  free(off);
  free(seen);
  return XO_OK;
}

/* ------------------------------------------------------------------------ */
/* correct_trace (correction.py:79-186, _timeline.py:57-132)                 */
/* ------------------------------------------------------------------------ */
enum { ANN_START = 0, TRANSITION_HOOK = 1, API_INTERCEPT = 2, API_INTERNAL_HOOK = 3, ANN_END = 4 };
enum { H_ANN = 0, H_TRANS = 1, H_IC = 2, H_INT = 3 };

typedef struct {
  int64_t anchor;
  int64_t amount; /* scaled by L */
  int64_t owner;
  int64_t seq;
  int32_t subkind, tid, name, hook, pid;
} site_t;

static int cmp_site(int64_t a, int64_t b, const void* c) {
  /* Site.order_key (_timeline.py:52-54) = (anchor, subkind, tid, name); stable */
  const site_t* s = (const site_t*)c;
  int r;
  if ((r = CMP(s[a].pid, s[b].pid))) return r;
  if ((r = CMP(s[a].anchor, s[b].anchor))) return r;
  if ((r = CMP(s[a].subkind, s[b].subkind))) return r;
  if ((r = CMP(s[a].tid, s[b].tid))) return r;
  if ((r = CMP(s[a].name, s[b].name))) return r;
  return CMP(s[a].seq, s[b].seq);
}

static int64_t floor_div128(__int128 a, int64_t d) {
  __int128 q = a / d;
  if ((a % d != 0) && ((a < 0) != (d < 0))) q -= 1;
  return (int64_t)q;
}

typedef struct {
  int64_t K;
  const int64_t* a;
  const int64_t* b;
  const int64_t* prefix; /* K+1 */
} rmap_t;

/* RemovalMap.__call__ (_timeline.py:112-117) */
static int64_t rmap_apply(const rmap_t* m, int64_t y) {
  int64_t lo = 0, hi = m->K; /* bisect_right(ends, y) */
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (m->b[mid] <= y) lo = mid + 1;
    else hi = mid;
  }
  int64_t k = lo;
  int64_t removed = m->prefix[k];
  if (k < m->K && m->a[k] < y) removed += y - m->a[k];
  return y - removed;
}

int xo_correct(const xo_events_t* ev, const xo_profile_t* prof, int64_t* out_start, int64_t* out_dur,
               xo_corr_report_t* rep, int64_t n_queries, const int32_t* q_pid, const int64_t* q_val,
               int64_t* q_out) {
  rep->bad_event = -1;
  rep->original_total = 0;
  rep->corrected_total = 0;
  if (xo_validate_count(ev) != 0) return XO_INVALID;
  int32_t P = ev->n_pids;
  memset(rep->removed, 0, (size_t)P * 4 * sizeof(int64_t));
  memset(rep->shortfall, 0, (size_t)P * 4 * sizeof(int64_t));

  /* collect_sites (correction.py:79-112) */
  int64_t cap = 2 * ev->n + 16, ns = 0;
  site_t* sites = (site_t*)malloc((size_t)cap * sizeof(site_t));
  for (int64_t i = 0; i < ev->n; i++) {
    int c = ev->cat[i];
    if (c == 0) {
      site_t s0 = {ev->start[i], prof->ann_start, i, ns, ANN_START, ev->tid[i], ev->name[i], H_ANN, ev->pid[i]};
      sites[ns++] = s0;
      site_t s1 = {ev_end(ev, i), prof->ann_end, i, ns, ANN_END, ev->tid[i], ev->name[i], H_ANN, ev->pid[i]};
      sites[ns++] = s1;
    } else if (c == 4) {
      site_t s0 = {ev->start[i], prof->interception, i, ns, API_INTERCEPT, ev->tid[i], ev->name[i], H_IC, ev->pid[i]};
      sites[ns++] = s0;
      if (!prof->has_internal[ev->name[i]]) {
        rep->bad_event = i;
        free(sites);
        return XO_UNCALIBRATED;
      }
      site_t s1 = {ev->start[i], prof->internal[ev->name[i]], i, ns, API_INTERNAL_HOOK, ev->tid[i], ev->name[i],
                   H_INT, ev->pid[i]};
      sites[ns++] = s1;
    }
  }
  int64_t n_tr = 0;
  int32_t* tp = (int32_t*)malloc((size_t)(ev->n + 1) * sizeof(int32_t));
  int64_t* te = (int64_t*)malloc((size_t)(ev->n + 1) * sizeof(int64_t));
  xo_transition_sites(ev, 0x3, &n_tr, tp, te); /* WRAPPER_PAIRS (overlap.py:200-203) */
  if (ns + n_tr > cap) {
    cap = ns + n_tr;
    sites = (site_t*)realloc(sites, (size_t)cap * sizeof(site_t));
  }
  for (int64_t q = 0; q < n_tr; q++) {
    int64_t e = te[q];
    site_t s = {ev->start[e], prof->transition, e, ns, TRANSITION_HOOK, ev->tid[e], ev->name[e], H_TRANS, ev->pid[e]};
    sites[ns++] = s;
  }
  free(tp);
  free(te);
  int64_t* order = (int64_t*)malloc((size_t)(ns + 1) * sizeof(int64_t));
  for (int64_t q = 0; q < ns; q++) order[q] = q;
  stable_sort(order, ns, cmp_site, sites);

  /* spans */
  int64_t *off, *gidx;
  group_by_pid(ev, &off, &gidx);
  int64_t* lengths = (int64_t*)malloc((size_t)(ns + 1) * sizeof(int64_t));
  int64_t* ext_a = (int64_t*)malloc((size_t)(ns + 1) * sizeof(int64_t));
  int64_t* ext_b = (int64_t*)malloc((size_t)(ns + 1) * sizeof(int64_t));
  int64_t* sa = (int64_t*)malloc((size_t)(ns + 1) * sizeof(int64_t));
  int64_t* sb = (int64_t*)malloc((size_t)(ns + 1) * sizeof(int64_t));
  int64_t* pre = (int64_t*)malloc((size_t)(ns + 2) * sizeof(int64_t));
  int64_t* budget = (int64_t*)malloc((size_t)(ev->n + 1) * sizeof(int64_t));
  uint8_t* has_budget = (uint8_t*)calloc((size_t)ev->n + 1, 1);
  rmap_t* maps = (rmap_t*)calloc((size_t)P + 1, sizeof(rmap_t));
  int64_t* map_off = (int64_t*)calloc((size_t)P + 2, sizeof(int64_t));
  uint8_t* has_map = (uint8_t*)calloc((size_t)P + 1, 1);

  int64_t sp = 0;      /* cursor in sorted sites */
  int64_t slab_n = 0;  /* global nonzero slab storage cursor */
  for (int32_t p = 0; p < P; p++) {
    int64_t n = off[p + 1] - off[p];
    int64_t s0 = sp;
    while (sp < ns && sites[order[sp]].pid == p) sp++;
    if (n == 0) continue;
    const int64_t* E = gidx + off[p];
    int64_t lo = ev->start[E[0]], hi = ev_end(ev, E[0]);
    for (int64_t i = 1; i < n; i++) {
      if (ev->start[E[i]] < lo) lo = ev->start[E[i]];
      if (ev_end(ev, E[i]) > hi) hi = ev_end(ev, E[i]);
    }
    int64_t span_end = prof->span_end_in ? prof->span_end_in[p] : hi;
    rep->original_total += hi - lo;
    /* quantize_amounts (_timeline.py:57-67) + caps (correction.py:139-153) */
    __int128 cum = prof->residue_in ? prof->residue_in[p] : 0; /* floor(residue / L) = 0 */
    int64_t prev = 0;
    for (int64_t q = s0; q < sp; q++) {
      const site_t* s = &sites[order[q]];
      cum += s->amount;
      int64_t flo = floor_div128(cum, prof->L);
      int64_t amount = flo - prev;
      prev = flo;
      /* owner_index is never None for correction sites */
      if (!has_budget[s->owner]) {
        budget[s->owner] = ev->dur[s->owner];
        has_budget[s->owner] = 1;
      }
      int64_t capped = amount < budget[s->owner] ? amount : budget[s->owner];
      budget[s->owner] -= capped;
      rep->shortfall[(int64_t)p * 4 + s->hook] += amount - capped;
      lengths[q] = capped;
    }
    /* RemovalMap.__init__ (_timeline.py:93-110) */
    int have_prev = 0;
    int64_t prev_end = 0;
    int64_t base = slab_n;
    pre[base + 0] = 0;
    int64_t acc = 0;
    for (int64_t q = s0; q < sp; q++) {
      int64_t anchor = sites[order[q]].anchor, length = lengths[q];
      int64_t a = (!have_prev || anchor > prev_end) ? anchor : prev_end;
      int64_t b = a + length;
      ext_a[q] = a;
      ext_b[q] = b;
      if (length > 0) {
        sa[slab_n] = a;
        sb[slab_n] = b;
        slab_n++;
      }
      prev_end = (!have_prev || b > prev_end) ? b : prev_end;
      have_prev = 1;
    }
    (void)acc;
    map_off[p] = base;
    has_map[p] = 1;
    /* removed accounting (correction.py:155-157) */
    for (int64_t q = s0; q < sp; q++) {
      int64_t a = ext_a[q], b = ext_b[q];
      int64_t mb = b < span_end ? b : span_end;
      int64_t ma = a < span_end ? a : span_end;
      rep->removed[(int64_t)p * 4 + sites[order[q]].hook] += mb - ma;
    }
    maps[p].K = slab_n - base;
    maps[p].a = sa + base;
    maps[p].b = sb + base;
  }
  /* prefixes per pid: pre is laid out with one extra slot per pid */
  int64_t* prefix_all = (int64_t*)malloc((size_t)(slab_n + P + 1) * sizeof(int64_t));
  int64_t pcur = 0;
  for (int32_t p = 0; p < P; p++) {
    if (!has_map[p]) continue;
    int64_t base = map_off[p];
    int64_t* pr = prefix_all + pcur;
    pr[0] = 0;
    for (int64_t k = 0; k < maps[p].K; k++) pr[k + 1] = pr[k] + (sb[base + k] - sa[base + k]);
    maps[p].prefix = pr;
    pcur += maps[p].K + 1;
  }
  /* map_events (_timeline.py:120-132), positional (correction.py:158-165) */
  for (int64_t i = 0; i < ev->n; i++) {
    const rmap_t* m = &maps[ev->pid[i]];
    int64_t s = rmap_apply(m, ev->start[i]);
    out_start[i] = s;
    if (ev->cat[i] == 5) out_dur[i] = ev->dur[i];
    else out_dur[i] = rmap_apply(m, ev_end(ev, i)) - s;
  }
  /* fork/join remap (correction.py:166-182) */
  for (int64_t q = 0; q < n_queries; q++) {
    int32_t p = q_pid[q];
    q_out[q] = (p >= 0 && p < P && has_map[p]) ? rmap_apply(&maps[p], q_val[q]) : q_val[q];
  }
  /* corrected_total_ns = sum of pid_spans(out) */
  for (int32_t p = 0; p < P; p++) {
    int64_t n = off[p + 1] - off[p];
    if (n == 0) continue;
    const int64_t* E = gidx + off[p];
    int64_t lo = out_start[E[0]], hi = out_start[E[0]] + out_dur[E[0]];
    for (int64_t i = 1; i < n; i++) {
      int64_t s = out_start[E[i]], e = s + out_dur[E[i]];
      if (s < lo) lo = s;
      if (e > hi) hi = e;
    }
    rep->corrected_total += hi - lo;
  }
  free(prefix_all);
  free(maps);
  free(map_off);
  free(has_map);
  free(budget);
  free(has_budget);
  free(pre);
  free(sa);
  free(sb);
  free(ext_a);
  free(ext_b);
  free(lengths);
  free(order);
  free(sites);
  free(off);
  free(gidx);
  return XO_OK;
}
