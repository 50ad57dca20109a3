/*
 * xstrace_b200.h -- C ABI of the B200-native trace-analysis hot path.
 *
 * This is the drop-in boundary: the reference (RL-Scope / xstrace) is a
 * Python package whose hot path is
 *     compute_overlap(trace, attribution)    pkg/src/xstrace/overlap.py:106
 *     correct_trace(trace, profile)          pkg/src/xstrace/correction.py:115
 *     transition_sites(trace)                pkg/src/xstrace/overlap.py:263
 *     count_transitions(trace)               pkg/src/xstrace/overlap.py:292
 *     validate_trace / require_valid         pkg/src/xstrace/model.py:159,231
 * with its only native plugin point the per-pid sweep kernel
 *     sweep_pid(...)                         pkg/src/xstrace/_sweep.pyx:17
 * (selected at overlap.py:30-38 via the ``kernel=`` argument).  The Python
 * host package (paper_2102_04285_b200) keeps that API and binds these entry
 * points with ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - All array pointers inside xs_events_t are DEVICE pointers owned by the
 *     caller (the library never frees them).  Outputs named *_dev are device
 *     buffers allocated by the caller; everything else is host memory.
 *   - Every entry point is stream-ordered on `stream` and returns an
 *     xs_status (0 = ok).  Intermediate buffers live in the context's
 *     workspace, which grows on demand and is reused across calls.
 *   - Status codes map 1:1 to the reference's exceptions:
 *       XS_INVALID_TRACE -> InvalidTraceError   (model.py:115-122)
 *       XS_UNCALIBRATED  -> UncalibratedHookError (correction.py:38-39)
 *       XS_BAD_ARGUMENT  -> ValueError
 */
#ifndef XSTRACE_B200_H
#define XSTRACE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct xs_ctx xs_ctx_t;
typedef void* xs_stream_t; /* cudaStream_t */

typedef enum {
  XS_OK = 0,
  XS_INVALID_TRACE = 1,
  XS_UNCALIBRATED = 2,
  XS_CUDA_ERROR = 3,
  XS_BAD_ARGUMENT = 4,
  XS_UNSUPPORTED = 5,
  XS_NO_MEMORY = 6
} xs_status;

/* Columnar events (see paper_2102_04285_b200/columnar.py for the interning
 * rules that make integer compares equal the reference's Python compares). */
typedef struct {
  int64_t n;                  /* number of events (rows, trace order)       */
  const int64_t* start;       /* [n] ns                                      */
  const int64_t* dur;         /* [n] ns                                      */
  const int32_t* pid;         /* [n] dense pid index                         */
  const int32_t* tid;         /* [n] dense (pid, tid) group index            */
  const uint8_t* cat;         /* [n] Category 0..5                           */
  const int32_t* name;        /* [n] rank in the sorted name table           */
  const int64_t* corr;        /* [n] correlation id                          */
  const uint8_t* has_corr;    /* [n] 1 when correlation is not None          */
  int32_t n_pids;
  int32_t n_groups;
  int32_t n_names;
  int32_t reserved;
  const int32_t* group_pid;   /* [n_groups] pid index of each group          */
  const uint8_t* pid_has_meta;/* [n_pids] pid has a ProcessMeta              */
} xs_events_t;

/* Calibration profile, exact (fractions.Fraction in the reference,
 * calibration.py:142-149; per-site amounts correction.py:90-100): every
 * amount a is split as a = whole + frac / L with 0 <= frac < L, where L is the
 * common denominator of all amounts, held as `words` little-endian 64-bit
 * words (words = 1, 2, 4 or 8; L < 2^(64 words - 1)).  quantize_amounts
 * (_timeline.py:57-67) then needs only the fractional parts' running sum
 * modulo L: q_i = whole_i + [ (sum_{j<=i} frac_j mod L) < frac_i ], so no
 * profile is too fine-grained for the device. */
typedef struct {
  int32_t words;
  int32_t reserved;
  const uint64_t* L;           /* DEVICE [words]                                               */
  int64_t whole[4];            /* floor of ANN_START (annotation/2), ANN_END (annotation -     */
                               /* annotation/2), transition, api_interception                  */
  const uint64_t* frac;        /* DEVICE [(4 + n_names) * words]: (amount - whole) * L, rows   */
                               /* in the order of `whole`, then api_internal[name] per name    */
  const int64_t* internal;     /* DEVICE [n_names] floor(api_internal[name])                    */
  const uint8_t* has_internal; /* DEVICE [n_names]                                              */
  /* Window carries (a process corrected as consecutive time windows, each a
   * pid of its own in the call: distributed.analyze_sharded).  Both NULL for
   * the reference's whole-process semantics.
   *   residue_in  DEVICE [n_pids * words] or NULL: the running fractional sum
   *               (mod L, < L) of the process's amounts before this window --
   *               quantize_amounts' `cum` (_timeline.py:61-66) does not
   *               restart at a window;
   *   span_end_in DEVICE [n_pids] or NULL: absolute time at which removed_ns
   *               is clipped instead of the window's own last end (the
   *               process's span end, correction.py:155-156; the next cut
   *               for an inner window, which makes a slab running past the
   *               cut visible as removed < total slab length). */
  const uint64_t* residue_in;
  const int64_t* span_end_in;
} xs_profile_t;

/* Sizes of the last overlap result held by the context. */
typedef struct {
  int64_t n_cells;
  int32_t n_nodes;            /* path trie nodes; node 0 = empty path     */
  int32_t n_pids;
} xs_overlap_info_t;

typedef struct {
  int64_t original_total;     /* CorrectionReport.original_total_ns  */
  int64_t corrected_total;    /* CorrectionReport.corrected_total_ns */
  int64_t n_sites;
  int64_t n_slabs;
} xs_correct_info_t;

const char* xs_status_str(int status);
const char* xs_last_error(xs_ctx_t* ctx);
int xs_version(void);

int xs_ctx_create(int device, xs_ctx_t** out);
void xs_ctx_destroy(xs_ctx_t* ctx);
/* bytes currently held by the context workspace */
int64_t xs_ctx_workspace_bytes(xs_ctx_t* ctx);

/* validate_trace event rules (model.py:159-228) as one device pass plus the
 * OPERATION nesting check; *n_bad = number of event-level violations found
 * (0 => valid).  Process-metadata rules are O(#pids) and stay on the host. */
int xs_validate(xs_ctx_t* ctx, const xs_events_t* ev, int64_t* n_bad, xs_stream_t stream);

/* compute_overlap (overlap.py:106-188).  attribution: 0 INSTANT, 1 CORRELATION.
 * Results stay in the context until the next call; fetch with
 * xs_overlap_info / xs_overlap_fetch. */
int xs_overlap(xs_ctx_t* ctx, const xs_events_t* ev, int attribution, xs_stream_t stream);
int xs_overlap_info(xs_ctx_t* ctx, xs_overlap_info_t* info);
/* host outputs: cells (n_cells each), trie (n_nodes each), per-pid arrays (n_pids each) */
int xs_overlap_fetch(xs_ctx_t* ctx, int32_t* cell_pid, int32_t* cell_node, int32_t* cell_mask,
                     int64_t* cell_ns, int32_t* node_parent, int32_t* node_name, int64_t* span_lo,
                     int64_t* span_hi, int64_t* tracked, uint8_t* has_events, xs_stream_t stream);

/* correct_trace (correction.py:115-186): writes corrected start/duration in
 * trace order to caller device buffers; per-pid removed/shortfall via
 * xs_correct_report.  *bad_event receives the first ACCEL_API event index
 * whose name the profile lacks when XS_UNCALIBRATED is returned. */
int xs_correct(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof,
               int64_t* out_start_dev, int64_t* out_dur_dev, int64_t* bad_event, xs_stream_t stream);
/* removed/shortfall: host [n_pids*4] in HOOK_KINDS order */
int xs_correct_report(xs_ctx_t* ctx, xs_correct_info_t* info, int64_t* removed, int64_t* shortfall,
                      xs_stream_t stream);
/* RemovalMap of the last xs_correct applied to (pid, value) pairs (fork/join
 * remap, correction.py:166-182); all three arrays are device pointers. */
int xs_remap(xs_ctx_t* ctx, int64_t n, const int32_t* pid_dev, const int64_t* val_dev,
             int64_t* out_dev, xs_stream_t stream);

/* correct_trace + compute_overlap(corrected): the `xstrace analyze --profile`
 * path (cli.py:168-171) in one call; results as for the two calls above. */
int xs_analyze(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int attribution,
               int64_t* out_start_dev, int64_t* out_dur_dev, int64_t* bad_event, xs_stream_t stream);

/* xs_analyze plus the D2H of the corrected columns into caller host buffers
 * (pinned for the copy to overlap): the copy is issued on a side stream as
 * soon as the correction is final and overlaps the overlap pass; both are
 * complete when the call returns. */
int xs_analyze_to_host(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int attribution,
                       int64_t* out_start_dev, int64_t* out_dur_dev, int64_t* out_start_host, int64_t* out_dur_host,
                       int64_t* bad_event, xs_stream_t stream);
/* The same, returning with the D2H still in flight on the context's copy
 * stream: it overlaps the caller's next call (batched analyses).  The device
 * outputs must stay allocated and the host buffers unread until
 * xs_host_copy_wait, which waits for every copy issued so far. */
int xs_analyze_to_host_async(xs_ctx_t* ctx, const xs_events_t* ev, const xs_profile_t* prof, int attribution,
                             int64_t* out_start_dev, int64_t* out_dur_dev, int64_t* out_start_host,
                             int64_t* out_dur_host, int64_t* bad_event, xs_stream_t stream);
int xs_host_copy_wait(xs_ctx_t* ctx);

/* transition_sites (overlap.py:263-289) for the pairs selected by pair_mask
 * (bit k = TRANSITION_PAIRS[k]).  *n_out = number of sites; fetch the
 * (pair, event index) list, ordered per pair by Event.sort_key. */
int xs_transition_sites(xs_ctx_t* ctx, const xs_events_t* ev, int pair_mask, int64_t* n_out,
                        xs_stream_t stream);
int xs_transition_fetch(xs_ctx_t* ctx, int32_t* pair, int64_t* event, xs_stream_t stream);

/* Union time of one category (0..5): metrics._union_ns
 * (metrics.py:41-58).  per_pid = 0: one trace-wide union (busy_fraction,
 * metrics.py:87-91) -> out_ns[0]; per_pid = 1: one union per pid, the
 * gpu_busy_ns of procview.build_process_tree (procview.py:68-77) ->
 * out_ns[n_pids].  *span_lo / *span_hi receive the trace span
 * (metrics._trace_span, metrics.py:31-38; lo > hi when there are no events).
 * All outputs are host memory. */
int xs_union(xs_ctx_t* ctx, const xs_events_t* ev, int category, int per_pid, int64_t* out_ns, int64_t* span_lo,
             int64_t* span_hi, xs_stream_t stream);
/* sampled_utilization (metrics.py:61-84): *utilized = number of periods
 * [lo + kP, lo + (k+1)P) intersecting a GPU event of nonzero duration;
 * *n_intervals = number of disjoint GPU union intervals (fetch them, sorted,
 * with xs_union_intervals_fetch for utilization_samples). */
int xs_utilization(xs_ctx_t* ctx, const xs_events_t* ev, int64_t period_ns, int64_t* utilized, int64_t* n_intervals,
                   int64_t* span_lo, int64_t* span_hi, xs_stream_t stream);
int xs_union_intervals_fetch(xs_ctx_t* ctx, int64_t* out_lo, int64_t* out_hi, xs_stream_t stream);

/* XSTRACE1 chunk decoding (traceio._decode_chunk, traceio.py:214-240;
 * docs/trace-format.md:20-50), host memory in and out.  xs_chunk_info parses
 * the header and string table (str_off/str_len may be NULL for a sizes-only
 * pass); xs_chunk_decode writes the n_records rows into the columns, mapping
 * each chunk-local string index through name_map.  Non-zero returns carry the
 * reference's TraceFormatError message in err (xs_chunk_info returns 2 for a
 * bad magic, 3 for a bad version). */
typedef struct {
  int64_t clock_domain;
  int32_t chunk_index;
  int32_t n_records;
  int32_t n_strings;
  int32_t version;
  int64_t records_offset;
} xs_chunk_info_t;
int xs_chunk_info(const uint8_t* buf, int64_t len, const char* context, xs_chunk_info_t* info, int64_t* str_off,
                  int64_t* str_len, char* err, int errlen);
int xs_chunk_decode(const uint8_t* buf, int64_t len, const char* context, const xs_chunk_info_t* info,
                    const int32_t* name_map, int64_t* pid, int64_t* tid, uint8_t* cat, int32_t* name, int64_t* start,
                    int64_t* dur, int64_t* corr, uint8_t* has_corr, char* err, int errlen);

/* Packed upload format (the host -> device wire layout of a columnar trace;
 * ColumnarTrace.pinned builds it).  Every column keeps its exact values in
 * the narrowest width that holds them: start as a per-256-row int64 base
 * plus a 32-bit offset (or raw int64), dur / corr as 32 or 64 bits, pid / tid
 * / name indices as 8, 16 or 32 bits, and cat | has_corr << 7 in one byte.
 * A 32-bit start / dur / corr column may hold a few values that do not fit:
 * their slot holds 0xFFFFFFFF and the exact value sits in the exception
 * table (global row, column 0 start / 1 dur / 2 corr, value), sorted by row;
 * pass the exceptions whose rows fall in [row0, row0 + n).
 * xs_unpack widens rows [row0, row0 + n) of a packed trace (device pointers,
 * possibly a slice) into the xs_events_t columns (device buffers of n rows).
 * Replaces the per-column host -> device copies of the reference's in-process
 * Trace (model.py:78-88, the events tuple): the result is bit-identical to the
 * unpacked columns. */
typedef struct {
  int64_t n;                 /* rows to widen                                     */
  int64_t row0;              /* global row of the first (start bases are per 256 */
                             /* global rows; start_base[0] is block row0 >> 8)   */
  const void* start;         /* [n] uint32 offsets (start_w 4) or int64 (8)       */
  const int64_t* start_base; /* per 256-row block when start_w == 4               */
  const void* dur;           /* [n] uint32 / int64                                 */
  const void* pid;           /* [n] uint8 / uint16 / int32                         */
  const void* tid;
  const void* name;
  const void* corr;          /* [n] uint32 / int64                                 */
  const uint8_t* catf;       /* [n] cat | has_corr << 7                            */
  int32_t start_w, dur_w, pid_w, tid_w, name_w, corr_w;
  int64_t n_exc;             /* exceptions in this row range                      */
  const int64_t* exc_row;    /* [n_exc] global rows                               */
  const int64_t* exc_val;    /* [n_exc] exact values                              */
  const uint8_t* exc_col;    /* [n_exc] 0 start, 1 dur, 2 corr                    */
} xs_packed_t;
int xs_unpack(xs_ctx_t* ctx, const xs_packed_t* pk, int64_t* start, int64_t* dur, int32_t* pid, int32_t* tid,
              uint8_t* cat, int32_t* name, int64_t* corr, uint8_t* has_corr, xs_stream_t stream);

/* Host-side builder of the packed format (no device work; host threads).
 * `ev` holds HOST pointers to the engine-dtype columns.  xs_pack_plan reads
 * every column once and fixes widths, exception count and the block layout:
 * 13 sections, 16-byte aligned, in the order start, start_base, dur, corr,
 * pid, tid, name, catf, group_pid, pid_has_meta, exc_row, exc_val, exc_col
 * (the layout ColumnarTrace.pinned documents).  XS_UNSUPPORTED: cat >= 128 or
 * has_corr > 1 (not packable; upload the wide columns).  xs_pack_fill writes
 * the block (normally page-locked) with the same row partition; padding
 * bytes are zero.  n_threads <= 0 uses every hardware thread.  Replaces the
 * reference's in-process Trace hand-off (model.py:78-88) as the staging of
 * an analysis call's input. */
#define XS_PACK_MAX_THREADS 64
typedef struct {
  int64_t n, n_exc, total;
  int32_t start_w, dur_w, corr_w, pid_w, tid_w, name_w;
  int32_t n_threads, reserved;
  int64_t offset[13], nbytes[13];
  int64_t thread_exc[XS_PACK_MAX_THREADS]; /* first exception slot of each thread */
} xs_pack_layout_t;
int xs_pack_plan(const xs_events_t* ev, int n_threads, xs_pack_layout_t* lay);
int xs_pack_fill(const xs_events_t* ev, const xs_pack_layout_t* lay, void* block, int64_t block_bytes);

/* Device synthetic generator (TEST / BENCH INFRASTRUCTURE, SURVEY 8(f4);
 * synth.py:246-375 shape): n_pids processes x `iterations` DDPG-style
 * iterations, both twins at once (uninstrumented start/dur and the
 * instrumented start_inst/dur_inst with the given constant hook amounts).
 * xs_synth_plan sizes it (one sync) and returns the row count;
 * xs_synth_generate writes the columns (device buffers of that many rows,
 * pid-contiguous; tid = (pid, tid) group index with groups 0, [1], 1000 per
 * pid) and span[2*p] / span[2*p+1] = the end of pid p's uninstrumented /
 * instrumented timeline (every pid starts at 0).  names: DEVICE int32[11],
 * the name-table ranks of kernel, script, launch, memcpy, inference,
 * inference_backend, simulation, simulation_sim, backprop, backprop_backend,
 * and the outer op. */
typedef struct {
  int64_t iterations;
  uint64_t seed;
  int32_t n_pids;
  int32_t outer_op;          /* wrap each iteration's phases in one more op      */
  int32_t second_tid_ops;    /* mirror every phase op on tid 1                    */
  int32_t first_pid;         /* pid value of the first process (random streams   */
                             /* are per pid value: any block of pids regenerates */
                             /* the same processes)                               */
  int64_t ann_start, ann_end, transition, interception, launch, memcpy;
  const int32_t* names;
} xs_synth_spec_t;
int xs_synth_plan(xs_ctx_t* ctx, const xs_synth_spec_t* spec, int64_t* n_events, xs_stream_t stream);
int xs_synth_generate(xs_ctx_t* ctx, const xs_synth_spec_t* spec, int64_t* start, int64_t* dur, int64_t* start_inst,
                      int64_t* dur_inst, int32_t* pid, int32_t* tid, uint8_t* cat, int32_t* name, int64_t* corr,
                      uint8_t* has_corr, int64_t* span, xs_stream_t stream);

/* Number of kernel launches issued by the library since context creation
 * (instrumentation for the bench's gpu_launches field). */
int64_t xs_launch_count(xs_ctx_t* ctx);

/* Per-stage device timing with CUDA events recorded on the launching stream
 * (bench/roofline instrumentation).  enable resets the counters; read returns
 * the number of stages and fills accumulated milliseconds / occurrences. */
int xs_profile_enable(xs_ctx_t* ctx, int on);
int xs_profile_read(xs_ctx_t* ctx, double* ms, int64_t* calls, int n);
const char* xs_profile_stage_name(int stage);

#ifdef __cplusplus
}
#endif
#endif
