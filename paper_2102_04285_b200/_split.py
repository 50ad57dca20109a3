"""Process batches for traces one device call cannot take whole.

Every result of the path is per process (overlap.py:126, correction.py:132;
"parallelizable across pids"), so a trace can be
analysed as consecutive calls over disjoint pid batches and the results
merged exactly.  Two cases need it:

* more than ``MAX_EVENTS_PER_CALL`` events: the C ABI takes up to 2^30 rows
  per call, and the default bound (2^28) keeps one call's workspace plus its
  columns well inside one B200's 180 GB;
* endpoint keys wider than 64 bits: a call's keys are
  ``pid index | time relative to the pid's first event | code``, so
  ``bits(#pids - 1) + bits(max per-pid span) + 4`` must fit 64 bits.  A batch
  of fewer pids needs fewer pid bits: batches are packed so that each fits.

Only a single process spanning 2^60 ns (36.5 years) or more, or holding more
than ``MAX_EVENTS_PER_CALL`` events by itself, cannot be split this way; the
device then reports XS_UNSUPPORTED / XS_BAD_ARGUMENT and the caller gets a
RuntimeError naming the limit.
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from .columnar import ColumnarTrace

MAX_EVENTS_PER_CALL = 1 << 28
CODE_BITS = 4  # endpoint code bits of the widest key family (overlap endpoints)


def _bits(v: int) -> int:
    return int(v).bit_length()


def pid_rows(ct: ColumnarTrace) -> list:
    """Row indices of each pid index (stable, ascending)."""
    order = np.argsort(ct.pid, kind="stable")
    bounds = np.searchsorted(ct.pid[order], np.arange(ct.n_pids + 1, dtype=np.int32))
    return [order[bounds[p]:bounds[p + 1]] for p in range(ct.n_pids)]


def pid_spans_host(ct: ColumnarTrace):
    """(lo, hi) per pid index over every event (pid_spans, model.py:125-134)."""
    lo = np.full(ct.n_pids, np.iinfo(np.int64).max, np.int64)
    hi = np.full(ct.n_pids, np.iinfo(np.int64).min, np.int64)
    np.minimum.at(lo, ct.pid, ct.start)
    np.maximum.at(hi, ct.pid, ct.start + ct.dur)
    return lo, hi


def needs_split(ct: ColumnarTrace) -> bool:
    """More rows than one call takes (O(1)).  Keys too wide for all pids at
    once are found by the device itself (XS_UNSUPPORTED after pass 1): the
    callers then fall back to plan_batches -- no host pass over the columns
    on the common path."""
    return ct.n > MAX_EVENTS_PER_CALL


def plan_batches(ct: ColumnarTrace, max_events: int = 0) -> list:
    """Pid-index batches (ascending) whose calls fit the key width and row
    bound; pids without events are left out."""
    max_events = max_events or MAX_EVENTS_PER_CALL
    lo, hi = pid_spans_host(ct)
    counts = np.bincount(ct.pid, minlength=ct.n_pids)
    groups = np.bincount(ct.group_pid, minlength=ct.n_pids) if ct.n_groups else np.zeros(ct.n_pids, np.int64)
    out, cur, cur_tb, cur_n, cur_g = [], [], 0, 0, 0
    for p in range(ct.n_pids):
        if counts[p] == 0:
            continue
        tb = _bits(max(int(hi[p] - lo[p]), 0))
        ntb = max(cur_tb, tb)
        # (pid and (pid, tid) group keys: the wider of the two index widths)
        ib = max(_bits(len(cur)), _bits(max(cur_g + int(groups[p]) - 1, 0)))
        if cur and (ib + ntb + CODE_BITS > 64 or cur_n + counts[p] > max_events):
            out.append(cur)
            cur, cur_tb, cur_n, cur_g = [], 0, 0, 0
            ntb = tb
        cur.append(p)
        cur_tb = ntb
        cur_n += int(counts[p])
        cur_g += int(groups[p])
    if cur:
        out.append(cur)
    return out


def sub_trace(ct: ColumnarTrace, pids: list, rows_by_pid: list):
    """The events of the given pid indices as a trace whose pid and
    (pid, tid) tables hold only those pids (so its keys spend only the
    batch's pid bits); returns (sub, rows in ct)."""
    pids = sorted(pids)
    rows = np.concatenate([rows_by_pid[p] for p in pids]) if pids else np.zeros(0, np.int64)
    rows.sort()
    pid_map = np.full(ct.n_pids, -1, np.int32)
    pid_map[pids] = np.arange(len(pids), dtype=np.int32)
    gsel = np.flatnonzero(pid_map[ct.group_pid] >= 0)
    grp_map = np.full(max(ct.n_groups, 1), -1, np.int32)
    grp_map[gsel] = np.arange(gsel.size, dtype=np.int32)
    sub = ColumnarTrace(ct.clock_domain, ct.start[rows], ct.dur[rows], pid_map[ct.pid[rows]],
                        grp_map[ct.tid[rows]], ct.cat[rows], ct.name[rows], ct.corr[rows], ct.has_corr[rows],
                        ct.pids[pids], pid_map[ct.group_pid[gsel]], ct.group_tid[gsel], ct.names, ct.processes,
                        ct.pid_has_meta[pids])
    return sub, rows


# ---------------------------------------------------------------------------
# Processes too wide for one call's keys (compute_overlap only)
#
# A process whose span needs more than WIDE_BITS bits cannot be keyed even
# alone (time + 4 code bits > 64).  Its overlap is computed over time windows
# [c_k, c_{k+1}) of span < 2^WIDE_BITS cut at instants where:
#   * no OPERATION strictly contains the cut (ranks, nesting and paths are
#     then window-local: overlap.py:96-99, 132-142 only compare operations
#     active at one instant), nor a correlated GPU event;
#   * no correlated GPU event sits on the other side of the cut from its
#     launcher (the launcher -- the earliest ACCEL_API with the id,
#     overlap.py:144-163 -- and the path at its start are then in the GPU
#     event's window, and the dangling-correlation rule is window-local).
# Resource events are clipped to each window they overlap; operations and
# zero-duration events go to the window holding their start.  The sweep of a
# window accounts exactly its part of the timeline (_sweep_py.py:29-115 is a
# function of the active set at each instant), so cells and tracked time add
# up over windows and the span is the union of the window spans.
# ---------------------------------------------------------------------------
WIDE_BITS = 59


def wide_pids(ct: ColumnarTrace) -> list:
    """Pid indices whose own span needs more than WIDE_BITS bits."""
    if ct.n == 0:
        return []
    lo, hi = pid_spans_host(ct)
    return [p for p in range(ct.n_pids) if hi[p] >= lo[p] and _bits(int(hi[p]) - int(lo[p])) > WIDE_BITS]


def _forbidden(sub: ColumnarTrace) -> np.ndarray:
    """[k, 2] closed integer ranges of instants that may not be cuts (merged,
    sorted): (start, end) of every operation and correlated GPU event,
    (first, last] of every launcher / correlated GPU event pair."""
    rng = []
    # operations and correlated GPU events are never cut (a clipped GPU piece
    # would lose its launcher -- the fixed path -- and its dangling check)
    op = (sub.cat == 0) | ((sub.cat == 5) & (sub.has_corr == 1))
    s, e = sub.start[op], sub.start[op] + sub.dur[op]
    m = e - s > 1
    if m.any():
        rng.append(np.stack([s[m] + 1, e[m] - 1], axis=1))
    api = (sub.cat == 4) & (sub.has_corr == 1)
    gpu = (sub.cat == 5) & (sub.has_corr == 1)
    if api.any() and gpu.any():
        # launcher = earliest ACCEL_API per id by Event.sort_key; its start
        # is what matters, and the earliest start is a lower bound for it
        ac, ast = sub.corr[api], sub.start[api]
        order = np.lexsort((ast, ac))
        ac, ast = ac[order], ast[order]
        first = np.r_[True, ac[1:] != ac[:-1]]
        ids, lstart = ac[first], ast[first]
        gc, gs = sub.corr[gpu], sub.start[gpu]
        k = np.searchsorted(ids, gc)
        ok = (k < ids.size) & (ids[np.minimum(k, ids.size - 1)] == gc)
        ls = lstart[np.minimum(k, ids.size - 1)][ok]
        g = gs[ok]
        a, b = np.minimum(ls, g), np.maximum(ls, g)
        m = b > a
        if m.any():
            rng.append(np.stack([a[m] + 1, b[m]], axis=1))
    if not rng:
        return np.zeros((0, 2), np.int64)
    r = np.concatenate(rng)
    r = r[np.argsort(r[:, 0], kind="stable")]
    out = []
    cs, ce = int(r[0, 0]), int(r[0, 1])
    for a, b in r[1:]:
        a, b = int(a), int(b)
        if a <= ce + 1:
            ce = max(ce, b)
        else:
            out.append((cs, ce))
            cs, ce = a, b
    out.append((cs, ce))
    return np.asarray(out, np.int64)


def wide_cuts(sub: ColumnarTrace) -> list:
    """Cut instants for a one-process trace so that every window spans fewer
    than 2^WIDE_BITS ns; ValueError when a forbidden range (a long operation,
    or a launcher far from its kernel) is itself that wide."""
    lo = int(sub.start.min())
    hi = int((sub.start + sub.dur).max())
    step = 1 << (WIDE_BITS - 1)
    bad = _forbidden(sub)
    cuts, prev = [], lo
    while hi - prev >= (1 << WIDE_BITS) - 1:
        target = prev + step
        # the largest valid instant in (prev, target]: target itself unless a
        # forbidden range holds it, then just before that range
        k = int(np.searchsorted(bad[:, 0], target, side="right")) - 1 if bad.size else -1
        c = target
        if k >= 0 and bad[k, 1] >= target:
            c = int(bad[k, 0]) - 1
        if c <= prev:  # a forbidden range covers (prev, target]: cut right after it
            c = int(bad[k, 1]) + 1
            if c - prev >= 1 << WIDE_BITS:
                raise ValueError("a single operation (or a launcher / kernel pair) spans >= 2^59 ns: "
                                 "no operation-free instant to cut the process at")
        cuts.append(c)
        prev = c
    return cuts


def row_cuts(sub: ColumnarTrace, max_rows: int) -> list:
    """Cut instants for a one-process trace holding more than ``max_rows``
    events: near every max_rows/2-th start, moved out of the forbidden ranges
    (_forbidden); windows then hold about half a call each."""
    starts = np.sort(sub.start)
    bad = _forbidden(sub)
    step = max(1, max_rows // 2)
    cuts, prev = [], None
    for j in range(step, starts.size, step):
        c = int(starts[j])
        k = int(np.searchsorted(bad[:, 0], c, side="right")) - 1 if bad.size else -1
        if k >= 0 and bad[k, 1] >= c:  # inside a forbidden range: just before it, else just after it
            c = int(bad[k, 0]) - 1
            if prev is not None and c <= prev:
                c = int(bad[k, 1]) + 1
        if (prev is None or c > prev) and c > int(starts[0]):
            cuts.append(c)
            prev = c
    return cuts


def window_trace(sub: ColumnarTrace, a: Optional[int], b: Optional[int]) -> ColumnarTrace:
    """The events of a one-process trace in window [a, b): resource events
    clipped to it, operations and zero-duration events by their start."""
    lo = np.iinfo(np.int64).min if a is None else a
    hi = np.iinfo(np.int64).max if b is None else b
    end = sub.start + sub.dur
    point = ((sub.dur == 0) | (sub.cat == 0)) & (sub.start >= lo) & (sub.start < hi)
    span = (sub.dur > 0) & (sub.cat != 0) & (sub.start < hi) & (end > lo)
    rows = np.nonzero(point | span)[0]
    s = sub.start[rows]
    e = end[rows]
    clip = (sub.cat[rows] != 0) & (sub.dur[rows] > 0)
    s2 = np.where(clip, np.maximum(s, lo), s)
    e2 = np.where(clip, np.minimum(e, hi), e)
    return ColumnarTrace(sub.clock_domain, s2, e2 - s2, sub.pid[rows], sub.tid[rows], sub.cat[rows], sub.name[rows],
                         sub.corr[rows], sub.has_corr[rows], sub.pids, sub.group_pid, sub.group_tid, sub.names,
                         sub.processes, sub.pid_has_meta)


# ---------------------------------------------------------------------------
# Correction of processes too wide for one call's keys: exact gap compression
#
# correct_trace depends on times only through their order (site order,
# transition maximality and coverage, the remap's bisection), owner budgets
# (durations), and slab extents a = max(anchor, E), b = a + len
# (_timeline.py:93-117, correction.py:139-157).  Let B bound the process's
# total removable time (sum over its sites of |amount| + 1).  Shrinking every
# gap between consecutive event endpoints that is longer than L = B + 1 to
# length L changes none of these: order is kept (a strictly increasing map),
# a budget spanning a gap stays >= L > any one site's amounts, and the slab
# chain E can overrun an anchor by at most B < L, so no slab reaches a
# shrunk part and the slabs after a gap start at their anchors as before.
# The correction of the compressed process, shifted back by the compression
# offset of every endpoint, is the correction of the process
# (rmap(y) = rmap'(y') + offset(y); a time inside a shrunk gap maps with the
# gap's slope-1 tail).  Report totals are recomputed from the spans.
# ---------------------------------------------------------------------------
class Compression:
    """Per-pid gap compression: points[p] (sorted endpoints) and cum[p]
    (offset removed at or before each point), L[p]."""

    def __init__(self):
        self.points, self.cum, self.L = {}, {}, {}

    def offset_of(self, p: int, t: np.ndarray) -> np.ndarray:
        """Compression offset of endpoint times of pid p (every t is a point)."""
        pts, cum = self.points[p], self.cum[p]
        return cum[np.searchsorted(pts, t)]

    def compress_time(self, p: int, t: int) -> tuple:
        """(t', offset, tail) for an arbitrary time t of pid p: t' = the
        compressed time, and the corrected t = rmap'(t') + offset + tail."""
        pts, cum, L = self.points[p], self.cum[p], self.L[p]
        k = int(np.searchsorted(pts, t, side="right")) - 1
        if k < 0:
            return int(t), 0, 0
        base = int(pts[k])
        tail = max(0, int(t) - base - L)
        return int(t) - tail - int(cum[k]), int(cum[k]), tail


def removable_bound(ct: ColumnarTrace, rows: np.ndarray, profile) -> int:
    """Upper bound on the total time correct_trace can remove from these
    rows: every site's |amount| + 1 (correction.py:79-112)."""
    from fractions import Fraction
    import math

    cat = ct.cat[rows]
    n_op = int((cat == 0).sum())
    n_api = int((cat == 4).sum())
    n_bs = int(((cat == 2) | (cat == 3)).sum())
    ann = abs(Fraction(profile.annotation_ns))
    internal = max((abs(Fraction(v)) for v in profile.api_internal_ns.values()), default=Fraction(0))
    per_op = math.ceil(ann) + 2
    per_api = math.ceil(abs(Fraction(profile.api_interception_ns))) + math.ceil(internal) + 2
    per_bs = math.ceil(abs(Fraction(profile.transition_ns))) + 1
    return n_op * per_op + n_api * per_api + n_bs * per_bs


def compress_wide(ct: ColumnarTrace, pids: list, profile) -> tuple:
    """(compressed trace, Compression) for the given pid indices; the other
    pids' rows are unchanged.  ValueError when a compressed process is still
    too wide (its endpoints alone span 2^WIDE_BITS ns at gap length L)."""
    rows_by_pid = pid_rows(ct)
    start = ct.start.copy()
    end = ct.start + ct.dur
    new_end = end.copy()
    comp = Compression()
    for p in pids:
        rows = rows_by_pid[p]
        L = removable_bound(ct, rows, profile) + 1
        pts = np.unique(np.concatenate([ct.start[rows], end[rows]]))
        d = np.diff(pts)
        cum = np.concatenate([[0], np.cumsum(np.where(d > L, d - L, 0))]).astype(np.int64)
        comp.points[p], comp.cum[p], comp.L[p] = pts, cum, L
        start[rows] = ct.start[rows] - comp.offset_of(p, ct.start[rows])
        new_end[rows] = end[rows] - comp.offset_of(p, end[rows])
        if _bits(int(pts[-1] - cum[-1]) - int(pts[0])) > WIDE_BITS:
            raise ValueError("a process spans >= 2^59 ns even with every idle gap shrunk")
    procs = []
    pid_index = {int(v): i for i, v in enumerate(ct.pids.tolist())}
    from .model import ProcessMeta
    for m in ct.processes:
        p = pid_index.get(m.pid)
        if p in comp.points:
            fk = None if m.fork_ns is None else comp.compress_time(p, m.fork_ns)[0]
            jn = None if m.join_ns is None else comp.compress_time(p, m.join_ns)[0]
            m = ProcessMeta(m.pid, m.name, m.parent, fk, jn)
        procs.append(m)
    out = ColumnarTrace(ct.clock_domain, start, new_end - start, ct.pid, ct.tid, ct.cat, ct.name, ct.corr,
                        ct.has_corr, ct.pids, ct.group_pid, ct.group_tid, ct.names, tuple(procs), ct.pid_has_meta)
    return out, comp


def uncompress_columns(ct: ColumnarTrace, comp: Compression, start_c: np.ndarray, dur_c: np.ndarray) -> tuple:
    """Corrected columns of the compressed trace -> corrected columns of ct."""
    start = np.array(start_c, np.int64, copy=True)
    dur = np.array(dur_c, np.int64, copy=True)
    rows_by_pid = pid_rows(ct)
    end = ct.start + ct.dur
    for p in comp.points:
        rows = rows_by_pid[p]
        s_off = comp.offset_of(p, ct.start[rows])
        e_off = comp.offset_of(p, end[rows])
        new_s = start[rows] + s_off
        gpu = ct.cat[rows] == 5
        new_e = start[rows] + dur[rows] + e_off
        start[rows] = new_s
        dur[rows] = np.where(gpu, ct.dur[rows], new_e - new_s)  # GPU events shift only (_timeline.py:120-132)
    return start, dur
