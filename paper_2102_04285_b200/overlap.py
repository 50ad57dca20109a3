"""Cross-stack overlap accounting and transition counting (drop-in for
``pkg/src/xstrace/overlap.py``).

Same public names, signatures and return types as the reference; the work
runs on the GPU through ``libxstrace_b200.so``:

* ``compute_overlap``   overlap.py:106-188  -> xs_overlap (csrc/xs_overlap.cu)
* ``transition_sites``  overlap.py:263-289  -> xs_transition_sites (csrc/xs_transitions.cu)
* ``count_transitions`` overlap.py:292-295

``compute_overlap_columnar`` is the scalable twin taking a ``ColumnarTrace``
(no Python ``Event`` objects), which is what the bench and multi-GPU path use.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _engine, _lib, _split
from .columnar import ColumnarTrace, produced_columnar
from .model import Category, InvalidTraceError, Trace, format_violations, meta_violations


class Attribution(Enum):
    """How a GPU event picks its operation path (overlap.py:41-45)."""

    INSTANT = "instant"
    CORRELATION = "correlation"


class OverlapKey(tuple):
    """(pid, operation path, category set) of one overlap cell (overlap.py:48-58).

    Same fields, hashing-by-value, equality and labels as the reference's
    frozen dataclass; stored as a tuple so decoding millions of cells from the
    device stays cheap (config 5 produces ~4M cells)."""

    __slots__ = ()

    def __new__(cls, pid, path, categories):
        return tuple.__new__(cls, (pid, path, categories))

    pid = property(lambda self: self[0])
    path = property(lambda self: self[1])
    categories = property(lambda self: self[2])

    def __repr__(self) -> str:
        return f"OverlapKey(pid={self[0]!r}, path={self[1]!r}, categories={self[2]!r})"

    def __reduce__(self):
        return (OverlapKey, tuple(self))

    def category_label(self) -> str:
        return "+".join(c.name for c in sorted(self.categories))

    def path_label(self) -> str:
        return "/".join(self.path) if self.path else "-"


class Breakdown:
    """Accumulated ns per (pid, operation path, category set) (overlap.py:61-77).

    Same fields and methods as the reference's dataclass.  A Breakdown decoded
    from a device result keeps the cell arrays and builds the ``cells`` dict
    of OverlapKeys on first access: millions of deep-path cells (config 5)
    cost seconds of Python object construction, which callers that only read
    spans / untracked / the raw arrays never pay.
    """

    __slots__ = ("_cells", "_lazy", "spans", "untracked")

    def __init__(self, cells=None, spans=None, untracked=None):
        self._cells = {} if cells is None else cells
        self._lazy = None
        self.spans = {} if spans is None else spans
        self.untracked = {} if untracked is None else untracked

    @property
    def cells(self) -> dict:
        if self._lazy is not None:
            build, self._lazy = self._lazy, None
            self._cells = build()
        return self._cells

    @cells.setter
    def cells(self, value: dict) -> None:
        self._lazy = None
        self._cells = value

    def __eq__(self, other) -> bool:
        if not isinstance(other, Breakdown):
            return NotImplemented
        return self.cells == other.cells and self.spans == other.spans and self.untracked == other.untracked

    __hash__ = None

    def __repr__(self) -> str:
        return f"Breakdown(cells={self.cells!r}, spans={self.spans!r}, untracked={self.untracked!r})"

    def span_ns(self, pid: int) -> int:
        lo, hi = self.spans[pid]
        return hi - lo

    def pid_cells(self, pid: int) -> dict:
        return {k: v for k, v in self.cells.items() if k.pid == pid}

    def total_attributed(self, pid: int) -> int:
        return sum(v for k, v in self.cells.items() if k.pid == pid)


TRANSITION_PAIRS = (
    (Category.HIGH_LEVEL, Category.BACKEND),
    (Category.HIGH_LEVEL, Category.SIMULATOR),
    (Category.BACKEND, Category.ACCEL_API),
    (Category.SIMULATOR, Category.ACCEL_API),
)
WRAPPER_PAIRS = (
    (Category.HIGH_LEVEL, Category.BACKEND),
    (Category.HIGH_LEVEL, Category.SIMULATOR),
)


@dataclass(frozen=True)
class TransitionCounts:
    counts: tuple

    def get(self, src, dst) -> int:
        for f, t, c in self.counts:
            if f == src and t == dst:
                return c
        return 0

    def as_dict(self) -> dict:
        return {(f, t): c for f, t, c in self.counts}


_CATS = [Category(c) for c in range(6)]
_MASK_CATS = [frozenset(_CATS[c] for c in range(1, 6) if m & (1 << (c - 1))) for m in range(32)]


def _as_columnar(trace) -> ColumnarTrace:
    if isinstance(trace, ColumnarTrace):
        return trace
    ct = produced_columnar(trace)  # (a Trace correct_trace returned: its columns are at hand)
    return ct if ct is not None else ColumnarTrace.from_trace(trace)


def _source_trace(trace, ct: ColumnarTrace) -> Trace:
    if not isinstance(trace, ColumnarTrace):
        return trace
    return ct._source if ct._source is not None else ct.to_trace()


def _raise_invalid(trace, ct):
    raise InvalidTraceError(format_violations(_source_trace(trace, ct)))


def decode_paths(ct: ColumnarTrace, parents: np.ndarray, names: np.ndarray, needed=None) -> list:
    """Trie nodes -> name tuples (a parent is always allocated before its child)."""
    n = int(parents.shape[0])
    paths: list = [()] * max(n, 1)
    par = parents.tolist()
    nm = names.tolist()
    table = ct.names
    for i in range(1, n):
        paths[i] = paths[par[i]] + (table[nm[i]],)
    return paths


def decode_breakdown(ct: ColumnarTrace, raw, lazy: bool = True) -> Breakdown:
    """Breakdown of a device overlap result; the cells dict is built on first
    access unless ``lazy`` is False."""
    bd = _decode_breakdown(ct, raw)

    def build():
        # millions of small tuples: keep the cyclic GC from rescanning the
        # growing heap during the bulk build (they hold no cycles)
        import gc
        was = gc.isenabled()
        gc.disable()
        try:
            return _decode_cells(ct, raw)
        finally:
            if was:
                gc.enable()

    if lazy and raw.cell_ns.shape[0] > 4096:
        bd._lazy = build
    else:
        bd.cells = build()
    return bd


def _decode_cells(ct: ColumnarTrace, raw) -> dict:
    paths = decode_paths(ct, raw.node_parent, raw.node_name)
    pids = ct.pids.tolist()
    mk = tuple.__new__
    pv = [pids[p] for p in raw.cell_pid.tolist()] if len(pids) != 1 else [pids[0]] * raw.cell_pid.shape[0]
    return dict(zip((mk(OverlapKey, (p, paths[nd], _MASK_CATS[m])) for p, nd, m in
                     zip(pv, raw.cell_node.tolist(), raw.cell_mask.tolist())), raw.cell_ns.tolist()))


def _decode_breakdown(ct: ColumnarTrace, raw) -> Breakdown:
    bd = Breakdown()
    pids = ct.pids.tolist()
    for p in range(ct.n_pids):
        if raw.has_events[p]:
            lo, hi = int(raw.span_lo[p]), int(raw.span_hi[p])
            bd.spans[pids[p]] = (lo, hi)
            bd.untracked[pids[p]] = (hi - lo) - int(raw.tracked[p])
    return bd


def compute_overlap_columnar(ct: ColumnarTrace, attribution: Attribution = Attribution.INSTANT,
                             device_trace=None, _source=None) -> Breakdown:
    """compute_overlap over a ColumnarTrace (or an already-uploaded DeviceTrace)."""
    if meta_violations(ct.processes):
        _raise_invalid(_source if _source is not None else ct, ct)
    if device_trace is None and _split.needs_split(ct):
        return _overlap_batched(ct, attribution, _source)
    eng = _engine.get()
    dt = device_trace if device_trace is not None else _engine.DeviceTrace(ct, eng.device)
    attr = 1 if Attribution(attribution) is Attribution.CORRELATION else 0
    try:
        raw = eng.overlap(dt, attr)
    except _engine.XsError as exc:
        if exc.status == _lib.XS_INVALID_TRACE:
            _raise_invalid(_source if _source is not None else ct, ct)
        if exc.status == _lib.XS_UNSUPPORTED and device_trace is None:
            return _overlap_batched(ct, attribution, _source)  # keys too wide for all pids at once
        raise
    return decode_breakdown(ct, raw)


def merge_breakdowns(parts) -> Breakdown:
    """Breakdowns of disjoint pid sets -> one Breakdown."""
    bd = Breakdown()
    for b in parts:
        bd.cells.update(b.cells)
        bd.spans.update(b.spans)
        bd.untracked.update(b.untracked)
    return bd


def _merge_windows(parts) -> Breakdown:
    """Breakdowns of time windows of the same pids -> one Breakdown: cells
    and tracked time add up, spans are unions."""
    bd = Breakdown()
    cells, tracked = {}, {}
    for b in parts:
        for k, v in b.cells.items():
            cells[k] = cells.get(k, 0) + v
        for pid, (lo, hi) in b.spans.items():
            tracked[pid] = tracked.get(pid, 0) + (hi - lo) - b.untracked[pid]
            if pid in bd.spans:
                l0, h0 = bd.spans[pid]
                bd.spans[pid] = (min(l0, lo), max(h0, hi))
            else:
                bd.spans[pid] = (lo, hi)
    bd.cells = cells
    for pid, (lo, hi) in bd.spans.items():
        bd.untracked[pid] = (hi - lo) - tracked[pid]
    return bd


def _overlap_wide(ct: ColumnarTrace, p: int, rows_by_pid, attr: int, _source) -> Breakdown:
    """One process too wide for one call's keys, or holding more rows than
    one call takes, over operation-free time windows (_split.wide_cuts /
    row_cuts / window_trace)."""
    eng = _engine.get()
    sub, _ = _split.sub_trace(ct, [p], rows_by_pid)
    try:
        cuts = _split.wide_cuts(sub)
    except ValueError as exc:
        raise _engine.XsError(_lib.XS_UNSUPPORTED, f"xs_overlap: unsupported input {exc}") from None
    if sub.n > _split.MAX_EVENTS_PER_CALL:
        cuts = sorted(set(cuts) | set(_split.row_cuts(sub, _split.MAX_EVENTS_PER_CALL)))
    bounds = [None] + cuts + [None]
    parts = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        win = _split.window_trace(sub, a, b)
        if win.n == 0:
            continue
        try:
            raw = eng.overlap(_engine.DeviceTrace(win, eng.device), attr)
        except _engine.XsError as exc:
            if exc.status == _lib.XS_INVALID_TRACE:
                _raise_invalid(_source if _source is not None else ct, ct)
            raise
        parts.append(decode_breakdown(win, raw, lazy=False))
    return _merge_windows(parts)


def _overlap_batched(ct: ColumnarTrace, attribution, _source) -> Breakdown:
    """compute_overlap over pid batches (_split: more rows than one call
    takes, or keys wider than 64 bits over all pids); exact because every
    cell, span and untracked value is per pid (overlap.py:126).  A process
    too wide for one call's keys by itself goes through time windows."""
    eng = _engine.get()
    attr = 1 if Attribution(attribution) is Attribution.CORRELATION else 0
    rows_by_pid = _split.pid_rows(ct)
    parts = []
    wide = _split.wide_pids(ct)
    counts = np.bincount(ct.pid, minlength=ct.n_pids)
    wide += [p for p in np.nonzero(counts > _split.MAX_EVENTS_PER_CALL)[0].tolist() if p not in wide]
    for p in wide:
        parts.append(_overlap_wide(ct, p, rows_by_pid, attr, _source))
    todo = list(reversed([b for b in ([q for q in batch if q not in wide] for batch in _split.plan_batches(ct)) if b]))
    while todo:
        pids = todo.pop()
        sub, _ = _split.sub_trace(ct, pids, rows_by_pid)
        try:
            raw = eng.overlap(_engine.DeviceTrace(sub, eng.device), attr)
        except _engine.XsError as exc:
            if exc.status == _lib.XS_INVALID_TRACE:
                _raise_invalid(_source if _source is not None else ct, ct)
            if exc.status == _lib.XS_UNSUPPORTED and len(pids) > 1:  # (CORRELATION keys also hold path bits)
                h = len(pids) // 2
                todo += [pids[h:], pids[:h]]
                continue
            raise
        parts.append(decode_breakdown(sub, raw, lazy=False))
    return merge_breakdowns(parts)


def compute_overlap(trace, attribution: Attribution = Attribution.INSTANT, kernel=None) -> Breakdown:
    """Attribute every nanosecond of each pid's timeline to overlap cells.

    Rejects invalid traces with InvalidTraceError carrying the violations.
    ``kernel`` is accepted for signature compatibility with the reference's
    plugin point (overlap.py:106-113); the device pipeline is always used.
    """
    ct = _as_columnar(trace)
    return compute_overlap_columnar(ct, attribution, _source=trace)


def _transition_lists(trace, pair_mask: int):
    ct = _as_columnar(trace)
    if meta_violations(ct.processes):
        _raise_invalid(trace, ct)
    eng = _engine.get()
    dt = _engine.DeviceTrace(ct, eng.device)
    try:
        pair, event = eng.transition_sites(dt, pair_mask)
    except _engine.XsError as exc:
        if exc.status == _lib.XS_INVALID_TRACE:
            _raise_invalid(trace, ct)
        raise
    return ct, pair, event


def transition_sites(trace) -> dict:
    """Counted transitions per pair: maximal inner events whose start lies
    inside an active outer-category event on the same tid (overlap.py:263-289)."""
    ct, pair, event = _transition_lists(trace, 0xF)
    src = _source_trace(trace, ct)
    events = src.events
    out = {p: [] for p in TRANSITION_PAIRS}
    for k, e in zip(pair.tolist(), event.tolist()):
        out[TRANSITION_PAIRS[k]].append(events[e])
    return out


def transition_site_indices(trace, pair_mask: int = 0xF) -> dict:
    """Event row indices per pair (columnar-friendly form of transition_sites)."""
    _, pair, event = _transition_lists(trace, pair_mask)
    out = {p: [] for k, p in enumerate(TRANSITION_PAIRS) if (pair_mask >> k) & 1}
    for k, e in zip(pair.tolist(), event.tolist()):
        out[TRANSITION_PAIRS[k]].append(e)
    return out


def count_transitions(trace) -> TransitionCounts:
    """Count language transitions once per counted inner event (overlap.py:292-295)."""
    _, pair, _ = _transition_lists(trace, 0xF)
    counts = np.bincount(pair, minlength=4) if len(pair) else np.zeros(4, np.int64)
    return TransitionCounts(tuple((s, d, int(counts[k])) for k, (s, d) in enumerate(TRANSITION_PAIRS)))


def sweep_pid(starts, ends, cats, ranks, fixed_paths, add_order, rem_order, rank_name_ids, path_table):
    """The reference's kernel plugin protocol (overlap.py:30-38, 106-113;
    _sweep_py.py:29-115) served by the device pipeline: one pid's boundary
    walk -> ``(cells {(path_id << 6) | mask: ns}, tracked_ns)``, path ids
    interned in the caller's ``path_table`` (tuples of name ids).

    The pid's nonzero-duration events (``add_order``) become a one-pid
    ColumnarTrace; each operation sits on its own tid numbered by its rank,
    so the device's (start, -end, tid, name) rank order reproduces the given
    ``ranks`` and its multi-tid path merge is ``path_of``'s rank-ordered,
    adjacent-deduplicated name list.

    GPU events pinned to a launch-site path (``fixed_paths[i] >= 0``,
    CORRELATION, _sweep_py.py:70-79, 93-99, 107-111) run through the device's
    CORRELATION attribution: each distinct fixed path p gets a private instant
    after the pid's events where operations named ``path_table.paths[p]``
    (rank-ordered by tid) are the only active events, and a zero-duration
    ACCEL_API launcher there carries a correlation id shared with the pinned
    GPU events.  Operation-only intervals are untracked and zero-duration
    events add no cells, so the extra region changes nothing but the span,
    and ``tracked`` is read directly."""
    idx = list(add_order)
    n = len(idx)
    if n == 0:
        return {}, 0
    s = np.array([starts[i] for i in idx], np.int64)
    e = np.array([ends[i] for i in idx], np.int64)
    c = np.array([cats[i] for i in idx], np.uint8)
    fx = np.array([fixed_paths[i] for i in idx], np.int64)
    is_op = c == 0
    rk = np.array([ranks[i] for i in idx], np.int64)
    nid = [rank_name_ids[r] if op else None for r, op in zip(rk.tolist(), is_op.tolist())]
    tid = np.where(is_op, rk + 1, 0)
    corr = np.zeros(n, np.int64)
    has = np.zeros(n, np.uint8)
    pinned = sorted({int(p) for p in fx.tolist() if p >= 0})
    extra = []  # (start, dur, cat, tid, name id, corr, has_corr)
    if pinned:
        slot = {p: k for k, p in enumerate(pinned)}
        sel = fx >= 0
        corr[sel] = [slot[int(p)] + 1 for p in fx[sel].tolist()]
        has[sel] = 1
        t0 = int(e.max()) + 2
        tid_base = int(tid.max()) + 1
        for p in pinned:
            tp = t0 + 3 * slot[p]
            for j, name_id in enumerate(path_table.paths[p]):  # rank order = tid order (equal intervals)
                extra.append((tp, 2, 0, tid_base + j, name_id, 0, 0))
            extra.append((tp + 1, 0, 4, 0, None, slot[p] + 1, 1))  # the launcher
    names_used = {str(x) for x in nid if x is not None} | {str(x[4]) for x in extra if x[4] is not None} | {"_"}
    names = sorted(names_used)
    nrank = {x: k for k, x in enumerate(names)}
    name = np.array([nrank[str(x)] if x is not None else nrank["_"] for x in nid], np.int32)
    if extra:
        xs = list(zip(*extra))
        s = np.concatenate([s, np.array(xs[0], np.int64)])
        d = np.concatenate([e - s[:n], np.array(xs[1], np.int64)])
        c = np.concatenate([c, np.array(xs[2], np.uint8)])
        tid = np.concatenate([tid, np.array(xs[3], np.int64)])
        name = np.concatenate([name, np.array([nrank[str(x)] if x is not None else nrank["_"] for x in xs[4]],
                                              np.int32)])
        corr = np.concatenate([corr, np.array(xs[5], np.int64)])
        has = np.concatenate([has, np.array(xs[6], np.uint8)])
    else:
        d = e - s
    from .model import ProcessMeta
    m = s.shape[0]
    ct = ColumnarTrace.from_arrays(0, s, d, np.ones(m, np.int64), tid, c, name, names, corr=corr, has_corr=has,
                                   processes=(ProcessMeta(1, "pid"),))
    bd = compute_overlap_columnar(ct, Attribution.CORRELATION if pinned else Attribution.INSTANT)
    cells = {}
    for key, ns in bd.cells.items():
        pid_path = path_table.get_id(tuple(int(x) for x in key.path))
        mask = sum(1 << (int(cc) - 1) for cc in key.categories)
        cells[(pid_path << 6) | mask] = ns
    lo, hi = bd.spans[1]
    tracked = (hi - lo) - bd.untracked[1]
    return cells, tracked
