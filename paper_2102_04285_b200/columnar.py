"""Columnar (SoA) trace: the layout the device path consumes.

A ``Trace`` of Python ``Event`` objects cannot scale past a few million
events (~0.9 GB per 1M in the reference), so the engine's
native input is this structure of arrays.  The interning rules make integer
comparisons on the device equal the reference's Python comparisons:

* ``pid``  -- index into ``pids`` (sorted numeric pid values: events U metas),
* ``tid``  -- index into the sorted table of distinct (pid, tid) pairs, so two
  tids of one pid compare like the reference's ints (Site.order_key,
  _op_rank_order) and a group index is also the (pid, tid) key,
* ``name`` -- rank of the name in ``sorted(names)`` (Python str order), so name
  ties break exactly like ``str`` comparisons,
* ``corr`` / ``has_corr`` -- correlation id and a presence flag (None).

Row order is the trace's event order; the row index plays the role of the
reference's event index in every stable-sort tie-break.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .model import Category, Event, ProcessMeta, Trace


def _intern(values: np.ndarray):
    """(sorted distinct values, index of each value among them): a hash
    factorisation (O(n)) when pandas is present, else a sort."""
    values = np.asarray(values, dtype=np.int64)
    try:
        import pandas as pd
    except ImportError:  # pragma: no cover
        uniq, inv = np.unique(values, return_inverse=True)
        return uniq, inv.reshape(-1).astype(np.int64)
    codes, uniq = pd.factorize(values, sort=True)
    return np.asarray(uniq, dtype=np.int64), codes.astype(np.int64)


@dataclass
class ColumnarTrace:
    clock_domain: int
    start: np.ndarray       # int64
    dur: np.ndarray         # int64
    pid: np.ndarray         # int32 index into pids
    tid: np.ndarray         # int32 index into groups
    cat: np.ndarray         # uint8
    name: np.ndarray        # int32 rank into names
    corr: np.ndarray        # int64
    has_corr: np.ndarray    # uint8
    pids: np.ndarray        # int64 sorted pid values
    group_pid: np.ndarray   # int32 pid index of each group
    group_tid: np.ndarray   # int64 tid value of each group
    names: list             # sorted names
    processes: tuple = ()
    pid_has_meta: Optional[np.ndarray] = None  # uint8 [n_pids]
    _source: Optional[Trace] = field(default=None, repr=False)
    _pinned: Optional[dict] = field(default=None, repr=False)  # column -> pinned host tensor (see pinned())

    @property
    def n(self) -> int:
        return int(self.start.shape[0])

    @property
    def n_pids(self) -> int:
        return int(self.pids.shape[0])

    @property
    def n_groups(self) -> int:
        return int(self.group_pid.shape[0])

    def __post_init__(self):
        if self.pid_has_meta is None:
            meta = {m.pid for m in self.processes}
            self.pid_has_meta = np.array([int(p) in meta for p in self.pids], dtype=np.uint8)

    # -- construction --------------------------------------------------------
    @classmethod
    def from_trace(cls, trace: Trace) -> "ColumnarTrace":
        """Intern a Trace of Event-like objects (duck-typed: the reference's
        own ``xstrace.Event`` works too)."""
        evs = trace.events
        n = len(evs)
        start = np.fromiter((e.start for e in evs), dtype=np.int64, count=n)
        dur = np.fromiter((e.duration for e in evs), dtype=np.int64, count=n)
        pid_v = np.fromiter((e.pid for e in evs), dtype=np.int64, count=n)
        tid_v = np.fromiter((e.tid for e in evs), dtype=np.int64, count=n)
        cat = np.fromiter((int(e.category) for e in evs), dtype=np.uint8, count=n)
        corr_list = [e.correlation for e in evs]
        has_corr = np.fromiter((c is not None for c in corr_list), dtype=np.uint8, count=n)
        corr = np.fromiter((c if c is not None else 0 for c in corr_list), dtype=np.int64, count=n)
        name_list = [e.name for e in evs]
        names = sorted(set(name_list))
        rank = {s: i for i, s in enumerate(names)}
        name = np.fromiter((rank[s] for s in name_list), dtype=np.int32, count=n)
        return cls.from_arrays(trace.clock_domain, start, dur, pid_v, tid_v, cat, name, names,
                               corr, has_corr, trace.processes, _source=trace)

    @classmethod
    def from_arrays(cls, clock_domain, start, dur, pid_values, tid_values, cat, name, names,
                    corr=None, has_corr=None, processes=(), _source=None) -> "ColumnarTrace":
        """Build from raw columns: pid/tid are *values*, name are ranks into
        ``names`` (which must be sorted)."""
        n = int(np.asarray(start).shape[0])
        start = np.ascontiguousarray(start, dtype=np.int64)
        dur = np.ascontiguousarray(dur, dtype=np.int64)
        pid_values = np.asarray(pid_values, dtype=np.int64)
        tid_values = np.asarray(tid_values, dtype=np.int64)
        meta_pids = np.array(sorted({m.pid for m in processes}), dtype=np.int64)
        ev_pids, pid_codes = _intern(pid_values)
        pids = np.union1d(ev_pids, meta_pids).astype(np.int64)
        pid = np.searchsorted(pids, ev_pids).astype(np.int32)[pid_codes] if n else np.zeros(0, np.int32)
        if n:
            tids, tid_codes = _intern(tid_values)
            key = pid.astype(np.int64) * max(tids.shape[0], 1) + tid_codes  # (pid, tid) order = key order
            uniq, inv = _intern(key)
            group_pid = (uniq // max(tids.shape[0], 1)).astype(np.int32)
            group_tid = tids[uniq % max(tids.shape[0], 1)].astype(np.int64)
            tid = inv.astype(np.int32)
        else:
            group_pid = np.zeros(0, np.int32)
            group_tid = np.zeros(0, np.int64)
            tid = np.zeros(0, np.int32)
        if corr is None:
            corr = np.zeros(n, np.int64)
            has_corr = np.zeros(n, np.uint8)
        return cls(clock_domain, start, dur, pid, tid,
                   np.ascontiguousarray(cat, dtype=np.uint8),
                   np.ascontiguousarray(name, dtype=np.int32),
                   np.ascontiguousarray(corr, dtype=np.int64),
                   np.ascontiguousarray(has_corr, dtype=np.uint8),
                   pids, group_pid, group_tid, list(names), tuple(processes), _source=_source)

    def present_pid_mask(self) -> np.ndarray:
        """bool[n_pids]: pids with at least one event (memoised per trace)."""
        m = self.__dict__.get("_present_mask")
        if m is None:
            m = np.bincount(self.pid, minlength=self.n_pids)[: self.n_pids] > 0 if self.n else \
                np.zeros(self.n_pids, bool)
            self.__dict__["_present_mask"] = m
        return m

    _COLUMNS = ("start", "dur", "pid", "tid", "cat", "name", "corr", "has_corr", "group_pid", "pid_has_meta")

    def pinned(self, packed: bool = True) -> "ColumnarTrace":
        """The same trace staged in page-locked host memory as ONE block, so
        the device upload of each call is one asynchronous DMA at full PCIe
        rate.  ``packed`` (default) stores the block in the packed upload
        format (include/xstrace_b200.h, xs_packed_t: every column in the
        narrowest width that holds its exact values, ~17-22 B/event instead
        of 38; the device widens it with xs_unpack) and keeps the numpy
        columns as they are; ``packed=False`` makes the columns themselves
        16-byte-aligned views of the block."""
        import torch

        if packed:
            hold = {}

            def alloc(nbytes):
                hold["block"] = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
                return hold["block"].numpy()

            got = pack_native(self, alloc)  # native builder, host threads
            if got is not None:
                lay, block = got[0], hold["block"]
                return ColumnarTrace(self.clock_domain, self.start, self.dur, self.pid, self.tid, self.cat,
                                     self.name, self.corr, self.has_corr, self.pids, self.group_pid, self.group_tid,
                                     self.names, self.processes, self.pid_has_meta, self._source,
                                     {"_block": block, "_packed": lay})
        cols = [np.ascontiguousarray(getattr(self, k)) for k in self._COLUMNS]
        offs, total = [], 0
        for a in cols:
            offs.append(total)
            total += (a.nbytes + 15) // 16 * 16
        block = torch.empty(max(total, 16), dtype=torch.uint8).pin_memory()
        raw = block.numpy()
        tens, arrs = {"_block": block, "_offsets": offs}, {}
        for k, a, o in zip(self._COLUMNS, cols, offs):
            view = raw[o:o + a.nbytes].view(a.dtype)
            view[...] = a
            arrs[k] = view
            tens[k] = block[o:o + a.nbytes].view(torch.from_numpy(a[:0]).dtype)
        return ColumnarTrace(self.clock_domain, arrs["start"], arrs["dur"], arrs["pid"], arrs["tid"], arrs["cat"],
                             arrs["name"], arrs["corr"], arrs["has_corr"], self.pids, arrs["group_pid"],
                             self.group_tid, self.names, self.processes, arrs["pid_has_meta"], self._source, tens)

    # -- conversion back ------------------------------------------------------
    def pid_value(self, idx: int) -> int:
        return int(self.pids[idx])

    def to_events(self, start: Optional[np.ndarray] = None, dur: Optional[np.ndarray] = None) -> list:
        start = self.start if start is None else start
        dur = self.dur if dur is None else dur
        pid_v = self.pids[self.pid].tolist()
        tid_v = self.group_tid[self.tid].tolist()
        names = self.names
        nm = [names[i] for i in self.name.tolist()]
        cats = [Category(c) for c in range(6)]
        cat = [cats[c] for c in self.cat.tolist()]
        corr = [c if h else None for c, h in zip(self.corr.tolist(), self.has_corr.tolist())]
        return [Event(p, t, c, s_name, s, d, k) for p, t, c, s_name, s, d, k in
                zip(pid_v, tid_v, cat, nm, start.tolist(), dur.tolist(), corr)]

    def to_trace(self, start=None, dur=None, processes: Optional[Sequence[ProcessMeta]] = None) -> Trace:
        return Trace(self.clock_domain, self.to_events(start, dur),
                     self.processes if processes is None else processes)

    def select_pids(self, pid_indices) -> "ColumnarTrace":
        """Sub-trace holding only the given pid indices (keeps every table, so
        pid/tid/name indices stay valid); used for sharding."""
        keep = np.isin(self.pid, np.asarray(pid_indices, dtype=np.int32))
        return ColumnarTrace(self.clock_domain, self.start[keep], self.dur[keep], self.pid[keep],
                             self.tid[keep], self.cat[keep], self.name[keep], self.corr[keep],
                             self.has_corr[keep], self.pids, self.group_pid, self.group_tid,
                             self.names, self.processes, self.pid_has_meta)


# -- columns of Traces this package produced --------------------------------
# A Trace is immutable (frozen dataclass, events in a tuple), so the columns a
# correction produced stay valid for the Trace built from them:
# compute_overlap(correct_trace(t)[0]) -- the reference's call sequence
# (cli.py:168-171) -- then skips re-interning a million Event objects.
_PRODUCED: dict = {}


def remember_columnar(trace, ct: "ColumnarTrace") -> None:
    import weakref

    key = id(trace)
    _PRODUCED[key] = (weakref.ref(trace), ct)
    weakref.finalize(trace, _PRODUCED.pop, key, None)


def produced_columnar(trace) -> Optional["ColumnarTrace"]:
    hit = _PRODUCED.get(id(trace))
    if hit is not None and hit[0]() is trace:
        return hit[1]
    return None


# -- packed upload format (xs_packed_t) -------------------------------------
PACK_ROWS = 256  # rows per start base


def _index_width(a: np.ndarray) -> int:
    hi = int(a.max()) if a.size else 0
    return 1 if hi < 1 << 8 else 2 if hi < 1 << 16 else 4


def _fits_u32(a: np.ndarray) -> bool:
    return a.size == 0 or (int(a.min()) >= 0 and int(a.max()) < 1 << 32)


class PackedLayout:
    """Byte layout of a trace in the packed upload format: per column its
    width and offset in the block (16-byte aligned).  ``arrays`` holds the
    narrowed columns until ``fill`` copies them into the pinned block."""

    _INDEX = {1: np.uint8, 2: np.uint16, 4: np.int32}
    _WIDE = {4: np.uint32, 8: np.int64}

    def __init__(self, n: int, arrays: dict, widths: dict):
        self.n = n
        self.widths = widths
        self.arrays = arrays
        self.offsets, total = {}, 0
        for k, a in arrays.items():
            self.offsets[k] = total
            total += (a.nbytes + 15) // 16 * 16
        self.total = total
        self.nbytes = {k: a.nbytes for k, a in arrays.items()}
        self.n_exc = int(arrays["exc_row"].size)

    @classmethod
    def from_native(cls, nat) -> "PackedLayout":
        lay = cls.__new__(cls)
        lay.n = int(nat.n)
        lay.widths = {"start": nat.start_w, "dur": nat.dur_w, "corr": nat.corr_w, "pid": nat.pid_w,
                      "tid": nat.tid_w, "name": nat.name_w, "catf": 1}
        lay.arrays = None
        lay.offsets = {k: int(nat.offset[i]) for i, k in enumerate(_SECTIONS)}
        lay.nbytes = {k: int(nat.nbytes[i]) for i, k in enumerate(_SECTIONS)}
        lay.total = int(nat.total)
        lay.n_exc = int(nat.n_exc)
        return lay

    def fill(self, raw: np.ndarray) -> None:
        for k, a in self.arrays.items():
            o = self.offsets[k]
            raw[o:o + a.nbytes].view(a.dtype)[...] = a
        self.arrays = None  # (the block holds them now)

    def row_bytes(self, col: str) -> int:
        """Bytes per row of a per-row column."""
        return self.widths[col]


_EXC = 0xFFFFFFFF  # a 32-bit slot whose value sits in the exception table


def _narrow_u32(a: np.ndarray, fits: np.ndarray, n_max: int):
    """(uint32 column, exception rows) when all but <= n_max values fit."""
    bad = np.flatnonzero(~fits)
    if bad.size > n_max:
        return None
    return np.where(fits, a, _EXC).astype(np.uint32), bad


def _pack_layout(ct: "ColumnarTrace"):
    """The packed layout of ``ct``, or None when a column cannot be narrowed
    losslessly into the format (cat >= 128 or has_corr not 0/1).  start /
    dur / corr take 32 bits when at most 1/16 of their values need the
    exception table."""
    n = ct.n
    if n and (int(ct.cat.max()) >= 128 or int(ct.has_corr.max()) > 1):
        return None
    arrays, widths = {}, {}
    n_max = n // 16
    exc = []  # (rows, column id, exact values)
    s = ct.start
    got = None
    if n:
        base = np.minimum.reduceat(s, np.arange(0, n, PACK_ROWS))
        with np.errstate(over="ignore"):
            off = s - np.repeat(base, PACK_ROWS)[:n]
        got = _narrow_u32(off, (off >= 0) & (off < _EXC), n_max)
    if got is not None:
        arrays["start"], widths["start"] = got[0], 4
        arrays["start_base"] = base.astype(np.int64)
        exc.append((got[1], 0, s[got[1]]))
    else:
        arrays["start"], widths["start"] = np.ascontiguousarray(s, np.int64), 8
        arrays["start_base"] = np.zeros(1, np.int64)
    for cid, k in ((1, "dur"), (2, "corr")):
        a = getattr(ct, k)
        got = _narrow_u32(a, (a >= 0) & (a < _EXC), n_max)
        if got is not None:
            arrays[k], widths[k] = got[0], 4
            exc.append((got[1], cid, a[got[1]]))
        else:
            arrays[k], widths[k] = np.ascontiguousarray(a, np.int64), 8
    for k in ("pid", "tid", "name"):
        a = getattr(ct, k)
        w = _index_width(a)
        arrays[k], widths[k] = a.astype(PackedLayout._INDEX[w]), w
    arrays["catf"] = (ct.cat | (ct.has_corr.astype(np.uint8) << 7)).astype(np.uint8)
    widths["catf"] = 1
    arrays["group_pid"] = np.ascontiguousarray(ct.group_pid, np.int32)
    arrays["pid_has_meta"] = np.ascontiguousarray(ct.pid_has_meta, np.uint8)
    rows = np.concatenate([e[0] for e in exc]).astype(np.int64) if exc else np.zeros(0, np.int64)
    cols = np.concatenate([np.full(e[0].size, e[1], np.uint8) for e in exc]) if exc else np.zeros(0, np.uint8)
    vals = np.concatenate([e[2] for e in exc]).astype(np.int64) if exc else np.zeros(0, np.int64)
    order = np.argsort(rows, kind="stable")
    arrays["exc_row"], arrays["exc_val"], arrays["exc_col"] = rows[order], vals[order], cols[order]
    return PackedLayout(n, arrays, widths)


_SECTIONS = ("start", "start_base", "dur", "corr", "pid", "tid", "name", "catf", "group_pid", "pid_has_meta",
             "exc_row", "exc_val", "exc_col")  # xs_pack_layout_t section order


def _host_events(ct: "ColumnarTrace"):
    """xs_events_t over HOST column pointers (engine dtypes) + the arrays it references."""
    from . import _lib

    cols = [np.ascontiguousarray(getattr(ct, k), dt) for k, dt in
            (("start", np.int64), ("dur", np.int64), ("pid", np.int32), ("tid", np.int32), ("cat", np.uint8),
             ("name", np.int32), ("corr", np.int64), ("has_corr", np.uint8), ("group_pid", np.int32),
             ("pid_has_meta", np.uint8))]
    p = [a.ctypes.data if a.size else None for a in cols]
    ev = _lib.XsEvents(ct.n, *p[:8], ct.n_pids, ct.n_groups, len(ct.names), 0, p[8], p[9])
    return ev, cols


def pack_native(ct: "ColumnarTrace", alloc=None, n_threads: int = 0):
    """The packed block built by the native host builder (xs_pack_plan /
    xs_pack_fill, host threads; byte-identical to pack_block with zeroed
    padding).  ``alloc(nbytes)`` returns a writable uint8 numpy view (e.g. of
    a page-locked tensor) -- default: ordinary memory.  Returns (layout,
    block view) or None when the trace is not packable."""
    import ctypes as C

    from . import _lib

    lib = _lib.load()
    ev, keep = _host_events(ct)
    nat = _lib.XsPackLayout()
    st = lib.xs_pack_plan(C.byref(ev), int(n_threads), C.byref(nat))
    if st == _lib.XS_UNSUPPORTED:
        return None
    if st != 0:
        raise RuntimeError(f"xs_pack_plan: {lib.xs_status_str(st).decode()}")
    size = max(int(nat.total), 16)
    raw = alloc(size) if alloc is not None else np.empty(size, np.uint8)
    st = lib.xs_pack_fill(C.byref(ev), C.byref(nat), raw.ctypes.data, size)
    if st != 0:
        raise RuntimeError(f"xs_pack_fill: {lib.xs_status_str(st).decode()}")
    del keep
    return PackedLayout.from_native(nat), raw


def pack_block(ct: "ColumnarTrace"):
    """(layout, bytes) of ``ct`` in the packed upload format in ordinary host
    memory (ColumnarTrace.pinned puts the same bytes in a pinned block), or
    None when the trace cannot be packed."""
    lay = _pack_layout(ct)
    if lay is None:
        return None
    raw = np.zeros(max(lay.total, 16), np.uint8)
    lay.fill(raw)
    return lay, raw


def unpack_block(raw: np.ndarray, lay: PackedLayout, a: int = 0, b: Optional[int] = None) -> dict:
    """Host restatement of xs_unpack (tests): rows [a, b) of a packed block
    widened back to the engine's column dtypes."""
    b = lay.n if b is None else b

    def col(k, dt, lo, hi):
        o = lay.offsets[k]
        return raw[o:o + lay.nbytes[k]].view(dt)[lo:hi]

    w = lay.widths
    out = {}
    st = col("start", PackedLayout._WIDE[w["start"]], a, b).astype(np.int64)
    if w["start"] == 4:
        base = col("start_base", np.int64, 0, None)
        st = st + base[np.arange(a, b) // PACK_ROWS]
    out["start"] = st
    for k in ("dur", "corr"):
        out[k] = col(k, PackedLayout._WIDE[w[k]], a, b).astype(np.int64)
    for k in ("pid", "tid", "name"):
        out[k] = col(k, PackedLayout._INDEX[w[k]], a, b).astype(np.int32)
    cf = col("catf", np.uint8, a, b)
    out["cat"] = cf & 0x7F
    out["has_corr"] = cf >> 7
    rows = col("exc_row", np.int64, 0, None)
    sel = (rows >= a) & (rows < b)
    for r, c, v in zip(rows[sel], col("exc_col", np.uint8, 0, None)[sel], col("exc_val", np.int64, 0, None)[sel]):
        out[("start", "dur", "corr")[c]][r - a] = v
    return out
