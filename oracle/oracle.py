"""ctypes wrapper over ``libxs_oracle.so`` -- TEST INFRASTRUCTURE.

The CPU restatement of the reference path (see ``xs_oracle.c``).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker.
Results come back in the reference's observable shape:
``{(pid, path_names, frozenset(category ints)): ns}`` plus spans/untracked,
so they compare directly with golden vectors produced by the reference.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libxs_oracle.so")

_lib = None


class XoEvents(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("start", C.c_void_p), ("dur", C.c_void_p), ("pid", C.c_void_p), ("tid", C.c_void_p),
        ("cat", C.c_void_p), ("name", C.c_void_p), ("corr", C.c_void_p), ("has_corr", C.c_void_p),
        ("n_pids", C.c_int32), ("n_groups", C.c_int32), ("n_names", C.c_int32),
        ("pid_has_meta", C.c_void_p),
    ]


class XoOverlap(C.Structure):
    _fields_ = [
        ("n_cells", C.c_int64),
        ("cell_pid", C.POINTER(C.c_int32)), ("cell_node", C.POINTER(C.c_int32)),
        ("cell_mask", C.POINTER(C.c_int32)), ("cell_ns", C.POINTER(C.c_int64)),
        ("n_nodes", C.c_int32),
        ("node_parent", C.POINTER(C.c_int32)), ("node_name", C.POINTER(C.c_int32)),
        ("span_lo", C.POINTER(C.c_int64)), ("span_hi", C.POINTER(C.c_int64)),
        ("tracked", C.POINTER(C.c_int64)), ("has_events", C.POINTER(C.c_uint8)),
    ]


class XoProfile(C.Structure):
    _fields_ = [
        ("L", C.c_int64), ("ann_start", C.c_int64), ("ann_end", C.c_int64),
        ("transition", C.c_int64), ("interception", C.c_int64),
        ("internal", C.c_void_p), ("has_internal", C.c_void_p),
        ("residue_in", C.c_void_p), ("span_end_in", C.c_void_p),
    ]


class XoReport(C.Structure):
    _fields_ = [
        ("removed", C.c_void_p), ("shortfall", C.c_void_p),
        ("original_total", C.c_int64), ("corrected_total", C.c_int64), ("bad_event", C.c_int64),
    ]


def build() -> str:
    """Compile the oracle (``make -C oracle``)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
                os.path.join(HERE, "xs_oracle.c")):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.xo_validate_count.restype = C.c_int64
        _lib.xo_validate_count.argtypes = [C.POINTER(XoEvents)]
        _lib.xo_overlap.argtypes = [C.POINTER(XoEvents), C.c_int, C.POINTER(XoOverlap)]
        _lib.xo_free_overlap.argtypes = [C.POINTER(XoOverlap)]
        _lib.xo_transition_sites.argtypes = [C.POINTER(XoEvents), C.c_int, C.POINTER(C.c_int64),
                                             C.c_void_p, C.c_void_p]
        _lib.xo_correct.argtypes = [C.POINTER(XoEvents), C.POINTER(XoProfile), C.c_void_p, C.c_void_p,
                                    C.POINTER(XoReport), C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    return _lib


def _ptr(a):
    return a.ctypes.data if a.size else None


def _events(ct):
    keep = [ct.start, ct.dur, ct.pid, ct.tid, ct.cat, ct.name, ct.corr, ct.has_corr, ct.pid_has_meta]
    ev = XoEvents(ct.n, _ptr(ct.start), _ptr(ct.dur), _ptr(ct.pid), _ptr(ct.tid), _ptr(ct.cat),
                  _ptr(ct.name), _ptr(ct.corr), _ptr(ct.has_corr), ct.n_pids, ct.n_groups,
                  len(ct.names), _ptr(ct.pid_has_meta))
    return ev, keep


class OracleInvalid(Exception):
    pass


class OracleUncalibrated(Exception):
    def __init__(self, event_index):
        self.event_index = event_index
        super().__init__(f"uncalibrated API at event {event_index}")


def validate_count(ct) -> int:
    ev, _keep = _events(ct)
    return int(lib().xo_validate_count(C.byref(ev)))


def overlap(ct, attribution: int = 0):
    """compute_overlap restated; returns (cells, spans, untracked) keyed by pid value."""
    ev, _keep = _events(ct)
    out = XoOverlap()
    st = lib().xo_overlap(C.byref(ev), attribution, C.byref(out))
    if st == 1:
        raise OracleInvalid("invalid trace")
    if st != 0:
        raise RuntimeError(f"oracle overlap failed: {st}")
    try:
        parents = [out.node_parent[i] for i in range(out.n_nodes)]
        names = [out.node_name[i] for i in range(out.n_nodes)]
        paths = [()] * out.n_nodes
        for i in range(1, out.n_nodes):  # parents precede children
            paths[i] = paths[parents[i]] + (ct.names[names[i]],)
        cells = {}
        for k in range(out.n_cells):
            mask = out.cell_mask[k]
            cats = frozenset(c for c in range(1, 6) if mask & (1 << (c - 1)))
            key = (int(ct.pids[out.cell_pid[k]]), paths[out.cell_node[k]], cats)
            cells[key] = int(out.cell_ns[k])
        spans, untracked = {}, {}
        for p in range(ct.n_pids):
            if out.has_events[p]:
                pv = int(ct.pids[p])
                lo, hi = int(out.span_lo[p]), int(out.span_hi[p])
                spans[pv] = (lo, hi)
                untracked[pv] = (hi - lo) - int(out.tracked[p])
        return cells, spans, untracked
    finally:
        lib().xo_free_overlap(C.byref(out))


PAIRS = ((1, 2), (1, 3), (2, 4), (3, 4))


def transition_sites(ct, pair_mask: int = 0xF):
    ev, _keep = _events(ct)
    n = C.c_int64(0)
    op = np.zeros(max(ct.n, 1), np.int32)
    oe = np.zeros(max(ct.n, 1), np.int64)
    st = lib().xo_transition_sites(C.byref(ev), pair_mask, C.byref(n), op.ctypes.data, oe.ctypes.data)
    if st == 1:
        raise OracleInvalid("invalid trace")
    res = {PAIRS[k]: [] for k in range(4) if (pair_mask >> k) & 1}
    for k, e in zip(op[: n.value].tolist(), oe[: n.value].tolist()):
        res[PAIRS[k]].append(e)
    return res


def scale_profile(profile, names):
    """Exact rationals -> integers over one common denominator (oracle side)."""
    ann = Fraction(profile.annotation_ns)
    half = ann / 2
    base = [half, ann - half, Fraction(profile.transition_ns), Fraction(profile.api_interception_ns)]
    internal = {k: Fraction(v) for k, v in profile.api_internal_ns.items()}
    den = 1
    import math
    for v in base + list(internal.values()):
        den = den * v.denominator // math.gcd(den, v.denominator)
    ints = np.array([int(internal[n] * den) if n in internal else 0 for n in names], np.int64)
    has = np.array([n in internal for n in names], np.uint8)
    return den, [int(v * den) for v in base], ints, has


HOOKS = ("annotation", "transition", "api_interception", "api_internal")


def correct(ct, profile, queries=(), residue_in=None, span_end_in=None, arrays=False):
    """correct_trace restated; returns (start', dur', report dict, query results).
    ``residue_in`` ([n_pids] Fractions in [0, 1)) and ``span_end_in``
    ([n_pids] ints) are the window carries of the sharded window correction
    (None: the reference's whole-process semantics)."""
    ev, _keep = _events(ct)
    L, base, ints, has = scale_profile(profile, ct.names)
    res = spe = None
    if residue_in is not None:
        res = np.array([int(r * L) for r in residue_in], np.int64)
        assert all(int(r * L) == r * L and 0 <= r < 1 for r in residue_in)
    if span_end_in is not None:
        spe = np.ascontiguousarray(span_end_in, np.int64)
    prof = XoProfile(L, base[0], base[1], base[2], base[3], _ptr(ints) if ints.size else None,
                     _ptr(has) if has.size else None, _ptr(res) if res is not None else None,
                     _ptr(spe) if spe is not None else None)
    P = ct.n_pids
    removed = np.zeros(max(P, 1) * 4, np.int64)
    shortfall = np.zeros(max(P, 1) * 4, np.int64)
    rep = XoReport(removed.ctypes.data, shortfall.ctypes.data, 0, 0, -1)
    out_s = np.zeros(max(ct.n, 1), np.int64)
    out_d = np.zeros(max(ct.n, 1), np.int64)
    q_pid = np.array([q[0] for q in queries] or [0], np.int32)
    q_val = np.array([q[1] for q in queries] or [0], np.int64)
    q_out = np.zeros_like(q_val)
    st = lib().xo_correct(C.byref(ev), C.byref(prof), out_s.ctypes.data, out_d.ctypes.data, C.byref(rep),
                          len(queries), q_pid.ctypes.data, q_val.ctypes.data, q_out.ctypes.data)
    if st == 1:
        raise OracleInvalid("invalid trace")
    if st == 2:
        raise OracleUncalibrated(int(rep.bad_event))
    if st != 0:
        raise RuntimeError(f"oracle correct failed: {st}")
    if arrays:  # per pid index: (start', dur', removed [P, 4], shortfall [P, 4], query results)
        return (out_s[: ct.n], out_d[: ct.n], removed[: P * 4].reshape(P, 4), shortfall[: P * 4].reshape(P, 4),
                q_out[: len(queries)].tolist())
    present = np.zeros(P, bool)
    present[np.unique(ct.pid)] = True
    report = {
        "removed_ns": {int(ct.pids[p]): dict(zip(HOOKS, removed[p * 4:(p + 1) * 4].tolist()))
                       for p in range(P) if present[p]},
        "shortfall_ns": {int(ct.pids[p]): dict(zip(HOOKS, shortfall[p * 4:(p + 1) * 4].tolist()))
                         for p in range(P) if present[p]},
        "original_total_ns": int(rep.original_total),
        "corrected_total_ns": int(rep.corrected_total),
    }
    return out_s[: ct.n], out_d[: ct.n], report, q_out[: len(queries)].tolist()


# ---------------------------------------------------------------------------
# metrics (numpy restatement; test infrastructure only)

def union_ns(ct, category: int, per_pid: bool = False):
    """metrics._union_ns (metrics.py:41-58): sort (start, end) of the
    category's nonzero events, merge overlapping/touching, sum lengths --
    trace-wide, or {pid value: ns} per pid (procview.py:75)."""
    sel = (ct.cat == category) & (ct.dur > 0)
    groups = [(None, sel)] if not per_pid else [(int(ct.pids[p]), sel & (ct.pid == p)) for p in range(ct.n_pids)]
    out = {}
    for key, m in groups:
        s = ct.start[m]
        e = s + ct.dur[m]
        order = np.lexsort((e, s))
        total, cur_lo, cur_hi = 0, None, 0
        for lo, hi in zip(s[order].tolist(), e[order].tolist()):
            if cur_lo is None:
                cur_lo, cur_hi = lo, hi
            elif lo <= cur_hi:
                cur_hi = max(cur_hi, hi)
            else:
                total += cur_hi - cur_lo
                cur_lo, cur_hi = lo, hi
        if cur_lo is not None:
            total += cur_hi - cur_lo
        out[key] = total
    return out[None] if not per_pid else out


def trace_span(ct):
    if ct.n == 0:
        return None
    return int(ct.start.min()), int((ct.start + ct.dur).max())


def utilization_flags(ct, period_ns: int):
    """metrics.utilization_samples (metrics.py:61-79): per period, does it
    intersect a nonzero-duration GPU event (the reference's two-pointer walk)."""
    lo, hi = trace_span(ct)
    sel = (ct.cat == 5) & (ct.dur > 0)
    s = ct.start[sel]
    e = s + ct.dur[sel]
    order = np.lexsort((e, s))
    gpu = list(zip(s[order].tolist(), e[order].tolist()))
    flags, idx, start = [], 0, lo
    while start < hi:
        while idx < len(gpu) and gpu[idx][1] <= start:
            idx += 1
        flags.append(idx < len(gpu) and gpu[idx][0] < start + period_ns)
        start += period_ns
    return flags
