"""Derived metrics: busy fractions, sampled utilization, report rows (drop-in
for ``pkg/src/xstrace/metrics.py``).

Same names, signatures, return types and errors as the reference.  The
interval unions run on the GPU (``xs_union`` / ``xs_utilization`` in
``csrc/xs_metrics.cu``): one endpoint sort + coverage prefix sum replaces the
reference's Python ``sorted`` + merge loop (metrics.py:41-58, 61-84).
``summarize`` is a pure function of a ``Breakdown`` and stays on the host.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _engine
from .columnar import ColumnarTrace
from .model import Category, require_valid
from .overlap import Breakdown, OverlapKey


@dataclass(frozen=True)
class UtilizationSample:
    """One sampler period; lengths tile the span without overlap (metrics.py:21-27)."""

    period_start: int
    period_ns: int
    utilized: bool


def _device(trace):
    ct = trace if isinstance(trace, ColumnarTrace) else ColumnarTrace.from_trace(trace)
    eng = _engine.get()
    return eng, _engine.DeviceTrace(ct, eng.device)


def _check_span(lo: int, hi: int) -> tuple:
    """metrics._trace_span (metrics.py:30-38) from the device span reduction."""
    if lo > hi:
        raise ValueError("no span: trace has no events")
    if hi <= lo:
        raise ValueError("no span: trace covers zero nanoseconds")
    return lo, hi


def _union_ns(trace, category: Category) -> int:
    """Union length of one category's nonzero-duration intervals, all pids
    together (metrics.py:41-58)."""
    eng, dt = _device(trace)
    out, _, _ = eng.union(dt, int(category), per_pid=False)
    return int(out[0])


def union_ns_per_pid(trace, category: Category) -> dict:
    """{pid: union ns} of one category, each pid on its own (the per-process
    ``_union_ns(sub, GPU)`` of procview.py:75) in one device call."""
    eng, dt = _device(trace)
    out, _, _ = eng.union(dt, int(category), per_pid=True)
    pids = dt.ct.pids.tolist()
    return {pids[p]: int(out[p]) for p in range(len(pids))}


def _utilization(trace, period_ns: int, intervals: bool):
    if period_ns <= 0:
        raise ValueError(f"period_ns must be > 0, got {period_ns}")
    require_valid(trace)
    eng, dt = _device(trace)
    res = eng.utilization(dt, period_ns, intervals=intervals)
    lo, hi = _check_span(res[1], res[2])
    n_periods = -(-(hi - lo) // period_ns)
    return res, lo, hi, n_periods


def utilization_samples(trace, period_ns: int) -> list:
    """Fixed-cadence sampler periods anchored at the trace's earliest
    timestamp; the final partial period still counts (metrics.py:61-79)."""
    (util, _, _, ilo, ihi), lo, hi, k = _utilization(trace, period_ns, True)
    starts = lo + period_ns * np.arange(k, dtype=np.int64)
    lengths = np.minimum(starts + period_ns, hi) - starts
    mark = np.zeros(k + 1, np.int64)
    if ilo.size:
        np.add.at(mark, (ilo - lo) // period_ns, 1)
        np.add.at(mark, (ihi - 1 - lo) // period_ns + 1, -1)
    used = np.cumsum(mark[:k]) > 0
    assert int(used.sum()) == util
    return [UtilizationSample(s, n, u) for s, n, u in zip(starts.tolist(), lengths.tolist(), used.tolist())]


def sampled_utilization(trace, period_ns: int) -> float:
    """Utilized periods / total periods; the coarse-monitor estimate (metrics.py:82-85)."""
    (util, _, _), _, _, k = _utilization(trace, period_ns, False)
    return util / k


def busy_fraction(trace, category: Category) -> float:
    """Union time of one category's intervals divided by the trace span (metrics.py:87-91)."""
    require_valid(trace)
    eng, dt = _device(trace)
    out, lo, hi = eng.union(dt, int(category), per_pid=False)
    lo, hi = _check_span(lo, hi)
    return int(out[0]) / (hi - lo)


@dataclass(frozen=True)
class ReportRow:
    pid: int
    path: tuple
    categories: Optional[frozenset]  # None marks the untracked residual
    ns: int
    percent: float

    def labels(self) -> tuple:
        if self.categories is None:
            return ("-", "untracked")
        key = OverlapKey(self.pid, self.path, self.categories)
        return (key.path_label(), key.category_label())


def summarize(breakdown: Breakdown) -> list:
    """Report-ready rows: ns and percent of pid span, largest first, with the
    per-pid residual labeled untracked (metrics.py:107-126)."""
    by_pid: dict = {}
    for key, ns in breakdown.cells.items():
        by_pid.setdefault(key.pid, []).append((key, ns))
    rows = []
    for pid in sorted(breakdown.spans):
        span = breakdown.span_ns(pid)
        cells = sorted(by_pid.get(pid, ()), key=lambda kv: (-kv[1], kv[0].path, kv[0].category_label()))
        for key, ns in cells:
            rows.append(ReportRow(pid, key.path, key.categories, ns, (100.0 * ns / span) if span else 0.0))
        untracked = breakdown.untracked.get(pid, 0)
        if untracked:
            rows.append(ReportRow(pid, (), None, untracked, (100.0 * untracked / span) if span else 0.0))
    return rows
