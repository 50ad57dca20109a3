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
