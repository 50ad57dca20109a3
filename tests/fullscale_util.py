"""Full-scale parity checking (TEST INFRASTRUCTURE).

The device result of one call over a whole BASELINE-size trace is compared
with two CPU checkers, pid by pid in a fork process pool (per-pid results are
independent: overlap.py:126, correction.py:132, so a pid's oracle result over
the sub-trace of its events is exactly its share of the whole-trace result):

* the C restatement (oracle/xs_oracle.c) on EVERY pid: corrected start/dur
  columns, CorrectionReport rows, and compute_overlap(corrected) cells /
  spans / untracked;
* the reference itself (oracle/_ref, the unmodified xstrace package built by
  oracle/build_ref.sh) on a sample of pids, through its own public API:
  correct_trace(Trace, CalibrationProfile) then compute_overlap(corrected)
  (cli.py:168-171).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")

def have_reference() -> bool:
    return os.path.isdir(os.path.join(REF, "xstrace"))


def pid_bounds(ct) -> np.ndarray:
    """Row ranges of each pid index (rows are pid-contiguous in every
    generated trace; asserted)."""
    assert ct.n == 0 or np.all(np.diff(ct.pid) >= 0), "rows must be grouped by pid"
    return np.searchsorted(ct.pid, np.arange(ct.n_pids + 1, dtype=np.int32))


def sub_trace(ct, pids, bounds):
    from paper_2102_04285_b200 import ColumnarTrace
    rows = np.concatenate([np.arange(bounds[p], bounds[p + 1]) for p in pids]) if pids else np.zeros(0, np.int64)
    cols = [getattr(ct, k)[rows] for k in ("start", "dur", "pid", "tid", "cat", "name", "corr", "has_corr")]
    return ColumnarTrace(ct.clock_domain, *cols, ct.pids, ct.group_pid, ct.group_tid, ct.names, ct.processes,
                         ct.pid_has_meta), rows


def cells_by_pid(bd) -> dict:
    """{pid value: {(path, frozenset(cat ints)): ns}} of a Breakdown."""
    out: dict = {}
    for k, v in bd.cells.items():
        out.setdefault(k.pid, {})[(k.path, frozenset(int(c) for c in k.categories))] = v
    return out


def _oracle_worker(job):
    """One pid batch vs the C oracle (runs in a spawned process: everything
    it needs arrives in ``job``)."""
    import oracle
    from paper_2102_04285_b200 import ColumnarTrace
    sub, prof, rows, pids = job["sub"], job["profile"], job["rows"], job["pids"]
    errs = []
    if prof is not None:
        s, d, rep, _ = oracle.correct(sub, prof)
        if not (np.array_equal(job["start"], s) and np.array_equal(job["dur"], d)):
            bad = np.flatnonzero((job["start"] != s) | (job["dur"] != d))
            errs.append(f"pids {pids}: corrected columns differ at {len(bad)} rows, first row {rows[bad[0]]}")
        for pv, hooks in rep["removed_ns"].items():
            if job["removed"].get(pv) != hooks:
                errs.append(f"pid {pv}: removed_ns {job['removed'].get(pv)} != oracle {hooks}")
        for pv, hooks in rep["shortfall_ns"].items():
            if job["shortfall"].get(pv) != hooks:
                errs.append(f"pid {pv}: shortfall_ns {job['shortfall'].get(pv)} != oracle {hooks}")
        sub = ColumnarTrace(sub.clock_domain, s, d, sub.pid, sub.tid, sub.cat, sub.name, sub.corr, sub.has_corr,
                            sub.pids, sub.group_pid, sub.group_tid, sub.names, sub.processes, sub.pid_has_meta)
    cells, spans, untracked = oracle.overlap(sub, job["attribution"])
    per: dict = {}
    for (pv, path, cats), ns in cells.items():
        per.setdefault(pv, {})[(path, cats)] = ns
    for pv in pids:
        if per.get(pv, {}) != job["cells"].get(pv, {}):
            errs.append(f"pid {pv}: {len(job['cells'].get(pv, {}))} cells vs oracle {len(per.get(pv, {}))}, differ")
        if spans.get(pv) != job["spans"].get(pv) or untracked.get(pv) != job["untracked"].get(pv):
            errs.append(f"pid {pv}: span/untracked {job['spans'].get(pv)}/{job['untracked'].get(pv)} vs oracle "
                        f"{spans.get(pv)}/{untracked.get(pv)}")
    return errs


def _job(ct, bounds, pid_idx, bd_cells, bd, profile, start, dur, report, attribution):
    sub, rows = sub_trace(ct, pid_idx, bounds)
    pvs = [int(ct.pids[p]) for p in pid_idx]
    job = {"sub": sub, "rows": rows, "pids": pvs, "profile": profile, "attribution": attribution,
           "cells": {pv: bd_cells.get(pv, {}) for pv in pvs},
           "spans": {pv: bd.spans.get(pv) for pv in pvs}, "untracked": {pv: bd.untracked.get(pv) for pv in pvs}}
    if profile is not None:
        job.update(start=np.asarray(start)[rows], dur=np.asarray(dur)[rows],
                   removed={pv: report.removed_ns.get(pv) for pv in pvs},
                   shortfall={pv: report.shortfall_ns.get(pv) for pv in pvs})
    return job


def _pool(n):
    # spawned workers: forking a process that holds a CUDA context and
    # helper threads can deadlock or abort the child
    return mp.get_context("spawn").Pool(max(1, n))


def _batches(ct, bounds, max_events: int) -> list:
    sizes = np.diff(bounds)
    out, cur, tot = [], [], 0
    for p in range(ct.n_pids):
        if sizes[p] == 0:
            continue
        if cur and tot + sizes[p] > max_events:
            out.append(cur)
            cur, tot = [], 0
        cur.append(p)
        tot += int(sizes[p])
    if cur:
        out.append(cur)
    return out


def oracle_check(ct, bd, profile=None, start=None, dur=None, report=None, attribution: int = 0,
                 workers: int = 0, max_events: int = 2_000_000) -> list:
    """Every pid of the device result vs the C oracle; returns mismatches."""
    bounds = pid_bounds(ct)
    cells = cells_by_pid(bd)
    jobs = [_job(ct, bounds, j, cells, bd, profile, start, dur, report, attribution)
            for j in _batches(ct, bounds, max_events)]
    workers = workers or min(len(jobs), os.cpu_count() or 1)
    if workers <= 1:
        res = [_oracle_worker(j) for j in jobs]
    else:
        with _pool(min(workers, len(jobs))) as pool:
            res = pool.map(_oracle_worker, jobs, chunksize=1)
    return [e for r in res for e in r]


# ---------------------------------------------------------------------------
def _ref_worker(job):
    sys.path.insert(0, REF)
    from xstrace import model as RM
    from xstrace.calibration import CalibrationProfile as RP
    from xstrace.correction import correct_trace as ref_correct
    from xstrace.overlap import compute_overlap as ref_overlap

    sub, prof = job["sub"], job["profile"]
    (pv,) = job["pids"]
    cats = [RM.Category(c) for c in range(6)]
    names = sub.names
    events = [RM.Event(int(sub.pids[p]), int(sub.group_tid[t]), cats[c], names[nm], s, d, k if h else None)
              for p, t, c, nm, s, d, k, h in zip(sub.pid.tolist(), sub.tid.tolist(), sub.cat.tolist(),
                                                 sub.name.tolist(), sub.start.tolist(), sub.dur.tolist(),
                                                 sub.corr.tolist(), sub.has_corr.tolist())]
    metas = [RM.ProcessMeta(m.pid, m.name, m.parent, m.fork_ns, m.join_ns) for m in sub.processes]
    trace = RM.Trace(sub.clock_domain, events, metas)
    errs = []
    if prof is not None:
        rp = RP(prof.annotation_ns, prof.transition_ns, prof.api_interception_ns, dict(prof.api_internal_ns))
        out, rep = ref_correct(trace, rp)
        rs = np.fromiter((e.start for e in out.events), np.int64, len(out.events))
        rd = np.fromiter((e.duration for e in out.events), np.int64, len(out.events))
        if not (np.array_equal(rs, job["start"]) and np.array_equal(rd, job["dur"])):
            errs.append(f"pid {pv}: corrected columns differ from the reference")
        if dict(rep.removed_ns.get(pv, {})) != job["removed"].get(pv) or \
                dict(rep.shortfall_ns.get(pv, {})) != job["shortfall"].get(pv):
            errs.append(f"pid {pv}: report rows differ from the reference")
        trace = out
    bd = ref_overlap(trace)
    cells = {(tuple(k.path), frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items()}
    if cells != job["cells"].get(pv, {}):
        errs.append(f"pid {pv}: cells differ from the reference ({len(cells)} vs {len(job['cells'].get(pv, {}))})")
    if bd.spans.get(pv) != job["spans"].get(pv) or bd.untracked.get(pv) != job["untracked"].get(pv):
        errs.append(f"pid {pv}: span/untracked differ from the reference")
    return errs, len(events)


def reference_check(ct, bd, pid_indices, profile=None, start=None, dur=None, report=None) -> tuple:
    """Sampled pids of the device result vs the unmodified reference;
    returns (mismatches, events checked)."""
    bounds = pid_bounds(ct)
    cells = cells_by_pid(bd)
    jobs = [_job(ct, bounds, [p], cells, bd, profile, start, dur, report, 0) for p in pid_indices]
    with _pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        res = pool.map(_ref_worker, jobs, chunksize=1)
    return [e for r, _ in res for e in r], sum(n for _, n in res)
