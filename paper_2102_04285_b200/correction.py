"""Overhead correction by timeline surgery (drop-in for
``pkg/src/xstrace/correction.py``).

``correct_trace`` keeps the reference's signature, output and errors; the
pipeline (transition sites, hook sites, exact rational quantization, budget
caps, the (max,+) RemovalMap scan and the per-event remap) runs on the GPU
(csrc/xs_correct.cu).  ``correct_trace_columnar`` and ``analyze_columnar``
are the columnar fast paths (the latter is ``xstrace analyze --profile``:
correction followed by overlap of the corrected trace, cli.py:168-171).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from types import SimpleNamespace
from typing import Optional

import numpy as np

from . import _engine, _lib, _split
from .calibration import HOOK_KINDS, CalibrationProfile
from .columnar import ColumnarTrace, remember_columnar
from .model import Event, InvalidTraceError, ProcessMeta, Trace, format_violations, meta_violations


class UncalibratedHookError(ValueError):
    """The trace contains a hook kind the profile does not cover (correction.py:38-39)."""


@dataclass
class CorrectionReport:
    """Accounting for one correction pass (correction.py:42-60)."""

    removed_ns: dict = field(default_factory=dict)
    shortfall_ns: dict = field(default_factory=dict)
    original_total_ns: int = 0
    corrected_total_ns: int = 0
    bias: Optional[float] = None

    def removed_total(self, pid: Optional[int] = None) -> int:
        pids = [pid] if pid is not None else list(self.removed_ns)
        return sum(sum(self.removed_ns[p].values()) for p in pids)


def correction_bias(corrected_total: int, uninstrumented_total: int) -> float:
    """Signed deviation of the corrected total from uninstrumented reality (correction.py:63-67)."""
    if uninstrumented_total <= 0:
        raise ValueError(f"uninstrumented_total must be > 0, got {uninstrumented_total}")
    return (corrected_total - uninstrumented_total) / uninstrumented_total


def _source(trace, ct):
    if not isinstance(trace, ColumnarTrace):
        return trace
    return ct._source if ct._source is not None else ct.to_trace()


def _run(ct: ColumnarTrace, profile: CalibrationProfile, src, attribution: Optional[int] = None,
         device_trace=None, host_out=None):
    if meta_violations(ct.processes):
        raise InvalidTraceError(format_violations(_source(src, ct)))
    scaled = profile.scaled(ct.names)
    eng = _engine.get()
    dt = device_trace if device_trace is not None else _engine.DeviceTrace(ct, eng.device)
    try:
        raw = eng.correct(dt, scaled, attribution, host_out=host_out)
    except _engine.UncalibratedEvent as exc:
        name = ct.names[int(ct.name[exc.index])]
        raise UncalibratedHookError(f"uncalibrated hook: API_INTERNAL({name!r}) missing from profile") from None
    except _engine.XsError as exc:
        if exc.status == _lib.XS_INVALID_TRACE:
            raise InvalidTraceError(format_violations(_source(src, ct))) from None
        raise
    return eng, dt, raw


def _report(ct: ColumnarTrace, raw) -> CorrectionReport:
    rep = CorrectionReport()
    present = ct.present_pid_mask()
    pids = ct.pids.tolist()
    for p in range(ct.n_pids):
        if present[p]:
            rep.removed_ns[pids[p]] = dict(zip(HOOK_KINDS, raw.removed[p].tolist()))
            rep.shortfall_ns[pids[p]] = dict(zip(HOOK_KINDS, raw.shortfall[p].tolist()))
    rep.original_total_ns = raw.original_total
    rep.corrected_total_ns = raw.corrected_total
    return rep


def _remap_processes(eng, ct: ColumnarTrace) -> tuple:
    present = set(np.nonzero(ct.present_pid_mask())[0].tolist())
    pid_index = {int(p): i for i, p in enumerate(ct.pids.tolist())}
    q_pid, q_val, slots = [], [], []
    for k, m in enumerate(ct.processes):
        idx = pid_index.get(m.pid)
        if idx is None or idx not in present:
            continue
        for which, v in (("fork_ns", m.fork_ns), ("join_ns", m.join_ns)):
            if v is not None:
                q_pid.append(idx)
                q_val.append(v)
                slots.append((k, which))
    out = eng.remap(np.array(q_pid, np.int32), np.array(q_val, np.int64)) if q_val else []
    new = {}
    for (k, which), v in zip(slots, list(out)):
        new.setdefault(k, {})[which] = int(v)
    procs = []
    for k, m in enumerate(ct.processes):
        if k in new:
            procs.append(ProcessMeta(m.pid, m.name, m.parent, new[k].get("fork_ns", m.fork_ns),
                                     new[k].get("join_ns", m.join_ns)))
        else:
            procs.append(m)
    return tuple(procs)


def _batched(ct: ColumnarTrace, profile: CalibrationProfile, src, attribution: Optional[int]):
    """correct_trace (+ compute_overlap of the corrected trace when
    ``attribution`` is given) over pid batches (_split: more rows than one
    call takes, or keys wider than 64 bits over all pids).  Exact: sites,
    quantization, slabs and the removal map are per pid (correction.py:132-157).
    Errors keep the whole-trace semantics: any invalid batch raises the whole
    trace's violations; otherwise the uncalibrated hook of the smallest row.
    Returns (start, dur, report, processes, Breakdown or None)."""
    from .overlap import decode_breakdown, merge_breakdowns

    if meta_violations(ct.processes):
        raise InvalidTraceError(format_violations(_source(src, ct)))
    eng = _engine.get()
    rows_by_pid = _split.pid_rows(ct)
    start = np.empty(ct.n, np.int64)
    dur = np.empty(ct.n, np.int64)
    rep = CorrectionReport()
    procs = {}
    parts, errs = [], []
    todo = list(reversed(_split.plan_batches(ct)))
    while todo:
        pids = todo.pop()
        if len(pids) == 1 and rows_by_pid[pids[0]].shape[0] > _split.MAX_EVENTS_PER_CALL:
            try:  # one process larger than a call: its time windows, call by call, with the carries
                r, s_, d_, r_rep, r_bd, r_procs = _huge_process(ct, pids[0], rows_by_pid, profile, attribution, eng)
            except InvalidTraceError:
                errs.append(_BatchError("invalid", int(rows_by_pid[pids[0]][0])))
                continue
            except UncalibratedHookError:
                from .distributed import _first_uncalibrated_row
                sub, rows = _split.sub_trace(ct, pids, rows_by_pid)
                errs.append(_BatchError("uncalibrated", _first_uncalibrated_row(sub, profile, rows)))
                continue
            start[r], dur[r] = s_, d_
            rep.removed_ns.update(r_rep.removed_ns)
            rep.shortfall_ns.update(r_rep.shortfall_ns)
            rep.original_total_ns += r_rep.original_total_ns
            rep.corrected_total_ns += r_rep.corrected_total_ns
            procs.update(r_procs)
            if attribution is not None:
                parts.append(r_bd)
            continue
        sub, rows = _split.sub_trace(ct, pids, rows_by_pid)
        scaled = profile.scaled(sub.names)
        try:
            raw = eng.correct(_engine.DeviceTrace(sub, eng.device), scaled, attribution)
        except _engine.UncalibratedEvent as exc:
            errs.append(_BatchError("uncalibrated", int(rows[exc.index])))
            continue
        except _engine.XsError as exc:
            if exc.status == _lib.XS_INVALID_TRACE:
                errs.append(_BatchError("invalid", int(rows[0])))
                continue
            if exc.status == _lib.XS_UNSUPPORTED and len(pids) > 1:  # (CORRELATION keys also hold path bits)
                h = len(pids) // 2
                todo += [pids[h:], pids[:h]]
                continue
            raise
        if attribution is not None:
            parts.append(decode_breakdown(sub, eng.fetch_overlap(), lazy=False))
        start[rows] = raw.start.cpu().numpy()
        dur[rows] = raw.dur.cpu().numpy()
        r = _report(sub, raw)
        rep.removed_ns.update(r.removed_ns)
        rep.shortfall_ns.update(r.shortfall_ns)
        rep.original_total_ns += r.original_total_ns
        rep.corrected_total_ns += r.corrected_total_ns
        live = set(sub.pids.tolist())
        for k, m in enumerate(_remap_processes(eng, sub)):
            if m.pid in live:
                procs[k] = m
    if errs:
        if any(e.kind == "invalid" for e in errs):
            raise InvalidTraceError(format_violations(_source(src, ct)))
        first = min(errs, key=lambda e: e.row)
        name = ct.names[int(ct.name[first.row])]
        raise UncalibratedHookError(f"uncalibrated hook: API_INTERNAL({name!r}) missing from profile")
    processes = tuple(procs.get(k, m) for k, m in enumerate(ct.processes))
    return start, dur, rep, processes, (merge_breakdowns(parts) if attribution is not None else None)


def _huge_process(ct: ColumnarTrace, p: int, rows_by_pid, profile: CalibrationProfile, attribution, eng):
    """correct_trace (+ overlap) of ONE process holding more rows than a
    device call takes: cut into time windows of about half a call and run
    window by window on this GPU with the window carries (quantize residue,
    slab-length prefix; distributed._analyze_windows).  Exact; raises
    XsError(XS_UNSUPPORTED) when the process has no usable cuts.  Returns
    (rows, start, dur, report, Breakdown, {process index: ProcessMeta})."""
    import torch

    from .distributed import SequentialWindowRunner, _analyze_windows

    sub, rows = _split.sub_trace(ct, [p], rows_by_pid)
    max_rows = _split.MAX_EVENTS_PER_CALL
    split = -(-sub.n // max(1, max_rows // 2))
    pv = int(ct.pids[p])
    qs, slots = [], []
    for k, m in enumerate(ct.processes):
        if m.pid == pv:
            for which in ("fork_ns", "join_ns"):
                if getattr(m, which) is not None:
                    qs.append((0, int(getattr(m, which))))
                    slots.append((k, which))
    qout: list = []
    out = _analyze_windows(sub, profile, 0 if attribution is None else attribution,
                           torch.device("cuda", eng.device), 1, 0, split, SequentialWindowRunner(eng),
                           queries=qs, query_out=qout, max_rows=max_rows)
    if out is None:
        raise _engine.XsError(_lib.XS_UNSUPPORTED, f"process {pv} has more than {max_rows} events and no time "
                                                   "window cuts that keep every window below that")
    r, s_, d_, rep, bd = out
    new: dict = {}
    for (k, which), v in zip(slots, qout):
        new.setdefault(k, {})[which] = v
    procs = {k: ProcessMeta(m.pid, m.name, m.parent, new.get(k, {}).get("fork_ns", m.fork_ns),
                            new.get(k, {}).get("join_ns", m.join_ns))
             for k, m in enumerate(ct.processes) if m.pid == pv}
    return rows[r], s_, d_, rep, bd, procs


def _span_total(pid: np.ndarray, start: np.ndarray, end: np.ndarray, n_pids: int) -> int:
    lo = np.full(n_pids, np.iinfo(np.int64).max, np.int64)
    hi = np.full(n_pids, np.iinfo(np.int64).min, np.int64)
    np.minimum.at(lo, pid, start)
    np.maximum.at(hi, pid, end)
    m = hi >= lo
    return int(sum(int(h) - int(l) for l, h in zip(lo[m].tolist(), hi[m].tolist())))


def _correct_wide(ct: ColumnarTrace, profile: CalibrationProfile, src, attribution: Optional[int]):
    """correct_trace (+ compute_overlap of the result) for a trace holding a
    process too wide for one call's keys (>= 2^59 ns): exact gap compression
    (_split.compress_wide), the device correction of the compressed trace,
    the columns shifted back; the overlap of the corrected trace goes through
    operation-free time windows.  Returns what _batched returns."""
    wide = _split.wide_pids(ct)
    try:
        ctc, comp = _split.compress_wide(ct, wide, profile)
    except ValueError as exc:
        raise _engine.XsError(_lib.XS_UNSUPPORTED, f"xs_correct: unsupported input {exc}") from None
    try:
        start_c, dur_c, rep, procs_c, _ = _batched(ctc, profile, ctc, None)
    except InvalidTraceError:
        raise InvalidTraceError(format_violations(_source(src, ct))) from None
    start, dur = _split.uncompress_columns(ct, comp, start_c, dur_c)
    pid_index = {int(v): i for i, v in enumerate(ct.pids.tolist())}
    procs = []
    for m0, m in zip(ct.processes, procs_c):
        p = pid_index.get(m0.pid)
        if p in comp.points:
            def back(t0, t1):
                if t0 is None:
                    return None
                _, off, tail = comp.compress_time(p, t0)
                return int(t1) + off + tail
            m = ProcessMeta(m.pid, m.name, m.parent, back(m0.fork_ns, m.fork_ns), back(m0.join_ns, m.join_ns))
        procs.append(m)
    rep.original_total_ns = _span_total(ct.pid, ct.start, ct.start + ct.dur, ct.n_pids)
    rep.corrected_total_ns = _span_total(ct.pid, start, start + dur, ct.n_pids)
    bd = None
    if attribution is not None:
        from .overlap import Attribution, compute_overlap_columnar

        out = ColumnarTrace(ct.clock_domain, start, dur, ct.pid, ct.tid, ct.cat, ct.name, ct.corr, ct.has_corr,
                            ct.pids, ct.group_pid, ct.group_tid, ct.names, tuple(procs), ct.pid_has_meta)
        bd = compute_overlap_columnar(out, Attribution.CORRELATION if attribution == 1 else Attribution.INSTANT)
    return start, dur, rep, tuple(procs), bd


def correct_trace_columnar(ct: ColumnarTrace, profile: CalibrationProfile, device_trace=None,
                           _src=None) -> tuple:
    """Columnar correct_trace: returns (corrected ColumnarTrace, CorrectionReport)."""
    if device_trace is None and _split.needs_split(ct):
        start, dur, rep, procs, _ = _batched(ct, profile, _src if _src is not None else ct, None)
        out = ColumnarTrace(ct.clock_domain, start, dur, ct.pid, ct.tid, ct.cat, ct.name, ct.corr, ct.has_corr,
                            ct.pids, ct.group_pid, ct.group_tid, ct.names, procs, ct.pid_has_meta)
        return out, rep
    try:
        eng, dt, raw = _run(ct, profile, _src if _src is not None else ct, None, device_trace)
    except _engine.XsError as exc:
        if exc.status != _lib.XS_UNSUPPORTED or device_trace is not None:
            raise
        if _split.wide_pids(ct):
            start, dur, rep, procs, _ = _correct_wide(ct, profile, _src if _src is not None else ct, None)
        elif ct.n_pids < 2:
            raise
        else:
            start, dur, rep, procs, _ = _batched(ct, profile, _src if _src is not None else ct, None)
        return ColumnarTrace(ct.clock_domain, start, dur, ct.pid, ct.tid, ct.cat, ct.name, ct.corr, ct.has_corr,
                             ct.pids, ct.group_pid, ct.group_tid, ct.names, procs, ct.pid_has_meta), rep
    procs = _remap_processes(eng, ct)
    start = raw.start.cpu().numpy()
    dur = raw.dur.cpu().numpy()
    out = ColumnarTrace(ct.clock_domain, start, dur, ct.pid, ct.tid, ct.cat, ct.name, ct.corr, ct.has_corr,
                        ct.pids, ct.group_pid, ct.group_tid, ct.names, procs, ct.pid_has_meta)
    return out, _report(ct, raw)


def correct_trace(trace, profile: CalibrationProfile) -> tuple:
    """Remove calibrated overhead at every hook site; returns (trace, report).

    The output keeps the input's event order; GPU events shift without
    shrinking; fork/join timestamps are remapped with their process.
    """
    ct = trace if isinstance(trace, ColumnarTrace) else ColumnarTrace.from_trace(trace)
    out, rep = correct_trace_columnar(ct, profile, _src=trace)
    if isinstance(trace, ColumnarTrace):
        return out, rep
    events = [Event(e.pid, e.tid, e.category, e.name, s, d, e.correlation)
              for e, s, d in zip(trace.events, out.start.tolist(), out.dur.tolist())]
    res = Trace(trace.clock_domain, events, out.processes)
    remember_columnar(res, out)  # (compute_overlap(corrected) reuses the columns just produced)
    return res, rep


def analyze_columnar(ct: ColumnarTrace, profile: CalibrationProfile, attribution=None, device_trace=None,
                     out=None):
    """``xstrace analyze --profile``: correct, then compute_overlap(corrected).

    Returns (corrected start, corrected duration, report, Breakdown).  One
    device call (xs_analyze) runs both stages; the columns are device tensors,
    or, with ``out`` = (start, dur) host int64 buffers of length n (pinned:
    e.g. ``torch.empty(n, dtype=torch.int64).pin_memory()``), those buffers,
    filled by a copy that overlaps the overlap pass (xs_analyze_to_host).
    """
    from .overlap import Attribution, decode_breakdown

    attr = 1 if attribution is not None and Attribution(attribution) is Attribution.CORRELATION else 0
    def batched(wide: bool = False):
        start, dur, rep, _, bd = (_correct_wide if wide else _batched)(ct, profile, ct, attr)
        if out is not None:
            np.asarray(out[0])[...] = start
            np.asarray(out[1])[...] = dur
            return out[0], out[1], rep, bd
        import torch
        dev = torch.device("cuda", _engine.get().device)
        return torch.from_numpy(start).to(dev), torch.from_numpy(dur).to(dev), rep, bd

    if device_trace is None and _split.needs_split(ct):
        return batched()
    try:
        eng, dt, raw = _run(ct, profile, ct, attr, device_trace, host_out=out)
    except _engine.XsError as exc:
        if exc.status != _lib.XS_UNSUPPORTED or device_trace is not None:
            raise
        if _split.wide_pids(ct):
            return batched(wide=True)  # a process too wide for one call's keys by itself
        if ct.n_pids < 2:
            raise
        return batched()  # keys too wide for all pids at once (CORRELATION keys also hold path bits)
    bd = decode_breakdown(ct, eng.fetch_overlap())
    if out is not None:
        return out[0], out[1], _report(ct, raw), bd
    return raw.start, raw.dur, _report(ct, raw), bd


_PIPE_BUFS: dict = {}  # analyze_columnar_pipelined's double buffers, kept across calls


def _pid_batches(ct: ColumnarTrace, batches: int) -> list:
    """Contiguous row ranges holding whole pids (pid column non-decreasing),
    about n / batches rows each; [] when the rows are not pid-contiguous."""
    if ct.n == 0 or ct.n_pids < 2:
        return []
    memo = ct.__dict__.get("_pid_starts")  # (checked once per trace object)
    if memo is None:
        contiguous = not np.any(ct.pid[1:] < ct.pid[:-1])
        memo = np.searchsorted(ct.pid, np.arange(ct.n_pids + 1, dtype=np.int32)) if contiguous else False
        ct.__dict__["_pid_starts"] = memo
    if memo is False:
        return []
    starts = memo  # first row of every pid
    cuts = [0]
    for b in range(1, batches):
        r = int(starts[np.searchsorted(starts, b * ct.n // batches)])  # next pid boundary
        if cuts[-1] < r < ct.n:
            cuts.append(r)
    cuts.append(ct.n)
    return list(zip(cuts[:-1], cuts[1:]))


def _row_slice(ct: ColumnarTrace, a: int, b: int) -> ColumnarTrace:
    """Rows [a, b) with every table kept (pid/tid/name indices stay valid);
    pinned columns stay pinned (views)."""
    pin = None
    if ct._pinned is not None:
        pin = {k: (t[a:b] if k in ("start", "dur", "pid", "tid", "cat", "name", "corr", "has_corr") else t)
               for k, t in ct._pinned.items() if not k.startswith("_")}  # (the whole-block DMA is per trace)
    return ColumnarTrace(ct.clock_domain, ct.start[a:b], ct.dur[a:b], ct.pid[a:b], ct.tid[a:b], ct.cat[a:b],
                         ct.name[a:b], ct.corr[a:b], ct.has_corr[a:b], ct.pids, ct.group_pid, ct.group_tid, ct.names,
                         ct.processes, ct.pid_has_meta, None, pin)


def analyze_columnar_pipelined(ct: ColumnarTrace, profile: CalibrationProfile, out, attribution=None,
                               batches: int = 9, workers: int = 3):
    """analyze_columnar for host-resident traces of many processes, with the
    upload of the next batch of pids overlapping the analysis of the current
    one (per-pid independence: overlap.py:126, correction.py:132).  Needs
    pid-contiguous rows (e.g. ``synth``/per-process ingest) and host output
    buffers ``out`` = (start, dur); falls back to one call otherwise.
    ``workers`` contexts (own workspace, graphs and streams, one host thread
    each) take the batches in turn, so their analyses also overlap each
    other (config 3, 100M events: 1 context 94 ms, 2: 83 ms, 3: 79 ms).
    Returns (start, dur, report, Breakdown) like analyze_columnar."""
    import torch

    from .overlap import Attribution, _decode_cells

    parts = _pid_batches(ct, batches)
    # a dominant pid (skewed traces) leaves nothing to overlap: one call is cheaper
    if len(parts) < 2 or max(b - a for a, b in parts) > 0.4 * ct.n:
        return analyze_columnar(ct, profile, attribution, out=out)
    if meta_violations(ct.processes):
        raise InvalidTraceError(format_violations(ct.to_trace()))
    attr = 1 if attribution is not None and Attribution(attribution) is Attribution.CORRELATION else 0
    eng = _engine.get()
    dev = torch.device("cuda", eng.device)
    scaled = profile.scaled(ct.names)
    subs = [_row_slice(ct, a, b) for a, b in parts]
    starts = ct.__dict__["_pid_starts"]
    has = starts[1:] > starts[:-1]
    for sub, (a, b) in zip(subs, parts):  # pids present in each batch, from the pid row ranges
        sub.__dict__["_present_mask"] = has & (starts[:-1] >= a) & (starts[:-1] < b)

    # per worker (one context and stream each, batches k = w, w + W, ...): two
    # persistent device buffer sets (double buffering) whose stable addresses
    # keep every batch's captured pipeline graph valid across calls
    W = max(1, min(int(workers), len(parts)))
    engines = [_engine.get_aux(eng.device, w) for w in range(W)]
    cols = ("start", "dur", "pid", "tid", "cat", "name", "corr", "has_corr")
    rows_max = max(b - a for a, b in parts)
    lay = (ct._pinned or {}).get("_packed")
    pcols = ("start", "dur", "pid", "tid", "name", "corr", "catf")
    key = (eng.device, rows_max, W, tuple(lay.widths[c] for c in pcols) if lay is not None else None)
    state = _PIPE_BUFS.get(key)
    if state is None:
        _PIPE_BUFS.clear()
        state = []
        for w in range(W):
            st = {"bufs": [{c: torch.empty(rows_max, dtype=_engine.torch_dtype(getattr(ct, c).dtype), device=dev)
                            for c in cols} for _ in range(2)]}
            if lay is not None:
                st["pbufs"] = [{c: torch.empty(rows_max * lay.widths[c] + 16, dtype=torch.uint8, device=dev)
                                for c in pcols} for _ in range(2)]
                for pb in st["pbufs"]:
                    pb["start_base"] = torch.empty((rows_max // 256 + 2) * 8, dtype=torch.uint8, device=dev)
            state.append(st)
        _PIPE_BUFS[key] = state
    for w in range(W):
        state[w]["copy"] = torch.cuda.Stream(dev)
        state[w]["compute"] = torch.cuda.Stream(dev)
    tables = {"group_pid": torch.from_numpy(np.ascontiguousarray(ct.group_pid, np.int32)).to(dev),
              "pid_has_meta": torch.from_numpy(np.ascontiguousarray(ct.pid_has_meta, np.uint8)).to(dev)}
    if lay is not None:  # packed pinned block: per batch, DMA the row slices, widen on the copy stream
        block = ct._pinned["_block"]
        e0 = lay.offsets["exc_row"]  # the exception table (rows, values, columns: adjacent), whole, once per call
        exc_dev = block[e0:e0 + max(lay.offsets["exc_col"] + lay.nbytes["exc_col"] - e0, 16)].to(dev, non_blocking=True)
    ready = torch.cuda.Event()
    ready.record(torch.cuda.current_stream(dev))

    def upload(k, w):
        a, b = parts[k]
        st = state[w]
        par = (k // W) % 2
        buf, copy, e = st["bufs"][par], st["copy"], engines[w]
        with torch.cuda.stream(copy):
            copy.wait_event(ready)
            tens = {c: buf[c][: b - a] for c in cols}
            if lay is not None:
                pb = st["pbufs"][par]
                for c in pcols:
                    o, wd = lay.offsets[c], lay.widths[c]
                    pb[c][: (b - a) * wd].copy_(block[o + a * wd:o + b * wd], non_blocking=True)
                o, b0, b1 = lay.offsets["start_base"], a // 256, (b - 1) // 256 + 1
                if lay.widths["start"] == 4:
                    pb["start_base"][: (b1 - b0) * 8].copy_(block[o + b0 * 8:o + b1 * 8], non_blocking=True)
                ptrs = {c: t.data_ptr() for c, t in pb.items()}
                ptrs.update({c: exc_dev.data_ptr() + lay.offsets[c] - lay.offsets["exc_row"]
                             for c in ("exc_row", "exc_val", "exc_col")})
                _engine.unpack_into(e, lay, ptrs, a, b, SimpleNamespace(**tens), stream=copy)
            elif subs[k]._pinned is None and _stage_batch(subs[k], st, par, e, tens, copy, b - a, W):
                pass  # ordinary host columns: packed natively into this worker's page-locked staging
            else:
                for c in cols:
                    src = subs[k]._pinned[c] if subs[k]._pinned is not None else \
                        torch.from_numpy(getattr(subs[k], c))
                    tens[c].copy_(src, non_blocking=True)
            tens.update(tables)
            ev = torch.cuda.Event()
            ev.record(copy)
        return _engine.DeviceTrace.from_tensors(subs[k], tens, eng.device), ev

    okey = (eng.device, "out", ct.n)  # corrected columns of every batch (disjoint slices: no reuse while copying)
    dev_out = _PIPE_BUFS.get(okey)
    if dev_out is None:
        dev_out = tuple(torch.empty(ct.n, dtype=torch.int64, device=dev) for _ in range(2))
        _PIPE_BUFS[okey] = dev_out
    results = [None] * len(parts)

    def worker(w):
        with torch.cuda.stream(state[w]["compute"]):
            _pipelined_batches(ct, engines[w], parts, list(range(w, len(parts), W)), subs, upload, w,
                               state[w]["compute"], scaled, attr, out, dev_out, results)

    try:
        if W == 1:
            worker(0)
        else:
            from concurrent.futures import ThreadPoolExecutor

            with ThreadPoolExecutor(W) as pool:  # (ctypes calls release the GIL: the contexts run concurrently)
                for f in [pool.submit(worker, w) for w in range(W)]:
                    f.result()
    finally:  # every batch's corrected columns are in `out` (also when a batch raised)
        for e in engines:
            e.host_copy_wait()
        # an upload queued for a batch that never ran may still be writing the
        # persistent buffers: drain every copy stream before they are reused
        for st in state:
            st["copy"].synchronize()
    # errors in trace order, like the reference's whole-trace require_valid
    # followed by collect_sites: any invalid batch wins over an uncalibrated
    # hook; among uncalibrated hooks the smallest global row is reported
    errs = [r for r in results if isinstance(r, _BatchError)]
    if errs:
        if any(e.kind == "invalid" for e in errs):
            raise InvalidTraceError(format_violations(ct.to_trace()))
        first = min(errs, key=lambda e: e.row)
        name = ct.names[int(ct.name[first.row])]
        raise UncalibratedHookError(f"uncalibrated hook: API_INTERNAL({name!r}) missing from profile")
    rep = CorrectionReport()
    bd_all = None
    raws = []
    for k, (r, ov, bd) in enumerate(results):
        rep.removed_ns.update(r.removed_ns)
        rep.shortfall_ns.update(r.shortfall_ns)
        rep.original_total_ns += r.original_total_ns
        rep.corrected_total_ns += r.corrected_total_ns
        raws.append((subs[k], ov))
        if bd_all is None:
            bd_all = bd
        else:
            bd_all.spans.update(bd.spans)
            bd_all.untracked.update(bd.untracked)

    def build():  # the cells dict, on first access (pids are disjoint across batches)
        cells = {}
        for sub, ov in raws:
            cells.update(_decode_cells(sub, ov))
        return cells

    bd_all._lazy = build
    return out[0], out[1], rep, bd_all


def _stage_batch(sub: ColumnarTrace, st: dict, par: int, eng, tens: dict, copy, rows: int, workers: int) -> bool:
    """Pack one batch's host columns (native builder, this worker's share of
    the host threads) into the worker's page-locked staging block of this
    parity, DMA it on the copy stream and widen it into ``tens``.  False when
    the batch is not packable (the caller copies the wide columns)."""
    import os

    import torch

    from .columnar import pack_native

    sp = st.setdefault("stage", [{}, {}])[par]
    if sp.get("ev") is not None:
        sp["ev"].synchronize()  # the last DMA out of this staging block is done

    def alloc(nbytes):
        h = sp.get("host")
        if h is None or h.numel() < nbytes:
            h = sp["host"] = torch.empty(int(nbytes * 1.25) + 16, dtype=torch.uint8, pin_memory=True)
        return h.numpy()[:nbytes]

    got = pack_native(sub, alloc, n_threads=max(1, (os.cpu_count() or 1) // max(workers, 1)))
    if got is None:
        return False
    lay = got[0]
    nb = max(lay.total, 16)
    d = sp.get("dev")
    if d is None or d.numel() < nb:
        d = sp["dev"] = torch.empty(int(nb * 1.25) + 16, dtype=torch.uint8, device=tens["start"].device)
    d[:nb].copy_(sp["host"][:nb], non_blocking=True)
    ev = sp.get("ev") or torch.cuda.Event()
    ev.record(copy)
    sp["ev"] = ev
    _engine.unpack_into(eng, lay, _engine.packed_ptrs(lay, d), 0, rows, SimpleNamespace(**tens), stream=copy)
    return True


@dataclass
class _BatchError:
    """A batch of analyze_columnar_pipelined that failed (kind, global row)."""

    kind: str  # "invalid" | "uncalibrated"
    row: int


def _pipelined_batches(ct, eng, parts, ks, subs, upload, w, compute, scaled, attr, out, dev_out, results):
    from .overlap import _decode_breakdown

    nxt = upload(ks[0], w)
    for i, k in enumerate(ks):
        a, b = parts[k]
        dt, ev = nxt
        compute.wait_event(ev)
        if i + 1 < len(ks):
            nxt = upload(ks[i + 1], w)  # overlaps the analysis below
        try:  # the batch's D2H overlaps the next batch's analysis (waited for by the caller)
            raw = eng.correct(dt, scaled, attr, host_out=(out[0][a:b], out[1][a:b]),
                              dev_out=(dev_out[0][a:b], dev_out[1][a:b]), async_copy=True)
        except _engine.UncalibratedEvent as exc:  # keep going: a later batch may hold an invalid event
            results[k] = _BatchError("uncalibrated", a + int(exc.index))
            continue
        except _engine.XsError as exc:
            if exc.status == _lib.XS_INVALID_TRACE:
                results[k] = _BatchError("invalid", a)
                continue
            raise
        ov = eng.fetch_overlap()
        results[k] = (_report(subs[k], raw), ov, _decode_breakdown(subs[k], ov))
        del dt
