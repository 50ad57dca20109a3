"""Multi-GPU sharding and the histogram merge.

Traces shard by process: overlap, spans and correction are independent per
pid (overlap.py:126, correction.py:132), so ranks analyse disjoint pid sets
with no data-path collective.  The only exchange is the merge of the small
per-rank results:

* path ids are internal to each rank's trie, so ranks first agree on a global
  path table (an all-gather of the name tuples their cells use -- a few KB);
* every rank turns its nonzero cells into exact int64 keys (pid, global
  path, mask) with their ns; one variable-length all-gather over NCCL
  exchanges them (bounded by the nonzero cells, not by pids x paths x 32)
  and every rank sums them by key -- integer sums are order independent, so
  the merge is bit-exact;
* spans and tracked time travel the same way, merged by MIN / MAX / SUM.

The same code runs on ``gloo`` (CPU tensors) for the world-size-2 tests.
"""

from __future__ import annotations

import numpy as np

from .columnar import ColumnarTrace
from .model import Category
from .overlap import Breakdown, OverlapKey, decode_paths

_MASK_CATS = [frozenset(Category(c) for c in range(1, 6) if m & (1 << (c - 1))) for m in range(32)]


def shard_pids(ct: ColumnarTrace, world: int) -> list:
    """LPT packing of pid indices onto ``world`` ranks by event count."""
    counts = np.bincount(ct.pid, minlength=ct.n_pids) if ct.n else np.zeros(ct.n_pids, np.int64)
    order = np.argsort(-counts, kind="stable")
    loads = [0] * world
    out: list = [[] for _ in range(world)]
    for p in order.tolist():
        r = min(range(world), key=lambda k: (loads[k], k))
        out[r].append(p)
        loads[r] += int(counts[p])
    return [sorted(x) for x in out]


def local_cells(ct: ColumnarTrace, raw) -> tuple:
    """(pid value, path tuple, mask, ns) rows + per-pid (lo, hi, tracked)."""
    paths = decode_paths(ct, raw.node_parent, raw.node_name)
    pids = ct.pids.tolist()
    rows = [(pids[p], paths[nd], m, ns) for p, nd, m, ns in
            zip(raw.cell_pid.tolist(), raw.cell_node.tolist(), raw.cell_mask.tolist(), raw.cell_ns.tolist())]
    per_pid = {pids[p]: (int(raw.span_lo[p]), int(raw.span_hi[p]), int(raw.tracked[p]))
               for p in range(ct.n_pids) if raw.has_events[p]}
    return rows, per_pid


_TABLES = {"paths": (), "pids": ()}  # global path / pid tables agreed by earlier merges (identical on all ranks)


def _gather_var(x, device, world):
    """all_gather of a variable-length 1-D int64 tensor: sizes first, then
    the padded payloads; returns the concatenation in rank order."""
    import torch
    import torch.distributed as dist

    n = torch.tensor([x.numel()], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(t.item()) for t in sizes]
    m = max(max(sizes), 1)
    buf = torch.zeros(m, dtype=torch.int64, device=device)
    buf[: x.numel()] = x
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    return torch.cat([o[:k] for o, k in zip(out, sizes)])


def merge_breakdown_raw(ct: ColumnarTrace, raw, device) -> Breakdown:
    """Merge every rank's overlap result into one Breakdown (all ranks get it);
    see merge_breakdown_parts."""
    return merge_breakdown_parts([(ct, raw)], device)


def merge_breakdown_parts(parts: list, device) -> Breakdown:
    """Merge every rank's overlap results -- each rank passes its list of
    (trace, raw device result) parts, e.g. one per pid batch -- into one
    Breakdown on every rank.

    Path ids are per-call trie nodes, so ranks first agree on a global table
    of the path tuples their cells use (an object all-gather of a few KB,
    cached: later merges skip it once one MIN all-reduce says every rank's
    paths are known).  Each nonzero cell then becomes one exact int64 key
    (global pid, global path, mask) with its ns; the keys and values of all
    ranks are all-gathered (variable length: the exchange is bounded by the
    nonzero cells, not by pids x paths x 32) and summed by key -- integer sums
    commute, so the merge is bit-exact and identical on every rank.  Per-pid
    spans and tracked time travel the same way (MIN / MAX / SUM by pid)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    decoded = []
    my_paths, my_pids = {()}, set()
    for ct, raw in parts:
        paths = decode_paths(ct, raw.node_parent, raw.node_name)
        node_ids = np.unique(raw.cell_node) if raw.cell_node.size else np.zeros(0, np.int32)
        my_paths |= {paths[i] for i in node_ids.tolist()}
        my_pids |= set(ct.pids[np.nonzero(raw.has_events)[0]].tolist())
        decoded.append((ct, raw, paths, node_ids))
    known = my_paths <= set(_TABLES["paths"]) and my_pids <= set(_TABLES["pids"])
    if world > 1:
        flag = torch.tensor([1 if known else 0], dtype=torch.int64, device=device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        known = bool(flag.item())
    if not known:  # grow the tables (first merge, or new paths): tiny object all-gather
        mine = (sorted(my_paths), sorted(my_pids))
        gathered = [None] * world
        if world > 1:
            dist.all_gather_object(gathered, mine)
        else:
            gathered = [mine]
        _TABLES["paths"] = tuple(sorted(set(_TABLES["paths"]) | {p for g in gathered for p in g[0]}))
        _TABLES["pids"] = tuple(sorted(set(_TABLES["pids"]) | {p for g in gathered for p in g[1]}))
    all_paths, all_pids = _TABLES["paths"], _TABLES["pids"]
    path_ix = {p: i for i, p in enumerate(all_paths)}
    pid_ix = {p: i for i, p in enumerate(all_pids)}
    Q = len(all_paths)
    keys_l, vals_l, rows_l = [], [], []
    for ct, raw, paths, node_ids in decoded:
        node_to_q = np.zeros(max(len(paths), 1), np.int64)
        for i in node_ids.tolist():
            node_to_q[i] = path_ix[paths[i]]
        pv = np.array([pid_ix.get(int(p), 0) for p in ct.pids.tolist()], np.int64)  # global pid index
        keys_l.append((pv[raw.cell_pid] * Q + node_to_q[raw.cell_node]) * 32 + raw.cell_mask.astype(np.int64))
        vals_l.append(raw.cell_ns.astype(np.int64))
        has = np.nonzero(raw.has_events)[0]
        if has.size:
            rows_l.append(np.stack([pv[has], raw.span_lo[has].astype(np.int64), raw.span_hi[has].astype(np.int64),
                                    raw.tracked[has].astype(np.int64)], axis=1).reshape(-1))
    keys = np.concatenate(keys_l) if keys_l else np.zeros(0, np.int64)
    vals = np.concatenate(vals_l) if vals_l else np.zeros(0, np.int64)
    pid_rows = np.concatenate(rows_l) if rows_l else np.zeros(0, np.int64)
    # exchange and sum by key on the device (NCCL all-gather, then one
    # sort-unique + index_add over the gathered cells)
    tk, tv, tp = (torch.from_numpy(np.ascontiguousarray(a)).to(device) for a in (keys, vals, pid_rows))
    if world > 1:
        tk, tv, tp = (_gather_var(x, device, world) for x in (tk, tv, tp))
    uk_t, inv_t = torch.unique(tk, sorted=True, return_inverse=True)
    sums_t = torch.zeros(uk_t.shape[0], dtype=torch.int64, device=tk.device).index_add_(0, inv_t, tv)
    uk, sums, pid_rows = uk_t.cpu().numpy(), sums_t.cpu().numpy(), tp.cpu().numpy()
    bd = Breakdown()
    mk = tuple.__new__
    for k, v in zip(uk.tolist(), sums.tolist()):
        if v:
            pid_q, m = divmod(k, 32)
            p, q = divmod(pid_q, Q)
            bd.cells[mk(OverlapKey, (all_pids[p], all_paths[q], _MASK_CATS[m]))] = v
    spans, tracked = {}, {}
    for p, lo, hi, t in pid_rows.reshape(-1, 4).tolist():
        a, b = spans.get(p, (lo, hi))
        spans[p] = (min(a, lo), max(b, hi))
        tracked[p] = tracked.get(p, 0) + t
    for p in sorted(spans):
        bd.spans[all_pids[p]] = spans[p]
        bd.untracked[all_pids[p]] = (spans[p][1] - spans[p][0]) - tracked[p]
    return bd


def compute_overlap_sharded(ct: ColumnarTrace, attribution=None, device=None, split: int = 2) -> Breakdown:
    """compute_overlap over ``world`` ranks (one GPU each): pids LPT-packed,
    giant pids cut into operation-free time windows (INSTANT attribution);
    every rank returns the merged Breakdown.  Invalid traces raise
    InvalidTraceError on every rank (the verdict is all-reduced first)."""
    import torch
    import torch.distributed as dist

    from . import _engine, _lib
    from .model import InvalidTraceError, format_violations
    from .overlap import Attribution

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    corr = attribution is not None and Attribution(attribution) is Attribution.CORRELATION
    plan = plan_shards(ct, world, 0 if corr else split)
    split_pids = sorted({p for sh in plan for p, a, b in sh if a is not None or b is not None})
    bad = 0 if check_split_correlations(ct, split_pids) else 1
    local = shard_trace(ct, plan[rank])
    eng = _engine.get(torch.cuda.current_device())
    dev = device or torch.device("cuda", eng.device)
    raw = None
    if not bad:
        try:
            raw = eng.overlap(_engine.DeviceTrace(local, eng.device), 1 if corr else 0)
        except _engine.XsError as exc:
            if exc.status != _lib.XS_INVALID_TRACE:
                raise
            bad = 1
    if world > 1:
        flag = torch.tensor([bad], dtype=torch.int64, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        bad = int(flag.item())
    if bad:
        raise InvalidTraceError(format_violations(ct.to_trace()))
    return merge_breakdown_raw(local, raw, dev)


# ---------------------------------------------------------------------------
# Time-window splitting of giant pids (partitioning (2))
#
# A pid with more than n / (world * split) events is cut into time windows at
# operation-free instants: cut c is valid when no OPERATION event of the pid
# (any tid) has start < c < end.  Then every operation lies inside one window,
# so a window's operation ranks, nesting checks and paths are those of the
# whole pid (overlap.py:96-99, 132-142 only compare operations active at one
# instant).  Resource events are clipped to each window they overlap; the
# sweep of a window then accounts exactly the window's part of the timeline
# (_sweep_py.py:29-115 is a function of the active set at each instant), so
# cells and tracked time add up over windows and spans merge by MIN/MAX.
# Zero-duration events go to the window holding their start (they only feed
# the spans).  INSTANT attribution only: CORRELATION pins a GPU event to its
# launcher's path, which may sit in another window; such traces shard by pid.


def op_free_gaps(ct: ColumnarTrace, p: int) -> np.ndarray:
    """[k, 2] closed intervals of valid cut instants for pid index p (the gaps
    between the union of its operations, plus the unbounded ends)."""
    sel = (ct.pid == p) & (ct.cat == 0)
    s = ct.start[sel]
    e = s + ct.dur[sel]
    big = np.iinfo(np.int64).max
    if s.size == 0:
        return np.array([[-big, big]], np.int64)
    o = np.argsort(s, kind="stable")
    s, e = s[o], e[o]
    run = np.maximum.accumulate(e)  # max end of ops starting up to here
    # a gap opens after op i when every op so far has ended by the next start
    gap_after = np.nonzero(run[:-1] <= s[1:])[0]
    lo = np.concatenate([[-big], run[gap_after], [run[-1]]])
    hi = np.concatenate([[s[0]], s[gap_after + 1], [big]])
    return np.stack([lo, hi], axis=1)


def window_cuts(ct: ColumnarTrace, p: int, parts: int) -> list:
    """Up to parts-1 cut instants for pid index p, near the event-count
    quantiles, each snapped into an operation-free gap."""
    if parts <= 1:
        return []
    starts = np.sort(ct.start[ct.pid == p])
    if starts.size == 0:
        return []
    gaps = op_free_gaps(ct, p)
    cuts = []
    for j in range(1, parts):
        q = int(starts[min(starts.size - 1, j * starts.size // parts)])
        k = int(np.searchsorted(gaps[:, 0], q, side="right")) - 1  # last gap opening at or before q
        best = None
        for g in (k, k + 1):
            if 0 <= g < gaps.shape[0]:
                c = min(max(q, int(gaps[g, 0])), int(gaps[g, 1]))
                if best is None or abs(c - q) < abs(best - q):
                    best = c
        if best is not None and (not cuts or best > cuts[-1]):
            cuts.append(best)
    return cuts


def plan_shards(ct: ColumnarTrace, world: int, split: int = 2) -> list:
    """Per rank, a list of shards (pid index, lo, hi): whole pids (lo = hi =
    None) or time windows [lo, hi) of giant pids; LPT-packed by event count."""
    counts = np.bincount(ct.pid, minlength=ct.n_pids) if ct.n else np.zeros(ct.n_pids, np.int64)
    target = max(1, -(-ct.n // max(1, world * split)))
    items = []
    for p in range(ct.n_pids):
        c = int(counts[p])
        if c == 0:
            continue
        parts = min(world * split, -(-c // target)) if world > 1 and split > 0 else 1
        cuts = window_cuts(ct, p, parts) if parts > 1 else []
        if not cuts:
            items.append((c, p, None, None))
            continue
        bounds = [None] + cuts + [None]
        st = ct.start[ct.pid == p]
        for a, b in zip(bounds[:-1], bounds[1:]):
            m = np.ones(st.shape[0], bool)
            if a is not None:
                m &= st >= a
            if b is not None:
                m &= st < b
            items.append((int(m.sum()), p, a, b))
    loads = [0] * world
    out: list = [[] for _ in range(world)]
    for c, p, a, b in sorted(items, key=lambda x: (-x[0], x[1], -(2**63) if x[2] is None else x[2])):
        r = min(range(world), key=lambda k: (loads[k], k))
        out[r].append((p, a, b))
        loads[r] += c
    return out


def check_split_correlations(ct: ColumnarTrace, pids: list) -> bool:
    """Dangling-correlation rule (model.py:207-217) for pids whose windows
    land on different ranks: every GPU correlation must name an ACCEL_API
    correlation of the same pid.  Host numpy over the split pids only."""
    for p in pids:
        sel = ct.pid == p
        api = np.unique(ct.corr[sel & (ct.cat == 4) & (ct.has_corr == 1)])
        gpu = ct.corr[sel & (ct.cat == 5) & (ct.has_corr == 1)]
        if gpu.size and not np.isin(gpu, api).all():
            return False
    return True


def shard_trace(ct: ColumnarTrace, shards: list) -> ColumnarTrace:
    """The rows (and clipped intervals) one rank analyses; row order is kept,
    so the reference's index tie-breaks are unchanged inside every pid."""
    n = ct.n
    keep = np.zeros(n, bool)
    lo_c = np.full(n, np.iinfo(np.int64).min, np.int64)
    hi_c = np.full(n, np.iinfo(np.int64).max, np.int64)
    split = np.zeros(n, bool)
    whole = [p for p, a, b in shards if a is None and b is None]
    if whole:
        keep |= np.isin(ct.pid, np.asarray(whole, np.int32))
    start = ct.start.copy()
    dur = ct.dur.copy()
    end = ct.start + ct.dur
    out_rows = []
    for p, a, b in shards:
        if a is None and b is None:
            continue
        lo = np.iinfo(np.int64).min if a is None else a
        hi = np.iinfo(np.int64).max if b is None else b
        sel = ct.pid == p
        point = sel & ((ct.dur == 0) | (ct.cat == 0)) & (ct.start >= lo) & (ct.start < hi)
        span = sel & (ct.dur > 0) & (ct.cat != 0) & (ct.start < hi) & (end > lo)
        rows = np.nonzero(point | span)[0]
        out_rows.append((rows, lo, hi))
        split |= sel
    # a pid with several windows on this rank contributes one piece per window
    idx = [np.nonzero(keep)[0]] + [r for r, _, _ in out_rows]
    lo_l = [np.full(idx[0].shape[0], np.iinfo(np.int64).min, np.int64)] + \
        [np.full(r.shape[0], lo, np.int64) for r, lo, _ in out_rows]
    hi_l = [np.full(idx[0].shape[0], np.iinfo(np.int64).max, np.int64)] + \
        [np.full(r.shape[0], hi, np.int64) for r, _, hi in out_rows]
    rows = np.concatenate(idx)
    lo_a, hi_a = np.concatenate(lo_l), np.concatenate(hi_l)
    order = np.argsort(rows, kind="stable")  # trace order (windows of one pid interleave by row)
    rows, lo_a, hi_a = rows[order], lo_a[order], hi_a[order]
    s = ct.start[rows]
    e = end[rows]
    clip = ct.cat[rows] != 0
    s2 = np.where(clip & (ct.dur[rows] > 0), np.maximum(s, lo_a), s)
    e2 = np.where(clip & (ct.dur[rows] > 0), np.minimum(e, hi_a), e)
    has_corr = ct.has_corr[rows].copy()
    # INSTANT never reads GPU correlations beyond the dangling rule, checked
    # on the host for split pids (check_split_correlations)
    has_corr[split[rows] & (ct.cat[rows] == 5)] = 0
    del start, dur, lo_c, hi_c
    return ColumnarTrace(ct.clock_domain, s2, e2 - s2, ct.pid[rows], ct.tid[rows], ct.cat[rows], ct.name[rows],
                         ct.corr[rows], has_corr, ct.pids, ct.group_pid, ct.group_tid, ct.names, ct.processes,
                         ct.pid_has_meta)


def merge_raw_list(parts: list) -> Breakdown:
    """Host merge of several (local trace, OverlapRaw) results -- the same sums
    and MIN/MAX as merge_breakdown_raw, without a process group (one GPU
    running every shard in turn, and the tests)."""
    cells: dict = {}
    spans: dict = {}
    tracked: dict = {}
    for ct, raw in parts:
        rows, per_pid = local_cells(ct, raw)
        for pv, path, m, ns in rows:
            k = (pv, path, m)
            cells[k] = cells.get(k, 0) + ns
        for pv, (a, b, t) in per_pid.items():
            lo, hi = spans.get(pv, (a, b))
            spans[pv] = (min(lo, a), max(hi, b))
            tracked[pv] = tracked.get(pv, 0) + t
    bd = Breakdown()
    for (pv, path, m), ns in cells.items():
        if ns:
            bd.cells[OverlapKey(pv, path, _MASK_CATS[m])] = ns
    for pv, (a, b) in spans.items():
        bd.spans[pv] = (a, b)
        bd.untracked[pv] = (b - a) - tracked[pv]
    return bd


# ---------------------------------------------------------------------------
# correct_trace + compute_overlap(corrected) over ranks (the analyze path)

def merge_reports(local_rep, device):
    """CorrectionReport rows of disjoint pid sets -> one report on every rank
    (tiny: 8 ints per pid, one object all-gather); totals add up because
    original/corrected totals are sums of per-pid spans (correction.py:159-186)."""
    import torch.distributed as dist

    from .correction import CorrectionReport

    world = dist.get_world_size() if dist.is_initialized() else 1
    mine = (local_rep.removed_ns, local_rep.shortfall_ns, local_rep.original_total_ns, local_rep.corrected_total_ns)
    parts = [None] * world
    if world > 1:
        dist.all_gather_object(parts, mine)
    else:
        parts = [mine]
    rep = CorrectionReport()
    for rm, sf, o, c in parts:
        rep.removed_ns.update(rm)
        rep.shortfall_ns.update(sf)
        rep.original_total_ns += o
        rep.corrected_total_ns += c
    rep.removed_ns = dict(sorted(rep.removed_ns.items()))
    rep.shortfall_ns = dict(sorted(rep.shortfall_ns.items()))
    return rep


def analyze_sharded(ct: ColumnarTrace, profile, attribution=None, device=None, gather_columns: bool = False,
                    split=None, runner=None):
    """``xstrace analyze --profile`` over ``world`` ranks, one GPU each:
    correct_trace then compute_overlap of the corrected trace, sharded by
    processes (LPT on event counts; per-pid independence,
    correction.py:132-157, overlap.py:126); with ``split`` > 0 a process
    holding more than n / (world * split) events is corrected as time
    windows spread over ranks, with the window carries (see
    _analyze_windows); default 2 when world > 1, 0 (whole processes: one
    fused device call) on a single rank.  Every rank returns the merged
    CorrectionReport and Breakdown (bit-exact: integer sums).  The corrected
    columns come back as this rank's rows (``rows``, ``start``, ``dur``) or,
    with ``gather_columns``, as the whole trace's columns on every rank.
    Errors keep whole-trace semantics on every rank: an invalid trace raises
    InvalidTraceError; else the uncalibrated hook of the smallest row raises
    UncalibratedHookError.  Returns (rows, start, dur, report, Breakdown)."""
    import torch
    import torch.distributed as dist

    from . import _engine, _lib
    from .correction import UncalibratedHookError, _report, _run
    from .model import InvalidTraceError, format_violations, meta_violations
    from .overlap import Attribution

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    eng = _engine.get(torch.cuda.current_device())
    dev = device or torch.device("cuda", eng.device)
    attr = 1 if attribution is not None and Attribution(attribution) is Attribution.CORRELATION else 0
    if split is None:
        split = 2 if world > 1 else 0
    if split > 0:
        out = _analyze_windows(ct, profile, attr, dev, world, rank, split, runner or DeviceWindowRunner(eng))
        if out is not None:
            rows, start, dur, rep, bd = out
            if gather_columns:
                return _gather_columns(ct, rows, start, dur, dev, world) + (rep, bd)
            return rows, start, dur, rep, bd
    shards = shard_pids(ct, world)
    keep = np.isin(ct.pid, np.asarray(shards[rank], np.int32))
    rows = np.nonzero(keep)[0]
    local = ct.select_pids(shards[rank])
    bad_invalid = 1 if meta_violations(ct.processes) else 0
    bad_row = np.iinfo(np.int64).max
    raw_c = raw_o = None
    if not bad_invalid:
        try:
            _, _, raw_c = _run(local, profile, local, attr)
            raw_o = eng.fetch_overlap()
        except InvalidTraceError:
            bad_invalid = 1
        except UncalibratedHookError:  # (_run maps the event; recover its row here)
            raw_c = None
            bad_row = _first_uncalibrated_row(local, profile, lrows)
    if world > 1:
        flags = torch.tensor([bad_invalid, -bad_row], dtype=torch.int64, device=dev)
        dist.all_reduce(flags, op=dist.ReduceOp.MAX)
        bad_invalid, bad_row = int(flags[0].item()), -int(flags[1].item())
    if bad_invalid:
        raise InvalidTraceError(format_violations(ct.to_trace()))
    if bad_row != np.iinfo(np.int64).max:
        name = ct.names[int(ct.name[bad_row])]
        raise UncalibratedHookError(f"uncalibrated hook: API_INTERNAL({name!r}) missing from profile")
    start = raw_c.start.cpu().numpy()
    dur = raw_c.dur.cpu().numpy()
    rep = merge_reports(_report(local, raw_c), dev)
    bd = merge_breakdown_raw(local, raw_o, dev)
    if gather_columns:
        return _gather_columns(ct, rows, start, dur, dev, world) + (rep, bd)
    return rows, start, dur, rep, bd


def _gather_columns(ct: ColumnarTrace, rows, start, dur, dev, world: int) -> tuple:
    """Every rank's corrected rows -> the whole trace's columns on every rank."""
    import torch

    full_s = np.zeros(ct.n, np.int64)
    full_d = np.zeros(ct.n, np.int64)
    if world > 1:
        gr, gs, gd = (_gather_var(torch.from_numpy(np.ascontiguousarray(a, np.int64)).to(dev), dev, world)
                      for a in (rows, start, dur))
        rows_all, s_all, d_all = gr.cpu().numpy(), gs.cpu().numpy(), gd.cpu().numpy()
    else:
        rows_all, s_all, d_all = rows, start, dur
    full_s[rows_all] = s_all
    full_d[rows_all] = d_all
    return np.arange(ct.n), full_s, full_d


def _first_uncalibrated_row(local: ColumnarTrace, profile, rows) -> int:
    """Global row of the first ACCEL_API event whose name the profile lacks."""
    have = set(profile.api_internal_ns)
    bad_names = np.array([nm not in have for nm in local.names], bool)
    sel = np.nonzero((local.cat == 4) & bad_names[local.name])[0] if len(local.names) else np.zeros(0, np.int64)
    return int(rows[sel[0]]) if sel.size else np.iinfo(np.int64).max


# ---------------------------------------------------------------------------
# Window-split correction of giant pids (correction carries)
#
# correct_trace walks each pid's sites in order with two running states
# (correction.py:132-157): quantize_amounts' rational sum `cum`
# (_timeline.py:57-67) and the RemovalMap's slab chain end E
# (_timeline.py:90-117).  A giant pid is cut at instants c that no event of
# the pid reaches across (every event starting before c ends before c) and
# that no launcher -> GPU kernel correlation pair straddles.  Then, per window:
#   * sites, owners' budgets, transition maximality / coverage and operation
#     nesting are window-local (no event crosses a cut; the strict end < c
#     keeps every earlier window's site before every later one in
#     Site.order_key);
#   * `cum` enters as a carry: the fractional part of the amounts of all
#     earlier windows (their site counts per amount row; one all-gather),
#     passed to the device as xs_profile_t.residue_in;
#   * if no slab of an earlier window runs past the cut (E <= c), the
#     window's slabs are its local ones and the global map is the local map
#     minus P_in, the total slab length before the window (a second tiny
#     all-gather); the device clips removed_ns at the next cut
#     (xs_profile_t.span_end_in), so removed == total slab length proves it;
#   * the corrected window trace is overlapped on its own: exact when no
#     corrected event crosses the mapped cut (GPU events keep their duration
#     while CPU time shrinks: checked as the corrected window end <= the
#     locally mapped cut).
# Any failed check (rare: removable time larger than the idle gap at a cut)
# re-runs the analysis with whole-pid shards -- exact either way.
# ---------------------------------------------------------------------------


def correction_cut_gaps(ct: ColumnarTrace, p: int, gpu_free: bool = False) -> np.ndarray:
    """[k, 2] closed intervals of valid window cuts for pid index p: instants
    c that no OPERATION reaches (start < c <= end: its ANN_END site must
    order before the next window's sites at c), no BACKEND / SIMULATOR /
    ACCEL_API event strictly straddles (start < c < end), and no correlated
    launcher / GPU pair sits across.  HIGH_LEVEL events may straddle: they
    own no site and are only the outer side of the wrapper transitions, so
    they are clipped into every window they cover.  GPU events may straddle
    too: the correction only shifts them by their start (_timeline.py:
    120-132); their parts past a window's mapped cut join the next windows'
    overlap passes as clipped pieces -- except with ``gpu_free`` (CORRELATION
    attribution: a clipped kernel piece would lose its launcher's path), where
    GPU events may not straddle either."""
    sel = np.nonzero(ct.pid == p)[0]
    s = ct.start[sel]
    e = s + ct.dur[sel]
    cat = ct.cat[sel]
    op = cat == 0
    mid = (cat >= 2) & (cat <= (5 if gpu_free else 4))
    lo_r = [s[op] + 1, s[mid] + 1]
    hi_r = [e[op], e[mid] - 1]
    api = sel[(cat == 4) & (ct.has_corr[sel] == 1)]
    gpu = sel[(cat == 5) & (ct.has_corr[sel] == 1)]
    if api.size and gpu.size:
        ac, ast = ct.corr[api], ct.start[api]
        o = np.lexsort((ast, ac))
        ac, ast = ac[o], ast[o]
        first = np.r_[True, ac[1:] != ac[:-1]]
        ids, lstart = ac[first], ast[first]
        gc, gs = ct.corr[gpu], ct.start[gpu]
        k = np.minimum(np.searchsorted(ids, gc), ids.size - 1)
        ok = ids[k] == gc
        lo_r.append(np.minimum(lstart[k], gs)[ok] + 1)
        hi_r.append(np.maximum(lstart[k], gs)[ok])
    lo_a, hi_a = np.concatenate(lo_r), np.concatenate(hi_r)
    m = hi_a >= lo_a
    lo_a, hi_a = lo_a[m], hi_a[m]
    big = np.iinfo(np.int64).max
    if lo_a.size == 0:
        return np.array([[-big, big]], np.int64)
    o = np.argsort(lo_a, kind="stable")
    lo_a, hi_a = lo_a[o], hi_a[o]
    run = np.maximum.accumulate(hi_a)
    gap_after = np.nonzero(run[:-1] + 1 < lo_a[1:])[0]  # [run + 1, next lo - 1] is free
    glo = np.concatenate([[-big], run[gap_after] + 1, [run[-1] + 1]])
    ghi = np.concatenate([[lo_a[0] - 1], lo_a[gap_after + 1] - 1, [big]])
    return np.stack([glo, ghi], axis=1)


def correction_window_cuts(ct: ColumnarTrace, p: int, parts: int, gpu_free: bool = False) -> list:
    """Up to parts-1 cuts for pid index p near its event-count quantiles.
    A cut is the last valid instant of its gap (the next blocking event's
    start), leaving the whole idle room before it to the slabs of the
    window's last sites (the window check needs E <= c)."""
    if parts <= 1:
        return []
    starts = np.sort(ct.start[ct.pid == p])
    if starts.size == 0:
        return []
    gaps = correction_cut_gaps(ct, p, gpu_free)
    his = gaps[:, 1]
    his = his[(his > starts[0]) & (his <= starts[-1])]
    cuts = []
    for j in range(1, parts):
        if his.size == 0:
            break
        q = int(starts[min(starts.size - 1, j * starts.size // parts)])
        k = int(np.searchsorted(his, q))
        cand = [int(his[x]) for x in (k - 1, k) if 0 <= x < his.size]
        best = min(cand, key=lambda c: (abs(c - q), c))
        if not cuts or best > cuts[-1]:
            cuts.append(best)
    return cuts


def plan_correction_shards(ct: ColumnarTrace, world: int, split: int = 2, gpu_free: bool = False) -> list:
    """Per rank, shards (pid index, lo, hi): whole pids (None, None) or the
    correction windows [lo, hi) of giant pids; LPT-packed by event count."""
    counts = np.bincount(ct.pid, minlength=ct.n_pids) if ct.n else np.zeros(ct.n_pids, np.int64)
    target = max(1, -(-ct.n // max(1, world * split)))
    items = []
    for p in range(ct.n_pids):
        c = int(counts[p])
        if c == 0:
            continue
        parts = min(world * split, -(-c // target)) if split > 0 else 1
        cuts = correction_window_cuts(ct, p, parts, gpu_free) if parts > 1 else []
        if not cuts:
            items.append((c, p, None, None))
            continue
        st = np.sort(ct.start[ct.pid == p])
        bounds = [None] + cuts + [None]
        for a, b in zip(bounds[:-1], bounds[1:]):
            i0 = 0 if a is None else int(np.searchsorted(st, a, side="left"))
            i1 = st.size if b is None else int(np.searchsorted(st, b, side="left"))
            items.append((i1 - i0, p, a, b))
    loads = [0] * world
    out: list = [[] for _ in range(world)]
    for c, p, a, b in sorted(items, key=lambda x: (-x[0], x[1], -(2**63) if x[2] is None else x[2])):
        r = min(range(world), key=lambda k: (loads[k], k))
        out[r].append((p, a, b))
        loads[r] += c
    return out


def piece_trace(ct: ColumnarTrace, shards: list) -> tuple:
    """One device pid per shard (a whole pid, or one window [a, b) of a giant
    pid): (local trace, global row per local row, head, tail, pieces).  A
    window holds the pid's events starting in [a, b) plus the HIGH_LEVEL
    events reaching into it from earlier windows, each HIGH_LEVEL event
    clipped to [a, b); ``head`` marks the piece holding an event's start,
    ``tail`` the piece holding its end.  Rows keep trace order; each piece has
    its own (pid, tid) groups, so the correction's per-pid scans restart
    (with the carries) at every window."""
    neg = -(2**63)
    big = np.iinfo(np.int64).max
    pieces = sorted(shards, key=lambda s: (s[0], neg if s[1] is None else s[1]))
    order = np.argsort(ct.pid, kind="stable")
    bounds = np.searchsorted(ct.pid[order], np.arange(ct.n_pids + 1, dtype=np.int32))
    row_l, piece_l, s_l, e_l, head_l, tail_l = [], [], [], [], [], []
    for k, (p, a, b) in enumerate(pieces):
        r = order[bounds[p]:bounds[p + 1]]
        lo = neg if a is None else a
        hi = big if b is None else b
        st = ct.start[r]
        en = st + ct.dur[r]
        hl = ct.cat[r] == 1
        own = (st >= lo) & (st < hi)
        ghost = hl & (st < lo) & (en > lo)
        keep = own | ghost
        r, st, en, hl, own = r[keep], st[keep], en[keep], hl[keep], own[keep]
        clip_e = hl & (en > hi)
        row_l.append(r)
        piece_l.append(np.full(r.shape[0], k, np.int32))
        s_l.append(np.where(own, st, lo))
        e_l.append(np.where(clip_e, hi, en))
        head_l.append(own)
        tail_l.append(~clip_e)
    cat_ = lambda xs, dt: np.concatenate(xs) if xs else np.zeros(0, dt)
    rows, piece = cat_(row_l, np.int64), cat_(piece_l, np.int32)
    st, en = cat_(s_l, np.int64), cat_(e_l, np.int64)
    head, tail = cat_(head_l, bool), cat_(tail_l, bool)
    o = np.lexsort((piece, rows))  # trace order (a clipped row's pieces by window)
    rows, piece, st, en, head, tail = rows[o], piece[o], st[o], en[o], head[o], tail[o]
    G = max(ct.n_groups, 1)
    key = piece.astype(np.int64) * G + ct.tid[rows]
    ukey, new_tid = np.unique(key, return_inverse=True)
    pidx = np.array([p for p, _, _ in pieces], np.int64)
    local = ColumnarTrace(ct.clock_domain, st, en - st, piece, new_tid.astype(np.int32),
                          ct.cat[rows], ct.name[rows], ct.corr[rows], ct.has_corr[rows], ct.pids[pidx],
                          (ukey // G).astype(np.int32), ct.group_tid[ukey % G], ct.names, (),
                          ct.pid_has_meta[pidx] if ct.pid_has_meta is not None else None)
    return local, rows, head, tail, pieces


def _amount_sums(local: ColumnarTrace, profile, n_trans: np.ndarray):
    """Exact sum of the requested amounts of each piece's sites
    (collect_sites, correction.py:79-112)."""
    from fractions import Fraction

    P = local.n_pids
    ann = Fraction(profile.annotation_ns)
    ic = Fraction(profile.api_interception_ns)
    tr = Fraction(profile.transition_ns)
    n_op = np.bincount(local.pid[local.cat == 0], minlength=P)
    api = local.cat == 4
    n_api = np.bincount(local.pid[api], minlength=P)
    out = [ann * int(n_op[k]) + ic * int(n_api[k]) + tr * int(n_trans[k]) for k in range(P)]
    if api.any():
        nm = local.name[api].astype(np.int64)
        pk = local.pid[api].astype(np.int64)
        key, cnt = np.unique(pk * max(len(local.names), 1) + nm, return_counts=True)
        table = profile.api_internal_ns
        for kk, c in zip(key.tolist(), cnt.tolist()):
            k, n = divmod(kk, max(len(local.names), 1))
            v = table.get(local.names[n])
            if v is not None:
                out[k] += Fraction(v) * c
    return out


def _gather_objects(obj, world):
    import torch.distributed as dist

    if world == 1:
        return [obj]
    parts = [None] * world
    dist.all_gather_object(parts, obj)
    return parts


class DeviceWindowRunner:
    """The device side of the window analysis (tests substitute the C
    oracle): the wrapper transitions, one xs_correct call over this rank's
    pieces with the carries, one xs_overlap call over the corrected pieces."""

    def __init__(self, eng):
        self.eng = eng
        self.dt = None

    def _dt(self, local):
        from . import _engine

        if self.dt is None or self.dt.ct is not local:
            self.dt = _engine.DeviceTrace(local, self.eng.device)
        return self.dt

    def transition_rows(self, local: ColumnarTrace) -> np.ndarray:
        _, ev = self.eng.transition_sites(self._dt(local), 0x3)  # WRAPPER_PAIRS (overlap.py:200-203)
        return np.asarray(ev, np.int64)

    def correct(self, local: ColumnarTrace, profile, r_in: list, span_end: np.ndarray, queries=()):
        """-> (start, dur, removed [P, 4], shortfall [P, 4], mapped queries):
        ``queries`` = (piece, time) pairs mapped by that piece's local
        RemovalMap (xs_remap; fork / join instants)."""
        scaled = profile.scaled(local.names)
        residue = _residue_words(r_in, scaled, local.n_pids)
        raw = self.eng.correct(self._dt(local), scaled, None, carries=(residue, span_end))
        q = list(self.eng.remap(np.array([k for k, _ in queries], np.int32),
                                np.array([y for _, y in queries], np.int64))) if queries else []
        return raw.start.cpu().numpy(), raw.dur.cpu().numpy(), raw.removed, raw.shortfall, q

    def overlap(self, trace: ColumnarTrace, attr: int):
        from . import _engine

        return self.eng.overlap(_engine.DeviceTrace(trace, self.eng.device), attr)


def _residue_words(r_in: list, scaled, n_pids: int) -> np.ndarray:
    """xs_profile_t.residue_in: each piece's carried residue * L in words."""
    residue = np.zeros(max(n_pids, 1) * scaled.words, np.uint64)
    for k, r in enumerate(r_in):
        v = r * scaled.L
        assert v.denominator == 1 and 0 <= v < scaled.L
        residue[k * scaled.words:(k + 1) * scaled.words] = scaled.words_of(int(v))
    return residue


class SequentialWindowRunner(DeviceWindowRunner):
    """One device call per window (consecutive calls on one GPU): a single
    process with more rows than one call takes (_split.MAX_EVENTS_PER_CALL)
    is corrected window by window with the same carries."""

    def _pieces(self, trace: ColumnarTrace):
        from ._split import pid_rows, sub_trace

        by = pid_rows(trace)
        for k in range(trace.n_pids):
            sub, rows = sub_trace(trace, [k], by)
            yield k, sub, rows

    def transition_rows(self, local: ColumnarTrace) -> np.ndarray:
        from . import _engine

        out = []
        for _, sub, rows in self._pieces(local):
            if sub.n:
                _, ev = self.eng.transition_sites(_engine.DeviceTrace(sub, self.eng.device), 0x3)
                out.append(rows[np.asarray(ev, np.int64)])
        return np.sort(np.concatenate(out)) if out else np.zeros(0, np.int64)

    def correct(self, local: ColumnarTrace, profile, r_in: list, span_end: np.ndarray, queries=()):
        from . import _engine

        scaled = profile.scaled(local.names)
        P = local.n_pids
        start = np.zeros(local.n, np.int64)
        dur = np.zeros(local.n, np.int64)
        removed = np.zeros((max(P, 1), 4), np.int64)
        shortfall = np.zeros((max(P, 1), 4), np.int64)
        q = [0] * len(queries)
        for k, sub, rows in self._pieces(local):
            if not sub.n:
                continue
            raw = self.eng.correct(_engine.DeviceTrace(sub, self.eng.device), scaled, None,
                                   carries=(_residue_words([r_in[k]], scaled, 1), span_end[k:k + 1]))
            start[rows] = raw.start.cpu().numpy()
            dur[rows] = raw.dur.cpu().numpy()
            removed[k], shortfall[k] = raw.removed[0], raw.shortfall[0]
            mine = [i for i, (kk, _) in enumerate(queries) if kk == k]
            if mine:
                got = self.eng.remap(np.zeros(len(mine), np.int32), np.array([queries[i][1] for i in mine], np.int64))
                for i, v in zip(mine, list(got)):
                    q[i] = int(v)
        return start, dur, removed, shortfall, q

    def overlap(self, trace: ColumnarTrace, attr: int):
        from . import _engine

        return [(sub, self.eng.overlap(_engine.DeviceTrace(sub, self.eng.device), attr))
                for _, sub, _ in self._pieces(trace) if sub.n]


def _analyze_windows(ct: ColumnarTrace, profile, attr: int, dev, world: int, rank: int, split: int, runner,
                     queries=None, query_out=None, max_rows: int = 0):
    """analyze_sharded with giant pids corrected as windows (see above).
    Returns (rows, start, dur, report, Breakdown), or None when nothing was
    split, a window holds more than ``max_rows`` rows, or a window check
    failed on some rank (the caller then shards whole pids).  Raises like the
    reference on invalid / uncalibrated traces.  ``queries`` = (pid index,
    time) pairs (world 1) are mapped by the corrected process's RemovalMap
    into ``query_out`` (fork / join instants, correction.py:172-180)."""
    import math
    from fractions import Fraction

    import torch

    from . import _engine, _lib
    from ._split import pid_spans_host
    from .calibration import HOOK_KINDS
    from .correction import CorrectionReport, UncalibratedHookError
    from .model import InvalidTraceError, format_violations, meta_violations

    plan = plan_correction_shards(ct, world, split, gpu_free=attr == 1)
    if not any(a is not None or b is not None for sh in plan for _, a, b in sh):
        return None
    local, lrows, head, tail, pieces = piece_trace(ct, plan[rank])
    rows = lrows[head]
    assert world == 1 or not max_rows  # (a per-rank early return would desynchronise the collectives)
    if max_rows and local.n and int(np.bincount(local.pid).max()) > max_rows:
        return None
    rq = []
    for p, y in (queries or ()):
        ks = [k for k, (pp, a, b) in enumerate(pieces) if pp == p and (a is None or a <= y) and (b is None or y < b)]
        rq.append((ks[0], int(y)))
    P = local.n_pids
    neg, big = -(2**63), np.iinfo(np.int64).max
    win = [k for k, (_, a, b) in enumerate(pieces) if a is not None or b is not None]
    bad_invalid = 1 if meta_violations(ct.processes) else 0
    bad_row = big
    # phase A: each window's exact amount sum (its wrapper transitions
    # counted on the device); only the fractional parts travel
    n_trans = np.zeros(max(P, 1), np.int64)
    if win and not bad_invalid:
        try:
            n_trans = np.bincount(local.pid[runner.transition_rows(local)], minlength=max(P, 1))
        except _engine.XsError as exc:
            if exc.status != _lib.XS_INVALID_TRACE:
                raise
            bad_invalid = 1
    sums = _amount_sums(local, profile, n_trans)
    mine = [(pieces[k][0], neg if pieces[k][1] is None else pieces[k][1], sums[k] - math.floor(sums[k]))
            for k in win]
    fr = {}
    for part in _gather_objects(mine, world):
        for p, a, f in part:
            fr.setdefault(p, []).append((a, f))
    r_in = [Fraction(0)] * P
    for k in win:
        p, a, _ = pieces[k]
        a0 = neg if a is None else a
        r = sum((f for aa, f in fr[p] if aa < a0), Fraction(0))
        r_in[k] = r - math.floor(r)
    span_end = np.zeros(max(P, 1), np.int64)
    if local.n:
        span_end[:] = np.iinfo(np.int64).min
        np.maximum.at(span_end, local.pid, local.start + local.dur)
    for k in win:
        if pieces[k][2] is not None:
            span_end[k] = pieces[k][2]  # inner window: clip at the next cut
    res = None
    if not bad_invalid and P:
        try:
            res = runner.correct(local, profile, r_in, span_end, rq)
        except _engine.UncalibratedEvent:
            bad_row = _first_uncalibrated_row(local, profile, lrows)
        except _engine.XsError as exc:
            if exc.status != _lib.XS_INVALID_TRACE:
                raise
            bad_invalid = 1
    if world > 1:
        import torch.distributed as dist

        flags = torch.tensor([bad_invalid, -bad_row], dtype=torch.int64, device=dev)
        dist.all_reduce(flags, op=dist.ReduceOp.MAX)
        bad_invalid, bad_row = int(flags[0].item()), -int(flags[1].item())
    if bad_invalid:
        raise InvalidTraceError(format_violations(ct.to_trace()))
    if bad_row != big:
        name = ct.names[int(ct.name[bad_row])]
        raise UncalibratedHookError(f"uncalibrated hook: API_INTERNAL({name!r}) missing from profile")
    if res is not None:
        start, dur, removed, shortfall, qv = res
        start = np.array(start, np.int64, copy=True)
        dur = np.asarray(dur, np.int64)
    else:
        start = dur = np.zeros(0, np.int64)
        removed = shortfall = np.zeros((0, 4), np.int64)
        qv = []
    # phase B: total slab length per window -> P_in; no slab may run past a cut
    summ = []
    for k in win:
        p, a, b = pieces[k]
        T = math.floor(r_in[k] + sums[k]) - int(shortfall[k].sum())
        ok = b is None or int(removed[k].sum()) == T  # (E <= c: removed is clipped at the cut)
        summ.append((p, neg if a is None else a, T, ok))
    allw = [x for part in _gather_objects(summ, world) for x in part]
    if not all(ok for *_, ok in allw):
        return None
    # shift each window by P_in; the mapped cuts [cut_lo, cut_hi) of each piece
    cut_lo = np.full(max(P, 1), neg, np.int64)
    cut_hi = np.full(max(P, 1), big, np.int64)
    for k in win:
        p, a, b = pieces[k]
        a0 = neg if a is None else a
        p_in = sum(T for pp, aa, T, _ in allw if pp == p and aa < a0)
        T_k = next(T for pp, aa, T, _ in allw if pp == p and aa == a0)
        if p_in:
            start[local.pid == k] -= p_in  # every event shifts: GPU events keep dur (_timeline.py:120-132)
        if a is not None:
            cut_lo[k] = a - p_in
        if b is not None:
            cut_hi[k] = b - p_in - T_k
    end = start + dur
    # GPU events running past their window's mapped cut: clipped pieces for the
    # later windows' overlap passes (INSTANT reads no GPU correlation beyond
    # the dangling rule, which the unclipped originals keep)
    lp = local.pid[: start.shape[0]]
    over = np.nonzero(end > cut_hi[lp])[0] if start.size else np.zeros(0, np.int64)
    strad = [(int(pieces[lp[i]][0]), int(start[i]), int(end[i]), int(local.group_tid[local.tid[i]]),
              int(local.cat[i]), int(local.name[i]), int(local.has_corr[i])) for i in over.tolist()]
    strad = [x for part in _gather_objects(strad, world) for x in part]
    if attr == 1 and any(x[6] for x in strad):
        return None  # a correlated kernel's clipped part would lose its launcher's path
    o_e = end.copy()
    clip = (local.cat[: start.size] != 0) & (o_e > cut_hi[lp])
    o_e[clip] = cut_hi[lp][clip]
    g_rows = []
    for k in win:
        p = pieces[k][0]
        for pp, s0, e0, tv, c, nm, _ in strad:
            if pp == p and s0 < cut_lo[k] < e0:
                g_rows.append((k, int(cut_lo[k]), min(e0, int(cut_hi[k])), tv, c, nm))
    otrace = _overlap_trace(local, start, o_e, g_rows) if P else local
    raw_o = runner.overlap(otrace, attr) if P else _empty_raw()
    bd = merge_breakdown_parts(raw_o if isinstance(raw_o, list) else [(otrace, raw_o)], dev)
    if queries is not None:  # mapped by the window holding the instant, then shifted by its P_in
        for (k, _), v in zip(rq, qv):
            p, a, _ = pieces[k]
            a0 = neg if a is None else a
            query_out.append(int(v) - sum(T for pp, aa, T, _ in allw if pp == p and aa < a0))
    # a clipped HIGH_LEVEL event: start from its first piece, end from its last
    cont = [(int(r), int(x)) for r, x in zip(lrows[tail & ~head].tolist(), end[tail & ~head].tolist())]
    ends = dict(x for part in _gather_objects(cont, world) for x in part)
    out_end = end[head].copy()
    for i in np.nonzero(~tail[head])[0].tolist():
        out_end[i] = ends[int(rows[i])]
    out_start = start[head]
    start, dur = out_start, out_end - out_start
    # report: per-pid sums over windows and ranks; totals from the spans
    acc = {}
    for k in (np.nonzero(local.present_pid_mask())[0].tolist() if P else []):
        pv = int(local.pids[k])
        r0, s0 = acc.get(pv, (np.zeros(4, np.int64), np.zeros(4, np.int64)))
        acc[pv] = (r0 + removed[k], s0 + shortfall[k])
    merged = {}
    for part in _gather_objects({p: (r.tolist(), s.tolist()) for p, (r, s) in acc.items()}, world):
        for p, (r, s) in part.items():
            r0, s0 = merged.get(p, ([0] * 4, [0] * 4))
            merged[p] = ([x + y for x, y in zip(r0, r)], [x + y for x, y in zip(s0, s)])
    rep = CorrectionReport()
    for p in sorted(merged):
        rep.removed_ns[p] = dict(zip(HOOK_KINDS, merged[p][0]))
        rep.shortfall_ns[p] = dict(zip(HOOK_KINDS, merged[p][1]))
    lo, hi = pid_spans_host(ct)
    has = ct.present_pid_mask()
    rep.original_total_ns = int(sum(int(hi[p]) - int(lo[p]) for p in range(ct.n_pids) if has[p]))
    rep.corrected_total_ns = int(sum(b - a for a, b in bd.spans.values()))
    return rows, start, dur, rep, bd


def _overlap_trace(local: ColumnarTrace, o_s, o_e, g_rows: list) -> ColumnarTrace:
    """The corrected pieces (resources clipped at their mapped cut) plus the
    clipped GPU pieces from earlier windows, placed after the rows of the
    piece they join."""
    n = local.n
    if not g_rows:
        return ColumnarTrace(local.clock_domain, o_s, o_e - o_s, local.pid, local.tid, local.cat, local.name,
                             local.corr, local.has_corr, local.pids, local.group_pid, local.group_tid,
                             local.names, (), local.pid_has_meta)
    g = np.array(g_rows, np.int64)
    piece = np.concatenate([local.pid.astype(np.int64), g[:, 0]])
    tidv = np.concatenate([local.group_tid[local.tid].astype(np.int64), g[:, 3]])
    ukey, new_tid = np.unique(np.stack([piece, tidv], axis=1), axis=0, return_inverse=True)
    new_tid = new_tid.reshape(-1)
    s = np.concatenate([o_s, g[:, 1]])
    e = np.concatenate([o_e, g[:, 2]])
    cat = np.concatenate([local.cat, g[:, 4].astype(np.uint8)])
    name = np.concatenate([local.name, g[:, 5].astype(np.int32)])
    corr = np.concatenate([local.corr, np.zeros(len(g_rows), np.int64)])
    hc = np.concatenate([local.has_corr, np.zeros(len(g_rows), np.uint8)])
    order = np.lexsort((np.r_[np.arange(n), np.full(len(g_rows), n)], piece))
    return ColumnarTrace(local.clock_domain, s[order], (e - s)[order], piece[order].astype(np.int32),
                         new_tid[order].astype(np.int32), cat[order], name[order], corr[order], hc[order],
                         local.pids, ukey[:, 0].astype(np.int32), ukey[:, 1], local.names, (),
                         local.pid_has_meta)


def _empty_raw():
    from ._engine import OverlapRaw

    z32, z64 = np.zeros(0, np.int32), np.zeros(0, np.int64)
    return OverlapRaw(z32, z32, z32, z64, np.array([-1], np.int32), np.array([-1], np.int32), z64, z64, z64,
                      np.zeros(0, np.uint8))
