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


def analyze_sharded(ct: ColumnarTrace, profile, attribution=None, device=None, gather_columns: bool = False):
    """``xstrace analyze --profile`` over ``world`` ranks, one GPU each:
    correct_trace then compute_overlap of the corrected trace, sharded by
    whole processes (LPT on event counts; per-pid independence,
    correction.py:132-157, overlap.py:126).  Every rank returns the merged
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
            bad_row = _first_uncalibrated_row(local, profile, rows)
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
        return np.arange(ct.n), full_s, full_d, rep, bd
    return rows, start, dur, rep, bd


def _first_uncalibrated_row(local: ColumnarTrace, profile, rows) -> int:
    """Global row of the first ACCEL_API event whose name the profile lacks."""
    have = set(profile.api_internal_ns)
    bad_names = np.array([nm not in have for nm in local.names], bool)
    sel = np.nonzero((local.cat == 4) & bad_names[local.name])[0] if len(local.names) else np.zeros(0, np.int64)
    return int(rows[sel[0]]) if sel.size else np.iinfo(np.int64).max
