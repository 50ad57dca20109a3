"""Multi-GPU sharding and the histogram merge.

Traces shard by process: overlap, spans and correction are independent per
pid (overlap.py:126, correction.py:132), so ranks analyse disjoint pid sets
with no data-path collective.  The only exchange is the merge of the small
per-rank results:

* path ids are internal to each rank's trie, so ranks first agree on a global
  path table (an all-gather of the name tuples their cells use -- a few KB);
* every rank scatters its cells into a dense int64 histogram
  [pid][global path][32 masks] (+ tracked in mask 0 of path 0) and one
  ``all_reduce(SUM)`` over NCCL merges them; integer sums are order
  independent, so the merge is bit-exact;
* spans merge with MIN/MAX all-reduces.

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


def merge_breakdown_raw(ct: ColumnarTrace, raw, device) -> Breakdown:
    """Merge every rank's overlap result into one Breakdown (all ranks get it)."""
    import torch
    import torch.distributed as dist

    rows, per_pid = local_cells(ct, raw)
    world = dist.get_world_size() if dist.is_initialized() else 1
    # global tables: pid values and path tuples (tiny; object all-gather)
    mine = (sorted({r[1] for r in rows}), sorted(per_pid))
    gathered = [None] * world
    if world > 1:
        dist.all_gather_object(gathered, mine)
    else:
        gathered = [mine]
    all_paths = sorted({p for g in gathered for p in g[0]} | {()})
    all_pids = sorted({p for g in gathered for p in g[1]})
    path_ix = {p: i for i, p in enumerate(all_paths)}
    pid_ix = {p: i for i, p in enumerate(all_pids)}
    P, Q = len(all_pids), len(all_paths)
    hist = torch.zeros(P * Q * 32, dtype=torch.int64, device=device)
    if rows:
        idx = torch.tensor([(pid_ix[r[0]] * Q + path_ix[r[1]]) * 32 + r[2] for r in rows], dtype=torch.int64)
        val = torch.tensor([r[3] for r in rows], dtype=torch.int64)
        hist.index_add_(0, idx.to(device), val.to(device))
    span = torch.full((2, max(P, 1)), 0, dtype=torch.int64, device=device)
    lo = torch.full((max(P, 1),), 2**63 - 1, dtype=torch.int64)
    hi = torch.full((max(P, 1),), -(2**63), dtype=torch.int64)
    tracked = torch.zeros(max(P, 1), dtype=torch.int64)
    for pv, (a, b, t) in per_pid.items():
        lo[pid_ix[pv]] = a
        hi[pid_ix[pv]] = b
        tracked[pid_ix[pv]] = t
    lo, hi, tracked = lo.to(device), hi.to(device), tracked.to(device)
    if world > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM)
        dist.all_reduce(tracked, op=dist.ReduceOp.SUM)
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    del span
    h = hist.cpu().numpy()
    lo_n, hi_n, tr_n = lo.cpu().numpy(), hi.cpu().numpy(), tracked.cpu().numpy()
    bd = Breakdown()
    nz = np.nonzero(h)[0]
    for i in nz.tolist():
        m = i & 31
        row = i >> 5
        p, q = divmod(row, Q)
        bd.cells[OverlapKey(all_pids[p], all_paths[q], _MASK_CATS[m])] = int(h[i])
    for k, pv in enumerate(all_pids):
        bd.spans[pv] = (int(lo_n[k]), int(hi_n[k]))
        bd.untracked[pv] = int(hi_n[k] - lo_n[k]) - int(tr_n[k])
    return bd


def compute_overlap_sharded(ct: ColumnarTrace, attribution=None, device=None) -> Breakdown:
    """Each rank analyses its LPT share of the pids; returns the merged Breakdown."""
    import torch
    import torch.distributed as dist

    from . import _engine
    from .overlap import Attribution

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    mine = shard_pids(ct, world)[rank]
    local = ct.select_pids(mine)
    eng = _engine.get(torch.cuda.current_device())
    attr = 1 if attribution is not None and Attribution(attribution) is Attribution.CORRELATION else 0
    raw = eng.overlap(_engine.DeviceTrace(local, eng.device), attr)
    return merge_breakdown_raw(local, raw, device or torch.device("cuda", eng.device))
