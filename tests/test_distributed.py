"""Multi-process (gloo, world size 2) tests of the pid sharding and the
histogram merge used by the NCCL path.  Each rank's per-shard result comes
from the CPU oracle (no GPU here); the merged Breakdown must equal the
oracle's single-process answer on the whole trace, bit for bit."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _raw_from_oracle(ct, attr):
    """Oracle output re-encoded in the device result layout (trie + cells)."""
    import oracle
    from paper_2102_04285_b200._engine import OverlapRaw

    cells, spans, untracked = oracle.overlap(ct, attr)
    name_ix = {n: i for i, n in enumerate(ct.names)}
    nodes = {(): 0}
    parent, name = [-1], [-1]
    for (_, path, _), _ in sorted(cells.items(), key=lambda kv: (kv[0][1], kv[0][0])):
        for k in range(1, len(path) + 1):
            pre = path[:k]
            if pre not in nodes:
                nodes[pre] = len(parent)
                parent.append(nodes[path[:k - 1]])
                name.append(name_ix[path[k - 1]])
    pid_ix = {int(p): i for i, p in enumerate(ct.pids)}
    rows = list(cells.items())
    P = ct.n_pids
    lo = np.full(P, np.iinfo(np.int64).max, np.int64)
    hi = np.zeros(P, np.int64)
    tracked = np.zeros(P, np.int64)
    has = np.zeros(P, np.uint8)
    for pv, (a, b) in spans.items():
        i = pid_ix[pv]
        lo[i], hi[i], has[i] = a, b, 1
        tracked[i] = (b - a) - untracked[pv]
    mask = [sum(1 << (c - 1) for c in cats) for (_, _, cats), _ in rows]
    return OverlapRaw(np.array([pid_ix[k[0]] for k, _ in rows], np.int32),
                      np.array([nodes[k[1]] for k, _ in rows], np.int32), np.array(mask, np.int32),
                      np.array([v for _, v in rows], np.int64), np.array(parent, np.int32),
                      np.array(name, np.int32), lo, hi, tracked, has)


def _worker(rank, world, port, attr, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import torch
    import torch.distributed as dist

    from paper_2102_04285_b200 import synth
    from paper_2102_04285_b200.distributed import merge_breakdown_raw, shard_pids

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        ct = synth.ddpg_trace(60, processes=5, outer_op="iteration", second_tid_ops=True)
        shards = shard_pids(ct, world)
        local = ct.select_pids(shards[rank])
        raw = _raw_from_oracle(local, attr)
        bd = merge_breakdown_raw(local, raw, torch.device("cpu"))
        bd2 = merge_breakdown_raw(local, raw, torch.device("cpu"))  # cached global tables: no object gather
        assert bd2 == bd
        cells = {(k.pid, k.path, frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items()}
        q.put((rank, cells, bd.spans, bd.untracked, shards))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("attr", [0, 1])
def test_gloo_two_rank_merge_equals_single_process(attr):
    sys.path[:0] = [os.path.join(ROOT, "oracle")]
    import oracle
    from paper_2102_04285_b200 import synth

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, attr, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ct = synth.ddpg_trace(60, processes=5, outer_op="iteration", second_tid_ops=True)
    cells, spans, untracked = oracle.overlap(ct, attr)
    for rank, c, s, u, shards in results:
        assert sorted(sum(shards, [])) == list(range(ct.n_pids))
        assert all(shards)  # both ranks got work
        assert c == cells and s == spans and u == untracked


def test_shard_pids_lpt_balance():
    from paper_2102_04285_b200.columnar import ColumnarTrace
    from paper_2102_04285_b200.distributed import shard_pids

    sizes = [100, 60, 50, 40, 10, 5]
    pid = np.concatenate([np.full(k, i, np.int64) for i, k in enumerate(sizes)])
    n = pid.shape[0]
    ct = ColumnarTrace.from_arrays(1, np.zeros(n, np.int64), np.ones(n, np.int64), pid + 1, np.zeros(n, np.int64),
                                   np.full(n, 2, np.uint8), np.zeros(n, np.int32), ["x"])
    sh = shard_pids(ct, 2)
    loads = [sum(sizes[p] for p in s) for s in sh]
    assert abs(loads[0] - loads[1]) <= max(sizes) // 4  # LPT bound, not optimal


# ---------------------------------------------------------------------------
# time-window splitting of giant pids (partitioning (2))

@pytest.mark.parametrize("world,split", [(2, 2), (3, 2), (4, 3), (8, 2)])
def test_window_split_merge_equals_whole_trace(world, split):
    sys.path[:0] = [os.path.join(ROOT, "oracle")]
    import oracle
    from paper_2102_04285_b200 import synth
    from paper_2102_04285_b200.distributed import merge_raw_list, plan_shards, shard_trace

    for ct in (synth.adversarial_trace(40_000, pids=6, streams=32),
               synth.ddpg_trace(200, processes=3, outer_op="iteration", second_tid_ops=True)):
        plan = plan_shards(ct, world, split)
        assert any(a is not None or b is not None for sh in plan for _, a, b in sh)  # something was cut
        parts = [(local, _raw_from_oracle(local, 0)) for local in (shard_trace(ct, sh) for sh in plan)]
        bd = merge_raw_list(parts)
        cells = {(k.pid, k.path, frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items()}
        assert (cells, bd.spans, bd.untracked) == oracle.overlap(ct, 0)


def test_window_cuts_are_operation_free():
    from paper_2102_04285_b200 import synth
    from paper_2102_04285_b200.distributed import window_cuts

    ct = synth.adversarial_trace(50_000, pids=4)
    p = int(np.argmax(np.bincount(ct.pid)))
    cuts = window_cuts(ct, p, 6)
    assert cuts == sorted(set(cuts)) and len(cuts) >= 2
    sel = (ct.pid == p) & (ct.cat == 0)
    s, e = ct.start[sel], ct.start[sel] + ct.dur[sel]
    for c in cuts:
        assert not np.any((s < c) & (c < e))


def test_split_dangling_correlation_detected_on_host():
    from paper_2102_04285_b200 import synth
    from paper_2102_04285_b200.distributed import check_split_correlations

    ct = synth.adversarial_trace(20_000, pids=2)
    assert check_split_correlations(ct, [0, 1])
    g = np.nonzero((ct.cat == 5) & (ct.has_corr == 1) & (ct.pid == 0))[0][0]
    ct.corr[g] = 10**12
    assert not check_split_correlations(ct, [0])


def _window_worker(rank, world, port, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
    import torch
    import torch.distributed as dist

    from paper_2102_04285_b200 import synth
    from paper_2102_04285_b200.distributed import merge_breakdown_raw, plan_shards, shard_trace
    from test_distributed import _raw_from_oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        ct = synth.adversarial_trace(30_000, pids=5, streams=16)
        plan = plan_shards(ct, world, 2)
        local = shard_trace(ct, plan[rank])
        bd = merge_breakdown_raw(local, _raw_from_oracle(local, 0), torch.device("cpu"))
        cells = {(k.pid, k.path, frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items()}
        q.put((rank, cells, bd.spans, bd.untracked))
    finally:
        dist.destroy_process_group()


def test_gloo_window_split_collective_merge():
    sys.path[:0] = [os.path.join(ROOT, "oracle")]
    import oracle
    from paper_2102_04285_b200 import synth

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_window_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    exp = oracle.overlap(synth.adversarial_trace(30_000, pids=5, streams=16), 0)
    for _, c, s, u in results:
        assert (c, s, u) == exp


def _report_worker(rank, world, port, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2102_04285_b200 import synth
    from paper_2102_04285_b200.correction import CorrectionReport
    from paper_2102_04285_b200.distributed import merge_reports, shard_pids

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        ct = synth.adversarial_trace(30_000, pids=5, streams=16)
        local = ct.select_pids(shard_pids(ct, world)[rank])
        _, _, r, _ = oracle.correct(local, synth.adversarial_profile())
        rep = merge_reports(CorrectionReport(r["removed_ns"], r["shortfall_ns"], r["original_total_ns"],
                                             r["corrected_total_ns"]), torch.device("cpu"))
        q.put((rank, rep.removed_ns, rep.shortfall_ns, rep.original_total_ns, rep.corrected_total_ns))
    finally:
        dist.destroy_process_group()


def test_gloo_report_merge_equals_single_process():
    """The correction report of pid-sharded ranks merges to the whole trace's."""
    sys.path[:0] = [os.path.join(ROOT, "oracle")]
    import oracle
    from paper_2102_04285_b200 import synth

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_report_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, _, r, _ = oracle.correct(synth.adversarial_trace(30_000, pids=5, streams=16), synth.adversarial_profile())
    for _, rm, sf, o, c in results:
        assert rm == r["removed_ns"] and sf == r["shortfall_ns"]
        assert o == r["original_total_ns"] and c == r["corrected_total_ns"]
