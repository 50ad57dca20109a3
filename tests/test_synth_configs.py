"""CPU checks of the config 3 / config 5 generators (test infrastructure):
valid traces per the oracle's validate_trace restatement, the advertised
shape (depth, skew, concurrency, zero-duration and duplicate-id fractions),
determinism, and pool == serial generation."""

import numpy as np

import oracle
from paper_2102_04285_b200 import synth

OP, GPU, API = 0, 5, 4


def _max_depth(ct, pid_idx, tid_value):
    g = [i for i in range(ct.n_groups) if ct.group_pid[i] == pid_idx and ct.group_tid[i] == tid_value][0]
    sel = (ct.tid == g) & (ct.cat == OP)
    s, e = ct.start[sel], ct.start[sel] + ct.dur[sel]
    ev = np.concatenate([np.stack([s, np.ones_like(s)], 1), np.stack([e, -np.ones_like(e)], 1)])
    ev = ev[np.lexsort((ev[:, 1], ev[:, 0]))]  # closes before opens at equal t
    return int(np.cumsum(ev[:, 1]).max())


def test_config3_shape_and_valid():
    ct = synth.config3_trace(processes=3, events_per_pid=30_000)
    assert oracle.validate_count(ct) == 0
    assert set(np.unique(ct.cat).tolist()) == set(range(6))
    assert abs(ct.n / 3 - 30_000) < 3_000
    assert _max_depth(ct, 0, 0) == 2 and _max_depth(ct, 0, 1) == 1


def test_config5_shape_and_valid():
    ct = synth.adversarial_trace(300_000, pids=16)
    assert oracle.validate_count(ct) == 0
    counts = np.bincount(ct.pid)
    assert counts.max() / ct.n > 0.3
    assert _max_depth(ct, int(np.argmax(counts)), 0) == 64
    res = ct.cat != OP
    zf = float((ct.dur[res] == 0).mean())
    assert 0.005 < zf < 0.02
    api = (ct.cat == API) & (ct.has_corr == 1)
    pid0 = ct.pid == np.argmax(counts)
    ids = ct.corr[api & pid0]
    assert 0.05 < 1 - np.unique(ids).size / ids.size < 0.15
    gpu_tids = np.unique(ct.tid[(ct.cat == GPU) & pid0])
    assert gpu_tids.size > 200


def test_generators_deterministic_and_pool_equal():
    a = synth.adversarial_trace(40_000, pids=4)
    b = synth.adversarial_trace(40_000, pids=4, workers=4)
    for f in ("start", "dur", "pid", "tid", "cat", "name", "corr", "has_corr", "group_pid", "group_tid"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    c = synth.config3_trace(processes=2, events_per_pid=5_000, workers=2)
    d = synth.config3_trace(processes=2, events_per_pid=5_000)
    assert np.array_equal(c.start, d.start) and np.array_equal(c.tid, d.tid)


def test_pid_batches_are_contiguous_whole_pids():
    from paper_2102_04285_b200.correction import _pid_batches

    ct = synth.config3_trace(processes=9, events_per_pid=5_000)
    parts = _pid_batches(ct, 4)
    assert parts[0][0] == 0 and parts[-1][1] == ct.n and len(parts) >= 2
    for (a, b), (c, _) in zip(parts, parts[1:]):
        assert b == c and ct.pid[b - 1] != ct.pid[b]  # cuts only at pid boundaries
    shuffled = ct.select_pids(list(range(ct.n_pids)))
    rev = np.argsort(-shuffled.start, kind="stable")  # rows no longer pid-contiguous
    from paper_2102_04285_b200.columnar import ColumnarTrace
    t2 = ColumnarTrace(ct.clock_domain, ct.start[rev], ct.dur[rev], ct.pid[rev], ct.tid[rev], ct.cat[rev],
                       ct.name[rev], ct.corr[rev], ct.has_corr[rev], ct.pids, ct.group_pid, ct.group_tid,
                       ct.names, ct.processes, ct.pid_has_meta)
    assert _pid_batches(t2, 4) == []
