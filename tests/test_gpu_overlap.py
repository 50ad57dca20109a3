"""GPU parity: compute_overlap through the C ABI vs reference golden vectors
and vs the CPU oracle on synthetic traces (bit-exact int64 cells)."""

import numpy as np
import pytest

import oracle
from golden_util import dec_trace, enc_breakdown, load
from paper_2102_04285_b200 import Attribution, ColumnarTrace, InvalidTraceError, compute_overlap
from paper_2102_04285_b200 import compute_overlap_columnar, synth

pytestmark = pytest.mark.gpu

OVERLAP = load("overlap_cases.json.gz")


def _attr(name):
    return Attribution.INSTANT if name == "instant" else Attribution.CORRELATION


@pytest.mark.parametrize("case", OVERLAP, ids=[c["name"] for c in OVERLAP])
def test_overlap_matches_reference_golden(case):
    trace = dec_trace(case["trace"])
    for attr, exp in case["expect"].items():
        if "invalid" in exp:
            with pytest.raises(InvalidTraceError) as ei:
                compute_overlap(trace, _attr(attr))
            got = [[v.rule, v.message, list(v.event_indices)] for v in ei.value.violations]
            assert got == exp["invalid"]
            continue
        bd = compute_overlap(trace, _attr(attr))
        assert enc_breakdown(bd) == exp, attr


def _oracle_bd(ct, attr):
    cells, spans, untracked = oracle.overlap(ct, attr)
    return cells, spans, untracked


def _ours(bd):
    cells = {(k.pid, k.path, frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items()}
    return cells, bd.spans, bd.untracked


@pytest.mark.parametrize("iters,procs,outer,tid2", [(2000, 1, None, False), (400, 3, "iteration", False),
                                                     (300, 2, "iteration", True)])
def test_overlap_synthetic_vs_oracle(iters, procs, outer, tid2):
    un, inst = synth.ddpg_trace(iters, processes=procs, outer_op=outer, second_tid_ops=tid2, both=True)
    for ct in (un, inst):
        for attr in (0, 1):
            bd = compute_overlap_columnar(ct, Attribution.CORRELATION if attr else Attribution.INSTANT)
            assert _ours(bd) == _oracle_bd(ct, attr)


def test_overlap_1m_ddpg_vs_oracle():
    ct = synth.ddpg_trace(27027)
    bd = compute_overlap_columnar(ct)
    assert _ours(bd) == _oracle_bd(ct, 0)
    # conservation (test_overlap.py:177-185)
    for pid, (lo, hi) in bd.spans.items():
        assert bd.total_attributed(pid) + bd.untracked[pid] == hi - lo


def test_overlap_repeat_calls_reuse_workspace():
    ct = synth.ddpg_trace(500, processes=2)
    a = compute_overlap_columnar(ct)
    b = compute_overlap_columnar(ct)
    assert a == b


def _dense_trace(n_same: int, seed: int = 0):
    """Many endpoints on a few identical timestamps: forces dense buckets."""
    from paper_2102_04285_b200.columnar import ColumnarTrace
    from paper_2102_04285_b200.model import ProcessMeta

    rng = np.random.default_rng(seed)
    start = np.concatenate([np.zeros(n_same, np.int64), rng.integers(0, 10**9, 4000)])
    dur = np.concatenate([rng.integers(1, 50, n_same), rng.integers(1, 10**6, 4000)])
    cat = rng.integers(1, 6, start.shape[0]).astype(np.uint8)
    cat[:3] = 0  # a few ops at t=0 (nested: equal start, distinct ends)
    dur[:3] = [10**9 + 10, 10**9 + 5, 10**9]
    n = start.shape[0]
    names = ["a", "b", "c", "x"]
    name = np.where(cat == 0, np.arange(n) % 3, 3).astype(np.int32)
    return ColumnarTrace.from_arrays(1, start, dur, np.ones(n, np.int64), np.zeros(n, np.int64), cat, name, names,
                                     processes=(ProcessMeta(1, "p"),))


@pytest.mark.parametrize("n_same", [200, 5000])
def test_overlap_dense_buckets_vs_oracle(n_same):
    """200 identical starts -> in-block radix sort branch; 5000 -> bucket overflow -> LSD fallback."""
    ct = _dense_trace(n_same)
    bd = compute_overlap_columnar(ct)
    assert _ours(bd) == _oracle_bd(ct, 0)


SWEEP = load("sweep_pid_cases.json.gz")


class _PathTable:  # the reference's PathTable protocol (overlap.py:80-93)
    def __init__(self):
        self._ids, self.paths = {}, []

    def get_id(self, key):
        if key not in self._ids:
            self._ids[key] = len(self.paths)
            self.paths.append(key)
        return self._ids[key]


@pytest.mark.parametrize("k", range(len(SWEEP)))
def test_sweep_pid_plugin_shim_matches_reference_kernel(k):
    """paper_2102_04285_b200.sweep_pid is a drop-in for the reference's
    `kernel=` plugin (the inputs recorded from the reference's compute_overlap)."""
    from paper_2102_04285_b200 import sweep_pid

    case = SWEEP[k]
    pt = _PathTable()
    for path in case.get("paths", []):  # CORRELATION calls: the ids fixed_paths refer to
        pt.get_id(tuple(path))
    cells, tracked = sweep_pid(*case["args"], pt)
    got = sorted([list(pt.paths[key >> 6]), key & 63, v] for key, v in cells.items())
    assert got == case["cells"] and tracked == case["tracked"]
