"""Host logic of the exact gap compression used to correct a process too
wide for one call's keys (_split.compress_wide / uncompress_columns,
correction._correct_wide): correcting the compressed trace with the C oracle
and shifting the columns back gives the oracle's (and, for the reference's
2^62-wide golden case, the reference's) correction of the original trace --
columns, removed / shortfall, and fork / join through compress_time."""

import numpy as np
import pytest

import oracle
from golden_util import dec_profile, dec_trace, load
from paper_2102_04285_b200 import _split, synth
from paper_2102_04285_b200.columnar import ColumnarTrace


def _via_compression(ct, prof, queries=()):
    pids = list(range(ct.n_pids))
    ctc, comp = _split.compress_wide(ct, pids, prof)
    qc, meta = [], []
    for p, t in queries:
        t2, off, tail = comp.compress_time(p, t)
        qc.append((p, t2))
        meta.append(off + tail)
    s, d, rep, q = oracle.correct(ctc, prof, qc)
    s2, d2 = _split.uncompress_columns(ct, comp, s, d)
    return s2, d2, rep, [int(v) + m for v, m in zip(q, meta)]


def test_wide_golden_case_correction():
    case = [c for c in load("edge_cases.json.gz") if c["name"] == "single_pid_span_2e62"][0]
    ct = ColumnarTrace.from_trace(dec_trace(case["trace"]))
    for exp in case["corrections"]:
        prof = dec_profile(exp["profile"])
        ctc, _ = _split.compress_wide(ct, [0], prof)
        span = int((ctc.start + ctc.dur).max() - ctc.start.min())
        assert span.bit_length() <= _split.WIDE_BITS  # now fits one call's keys
        s, d, rep, _ = _via_compression(ct, prof)
        assert s.tolist() == exp["start"] and d.tolist() == exp["dur"]
        assert {str(k): v for k, v in rep["removed_ns"].items()} == exp["removed_ns"]
        assert {str(k): v for k, v in rep["shortfall_ns"].items()} == exp["shortfall_ns"]


def _with_gaps(ct, seed):
    """The trace with huge idle gaps inserted at operation-free instants."""
    rng = np.random.default_rng(seed)
    from paper_2102_04285_b200.distributed import op_free_gaps
    start = ct.start.copy()
    end = ct.start + ct.dur
    for p in range(ct.n_pids):
        gaps = op_free_gaps(ct, p)
        inner = gaps[1:-1]
        if inner.shape[0] == 0:
            continue
        pick = inner[rng.choice(inner.shape[0], size=min(4, inner.shape[0]), replace=False)]
        for lo, hi in sorted(map(tuple, pick.tolist())):
            c = (lo + hi) // 2
            g = int(rng.integers(1 << 40, 1 << 50))
            sel = ct.pid == p
            # events that start at or after c move; events straddling c (not
            # operations) stretch
            start = np.where(sel & (start >= c), start + g, start)
            end = np.where(sel & (end > c), end + g, end)
    return ColumnarTrace(ct.clock_domain, start, end - start, ct.pid, ct.tid, ct.cat, ct.name, ct.corr,
                         ct.has_corr, ct.pids, ct.group_pid, ct.group_tid, ct.names, ct.processes, ct.pid_has_meta)


@pytest.mark.parametrize("seed", range(5))
def test_gapped_traces_correct_exactly(seed):
    base = synth.ddpg_trace(120, processes=2, seed=seed)
    ct = _with_gaps(base, seed)
    for prof in (synth.exact_profile(), synth.adversarial_profile()):
        s0, d0, rep0, q0 = oracle.correct(ct, prof, [(0, int(ct.start[ct.pid == 0].max()) + 7), (1, 12345)])
        s, d, rep, q = _via_compression(ct, prof, [(0, int(ct.start[ct.pid == 0].max()) + 7), (1, 12345)])
        assert np.array_equal(s, s0) and np.array_equal(d, d0)
        assert rep["removed_ns"] == rep0["removed_ns"] and rep["shortfall_ns"] == rep0["shortfall_ns"]
        assert list(q) == [int(v) for v in q0]


def test_compression_shrinks_only_long_gaps():
    ct = _with_gaps(synth.ddpg_trace(60, processes=1, seed=9), 9)
    prof = synth.exact_profile()
    ctc, comp = _split.compress_wide(ct, [0], prof)
    L = comp.L[0]
    pts = comp.points[0]
    newp = pts - comp.cum[0]
    d0, d1 = np.diff(pts), np.diff(newp)
    assert np.array_equal(d1, np.minimum(d0, L))  # gaps > L become L, the rest keep their length
