"""Pin the CPU oracle against the reference's own outputs (tests/golden)."""

import numpy as np
import pytest

import oracle
from golden_util import dec_profile, dec_trace, enc_cells, load
from paper_2102_04285_b200.columnar import ColumnarTrace

OVERLAP = load("overlap_cases.json.gz")
TRANS = load("transition_cases.json.gz")
CORR = load("correction_cases.json.gz")


@pytest.mark.parametrize("case", OVERLAP, ids=[c["name"] for c in OVERLAP])
def test_oracle_overlap_matches_reference(case):
    ct = ColumnarTrace.from_trace(dec_trace(case["trace"]))
    for attr, exp in case["expect"].items():
        if "invalid" in exp:
            assert oracle.validate_count(ct) > 0
            with pytest.raises(oracle.OracleInvalid):
                oracle.overlap(ct, 0 if attr == "instant" else 1)
            continue
        cells, spans, untracked = oracle.overlap(ct, 0 if attr == "instant" else 1)
        assert enc_cells(cells) == exp["cells"], attr
        assert sorted([p, lo, hi] for p, (lo, hi) in spans.items()) == exp["spans"]
        assert sorted([p, v] for p, v in untracked.items()) == exp["untracked"]


@pytest.mark.parametrize("case", TRANS, ids=[c["name"] for c in TRANS])
def test_oracle_transitions_match_reference(case):
    ct = ColumnarTrace.from_trace(dec_trace(case["trace"]))
    got = oracle.transition_sites(ct, 0xF)
    for (s, d), lst in got.items():
        assert lst == case["expect"][f"{s}-{d}"], (s, d)


@pytest.mark.parametrize("case", CORR, ids=[c["name"] for c in CORR])
def test_oracle_correction_matches_reference(case):
    trace = dec_trace(case["trace"])
    ct = ColumnarTrace.from_trace(trace)
    prof = dec_profile(case["profile"])
    exp = case["expect"]
    if "invalid" in exp:
        with pytest.raises(oracle.OracleInvalid):
            oracle.correct(ct, prof)
        return
    if "uncalibrated" in exp:
        with pytest.raises(oracle.OracleUncalibrated) as ei:
            oracle.correct(ct, prof)
        assert repr(trace.events[ei.value.event_index].name) in exp["uncalibrated"]
        return
    pid_index = {int(p): i for i, p in enumerate(ct.pids)}
    queries = []
    for m in trace.processes:
        for v in (m.fork_ns, m.join_ns):
            if v is not None:
                queries.append((pid_index[m.pid], v))
    s, d, rep, q = oracle.correct(ct, prof, queries)
    assert s.tolist() == exp["start"]
    assert d.tolist() == exp["dur"]
    assert {str(k): v for k, v in rep["removed_ns"].items()} == exp["removed_ns"]
    assert {str(k): v for k, v in rep["shortfall_ns"].items()} == exp["shortfall_ns"]
    assert rep["original_total_ns"] == exp["original_total_ns"]
    assert rep["corrected_total_ns"] == exp["corrected_total_ns"]
    present = {m.pid for m in trace.processes} & {e.pid for e in trace.events}
    qi = iter(q)
    for m, em in zip(trace.processes, exp["processes"]):
        fork = m.fork_ns if m.fork_ns is None else next(qi)
        join = m.join_ns if m.join_ns is None else next(qi)
        if m.pid in present:
            assert [fork, join] == em[3:5]
    # overlap of the corrected trace
    ct2 = ColumnarTrace.from_trace(trace)
    ct2.start = np.asarray(exp["start"], np.int64)
    ct2.dur = np.asarray(exp["dur"], np.int64)
    cells, _, _ = oracle.overlap(ct2, 0)
    assert enc_cells(cells) == exp["overlap_corrected"]["cells"]
