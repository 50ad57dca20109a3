"""GPU parity: correct_trace / transition_sites / analyze through the C ABI
vs reference golden vectors, the CPU oracle and the closure property."""

from fractions import Fraction

import numpy as np
import pytest

import oracle
from golden_util import dec_profile, dec_trace, enc_breakdown, load
from paper_2102_04285_b200 import (
    CalibrationProfile,
    ColumnarTrace,
    InvalidTraceError,
    UncalibratedHookError,
    analyze_columnar,
    compute_overlap,
    correct_trace,
    correct_trace_columnar,
    count_transitions,
    synth,
    transition_sites,
)
from paper_2102_04285_b200.overlap import TRANSITION_PAIRS, transition_site_indices

pytestmark = pytest.mark.gpu

CORR = load("correction_cases.json.gz")
TRANS = load("transition_cases.json.gz")


@pytest.mark.parametrize("case", TRANS, ids=[c["name"] for c in TRANS])
def test_transition_sites_match_reference(case):
    trace = dec_trace(case["trace"])
    got = transition_site_indices(trace, 0xF)
    for (s, d), lst in got.items():
        assert lst == case["expect"][f"{int(s)}-{int(d)}"], (s, d)
    counts = count_transitions(trace)
    for s, d in TRANSITION_PAIRS:
        assert counts.get(s, d) == len(case["expect"][f"{int(s)}-{int(d)}"])


def test_transition_sites_return_events():
    trace = dec_trace(TRANS[0]["trace"])
    sites = transition_sites(trace)
    for pair, evs in sites.items():
        for e in evs:
            assert e in trace.events


@pytest.mark.parametrize("case", CORR, ids=[c["name"] for c in CORR])
def test_correction_matches_reference(case):
    trace = dec_trace(case["trace"])
    prof = dec_profile(case["profile"])
    exp = case["expect"]
    if "invalid" in exp:
        with pytest.raises(InvalidTraceError) as ei:
            correct_trace(trace, prof)
        assert [[v.rule, v.message, list(v.event_indices)] for v in ei.value.violations] == exp["invalid"]
        return
    if "uncalibrated" in exp:
        with pytest.raises(UncalibratedHookError) as ei:
            correct_trace(trace, prof)
        assert str(ei.value) == exp["uncalibrated"]
        return
    out, rep = correct_trace(trace, prof)
    assert [e.start for e in out.events] == exp["start"]
    assert [e.duration for e in out.events] == exp["dur"]
    assert [[m.pid, m.name, m.parent, m.fork_ns, m.join_ns] for m in out.processes] == exp["processes"]
    assert {str(k): v for k, v in rep.removed_ns.items()} == exp["removed_ns"]
    assert {str(k): v for k, v in rep.shortfall_ns.items()} == exp["shortfall_ns"]
    assert rep.original_total_ns == exp["original_total_ns"]
    assert rep.corrected_total_ns == exp["corrected_total_ns"]
    assert enc_breakdown(compute_overlap(out)) == exp["overlap_corrected"]
    # one-call analyze path (correct + overlap(corrected)) gives the same
    s, d, rep2, bd = analyze_columnar(ColumnarTrace.from_trace(trace), prof)
    assert s.cpu().numpy().tolist() == exp["start"]
    assert rep2.corrected_total_ns == exp["corrected_total_ns"]
    assert enc_breakdown(bd) == exp["overlap_corrected"]


def _frac_profile():
    return CalibrationProfile(Fraction(4001, 3), Fraction(999, 7), Fraction(1501, 2),
                              {"launch": Fraction(3001, 11), "memcpy": Fraction(997, 13)})


@pytest.mark.parametrize("iters,procs,outer,tid2", [(1500, 1, None, False), (300, 3, "iteration", True)])
def test_correction_synthetic_vs_oracle(iters, procs, outer, tid2):
    un, inst = synth.ddpg_trace(iters, processes=procs, outer_op=outer, second_tid_ops=tid2, both=True)
    for prof in (synth.exact_profile(), _frac_profile()):
        out, rep = correct_trace_columnar(inst, prof)
        s, d, orep, _ = oracle.correct(inst, prof)
        assert np.array_equal(out.start, s) and np.array_equal(out.dur, d)
        assert rep.removed_ns == orep["removed_ns"] and rep.shortfall_ns == orep["shortfall_ns"]
        assert rep.original_total_ns == orep["original_total_ns"]
        assert rep.corrected_total_ns == orep["corrected_total_ns"]


def test_correction_closure_1m():
    """Size-independent property: the exact profile undoes the instrumentation."""
    un, inst = synth.ddpg_trace(27027, both=True)
    out, rep = correct_trace_columnar(inst, synth.exact_profile())
    assert np.array_equal(out.start, un.start)
    assert np.array_equal(out.dur, un.dur)
    assert rep.original_total_ns - sum(sum(v.values()) for v in rep.removed_ns.values()) == rep.corrected_total_ns
