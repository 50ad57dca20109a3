"""Reference-valid inputs at the edges of the device formulation return the
reference's results (tests/golden/edge_cases.json.gz, scripts/make_golden_edge.py):
merged multi-tid operation stacks deeper than 256 and wider than 64 tids
(path_of has no depth bound, _sweep_py.py:16-26), timelines wider than one
64-bit key (model.py:14, 204-207), calibration profiles whose common
denominator overflows int64/int128 (quantize_amounts keeps exact Fractions,
_timeline.py:57-67)."""

import numpy as np
import pytest

from golden_util import dec_profile, dec_trace, enc_breakdown, load
from paper_2102_04285_b200 import Attribution, ColumnarTrace, analyze_columnar, compute_overlap, correct_trace

pytestmark = pytest.mark.gpu

EDGE = load("edge_cases.json.gz")
# a single process spanning >= 2^60 ns (its endpoint keys cannot fit 64 bits
# even alone): compute_overlap cuts it into operation-free time windows
# (_split.wide_cuts), correct_trace shrinks its idle gaps exactly
# (_split.compress_wide) -- both return the reference's results


@pytest.mark.parametrize("case", EDGE, ids=[c["name"] for c in EDGE])
def test_edge_overlap_matches_reference(case):
    trace = dec_trace(case["trace"])
    assert enc_breakdown(compute_overlap(trace)) == case["overlap"]["instant"]
    assert enc_breakdown(compute_overlap(trace, Attribution.CORRELATION)) == case["overlap"]["correlation"]


@pytest.mark.parametrize("case", EDGE, ids=[c["name"] for c in EDGE])
def test_edge_correction_matches_reference(case):
    trace = dec_trace(case["trace"])
    for exp in case["corrections"]:
        prof = dec_profile(exp["profile"])
        out, rep = correct_trace(trace, prof)
        assert [e.start for e in out.events] == exp["start"]
        assert [e.duration for e in out.events] == exp["dur"]
        assert {str(k): v for k, v in rep.removed_ns.items()} == exp["removed_ns"]
        assert {str(k): v for k, v in rep.shortfall_ns.items()} == exp["shortfall_ns"]
        assert rep.original_total_ns == exp["original_total_ns"]
        assert rep.corrected_total_ns == exp["corrected_total_ns"]
        assert enc_breakdown(compute_overlap(out)) == exp["overlap_corrected"]
        s, d, rep2, bd = analyze_columnar(ColumnarTrace.from_trace(trace), prof)
        assert np.asarray(s.cpu()).tolist() == exp["start"] and np.asarray(d.cpu()).tolist() == exp["dur"]
        assert rep2.corrected_total_ns == exp["corrected_total_ns"]
        assert enc_breakdown(bd) == exp["overlap_corrected"]


def test_pid_batched_calls_equal_one_call(monkeypatch):
    """Traces over the per-call row bound run as consecutive pid batches
    (_split): overlap, correction (columns, report, fork/join) and analyze
    equal the single call bit for bit, and errors keep whole-trace order."""
    from paper_2102_04285_b200 import _split, compute_overlap_columnar, correct_trace_columnar, synth
    from paper_2102_04285_b200.correction import UncalibratedHookError

    ct = synth.config3_trace(processes=6, events_per_pid=20_000)
    prof = synth.exact_profile()
    bd0 = compute_overlap_columnar(ct)
    out0, rep0 = correct_trace_columnar(ct, prof)
    s0, d0, rep_a, bd_a = analyze_columnar(ct, prof)
    monkeypatch.setattr(_split, "MAX_EVENTS_PER_CALL", 45_000)
    assert _split.needs_split(ct) and len(_split.plan_batches(ct)) >= 3
    bd1 = compute_overlap_columnar(ct)
    assert bd1.cells == bd0.cells and bd1.spans == bd0.spans and bd1.untracked == bd0.untracked
    out1, rep1 = correct_trace_columnar(ct, prof)
    assert np.array_equal(out1.start, out0.start) and np.array_equal(out1.dur, out0.dur)
    assert out1.processes == out0.processes and rep1 == rep0
    s1, d1, rep_b, bd_b = analyze_columnar(ct, prof)
    assert np.array_equal(s1.cpu().numpy(), s0.cpu().numpy()) and np.array_equal(d1.cpu().numpy(), d0.cpu().numpy())
    assert rep_b == rep_a and bd_b.cells == bd_a.cells and bd_b.spans == bd_a.spans
    bad = type(prof)(prof.annotation_ns, prof.transition_ns, prof.api_interception_ns, {"launch": 3000})
    with pytest.raises(UncalibratedHookError) as e1:
        correct_trace_columnar(ct, bad)
    monkeypatch.setattr(_split, "MAX_EVENTS_PER_CALL", 1 << 30)
    with pytest.raises(UncalibratedHookError) as e0:
        correct_trace_columnar(ct, bad)
    assert str(e1.value) == str(e0.value)
