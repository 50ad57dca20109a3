"""A single process with more rows than one device call takes
(_split.MAX_EVENTS_PER_CALL, forced small here): correct_trace / analyze run
it as time windows, call by call, with the window carries; compute_overlap as
operation-free windows.  Results (columns, report, fork / join, Breakdown)
equal the one-call results."""

from dataclasses import replace

import numpy as np
import pytest

from paper_2102_04285_b200 import _split, analyze_columnar, compute_overlap_columnar, correct_trace_columnar
from paper_2102_04285_b200.model import ProcessMeta
from test_window_correction import _profiles, _trace

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prof", ["exact", "ladder"])
def test_huge_process_windows(monkeypatch, prof):
    ct = _trace("ddpg1")
    lo, hi = int(ct.start.min()), int((ct.start + ct.dur).max())
    ct = replace(ct, processes=(ProcessMeta(1, "ddpg", None, lo + (hi - lo) // 3, hi + 11),))
    profile = _profiles()[prof]
    out0, rep0 = correct_trace_columnar(ct, profile)
    s0, d0, rep_a, bd_a = analyze_columnar(ct, profile)
    bd0 = compute_overlap_columnar(ct)
    monkeypatch.setattr(_split, "MAX_EVENTS_PER_CALL", ct.n // 3)
    assert _split.needs_split(ct)
    out1, rep1 = correct_trace_columnar(ct, profile)
    assert np.array_equal(out1.start, out0.start) and np.array_equal(out1.dur, out0.dur)
    assert out1.processes == out0.processes and rep1 == rep0
    s1, d1, rep_b, bd_b = analyze_columnar(ct, profile)
    assert np.array_equal(s1.cpu().numpy(), s0.cpu().numpy()) and np.array_equal(d1.cpu().numpy(), d0.cpu().numpy())
    assert rep_b == rep_a and bd_b == bd_a
    assert compute_overlap_columnar(ct) == bd0
