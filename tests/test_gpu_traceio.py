"""GPU: write_trace validates on the device before encoding, and the ingest
-> analyze path (read_trace_columnar -> analyze_columnar) equals analysing
the in-memory trace (the CLI's `analyze --profile DIR` flow, cli.py:160-171)."""

import numpy as np
import pytest

from paper_2102_04285_b200 import InvalidTraceError, analyze_columnar, read_trace_columnar, synth, write_trace
from paper_2102_04285_b200.model import Category, Event, ProcessMeta, Trace

pytestmark = pytest.mark.gpu


def test_write_trace_rejects_invalid(tmp_path):
    bad = Trace(1, [Event(1, 0, Category.BACKEND, "x", -5, 10)], [ProcessMeta(1, "p")])
    with pytest.raises(InvalidTraceError):
        write_trace(bad, tmp_path)


def test_ingest_then_analyze_equals_in_memory(tmp_path):
    un, inst = synth.config3_trace(processes=3, events_per_pid=40_000, both=True)
    write_trace(inst, tmp_path, chunk_limit_bytes=1 << 20)
    back = read_trace_columnar(tmp_path)
    s, d, rep, bd = analyze_columnar(back, synth.exact_profile())
    s0, d0, rep0, bd0 = analyze_columnar(inst, synth.exact_profile())
    assert bd.cells == bd0.cells and bd.spans == bd0.spans and bd.untracked == bd0.untracked
    assert rep.removed_ns == rep0.removed_ns and rep.corrected_total_ns == rep0.corrected_total_ns
    assert sorted(zip(s.cpu().numpy().tolist(), d.cpu().numpy().tolist())) == \
        sorted(zip(s0.cpu().numpy().tolist(), d0.cpu().numpy().tolist()))
