"""GPU parity for the analyze-report companions:
busy_fraction, sampled_utilization, utilization_samples, summarize and
procview.build_process_tree through the C ABI (xs_union / xs_utilization),
bit-for-bit against the reference's own outputs (golden fixtures) and the
numpy oracle at larger sizes."""

import numpy as np
import pytest

import oracle
from golden_util import dec_trace, enc_breakdown, load
from paper_2102_04285_b200 import Category, synth
from paper_2102_04285_b200.metrics import busy_fraction, sampled_utilization, summarize, utilization_samples
from paper_2102_04285_b200.metrics import union_ns_per_pid
from paper_2102_04285_b200.overlap import compute_overlap
from paper_2102_04285_b200.procview import build_process_tree, render_tree, to_dot

pytestmark = pytest.mark.gpu

G = load("metrics_cases.json.gz")
MCASES, TCASES = G["metrics"], G["trees"]


def _run(fn):
    try:
        return fn()
    except ValueError as exc:  # InvalidTraceError is a ValueError, like the reference
        return {"error": type(exc).__name__}


@pytest.mark.parametrize("case", MCASES, ids=[c["name"] for c in MCASES])
def test_metrics_match_reference(case):
    tr = dec_trace(case["trace"])
    exp = case["expect"]
    for c, v in exp["busy"].items():
        assert _run(lambda: busy_fraction(tr, Category(int(c)))) == v, ("busy", c)
    for p, v in exp["sampled"].items():
        assert _run(lambda: sampled_utilization(tr, int(p))) == v, ("sampled", p)
    for p, v in exp["samples"].items():
        got = _run(lambda: utilization_samples(tr, int(p)))
        got = got if isinstance(got, dict) else [[s.period_start, s.period_ns, s.utilized] for s in got]
        assert got == v, ("samples", p)
    rows = _run(lambda: summarize(compute_overlap(tr)))
    rows = rows if isinstance(rows, dict) else [
        [r.pid, list(r.path), None if r.categories is None else sorted(int(c) for c in r.categories), r.ns, r.percent]
        for r in rows]
    assert rows == exp["summarize"]


@pytest.mark.parametrize("case", TCASES, ids=[c["name"] for c in TCASES])
def test_process_tree_matches_reference(case):
    traces = [dec_trace(t) for t in case["traces"]]

    def build():
        t = build_process_tree(traces)
        return {
            "nodes": sorted([n.pid, n.name, n.span_ns, n.gpu_busy_ns, enc_breakdown(n.breakdown)]
                            for n in t.nodes.values()),
            "children": sorted([k, list(v)] for k, v in t.children.items()),
            "roots": list(t.roots), "warnings": list(t.warnings), "render": render_tree(t), "dot": to_dot(t),
        }
    got = _run(build)
    exp = case["expect"]
    if "error" in exp:
        assert got == exp
        return
    got["nodes"] = [list(x) for x in got["nodes"]]
    assert got == exp


def test_union_and_utilization_vs_oracle_config3():
    ct = synth.config3_trace(processes=4, events_per_pid=60_000)
    per = union_ns_per_pid(ct, Category.GPU)
    assert per == oracle.union_ns(ct, 5, per_pid=True)
    lo, hi = oracle.trace_span(ct)
    for c in (1, 2, 3, 4, 5):
        assert busy_fraction(ct, Category(c)) == oracle.union_ns(ct, c) / (hi - lo)
    for period in (997, 50_000, 3_333_333):
        flags = oracle.utilization_flags(ct, period)
        assert sampled_utilization(ct, period) == sum(flags) / len(flags)
        got = utilization_samples(ct, period)
        assert [s.utilized for s in got] == flags


def test_union_adversarial_vs_oracle():
    ct = synth.adversarial_trace(200_000, pids=8)
    assert union_ns_per_pid(ct, Category.GPU) == oracle.union_ns(ct, 5, per_pid=True)
    assert union_ns_per_pid(ct, Category.BACKEND) == oracle.union_ns(ct, 2, per_pid=True)
    flags = oracle.utilization_flags(ct, 1 << 20)
    assert sampled_utilization(ct, 1 << 20) == sum(flags) / len(flags)
