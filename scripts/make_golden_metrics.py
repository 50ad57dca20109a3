#!/usr/bin/env python3
"""Generate tests/golden/metrics_cases.json.gz by running the REFERENCE here:
metrics.busy_fraction / sampled_utilization / utilization_samples / summarize
(metrics.py:61-126) and procview.build_process_tree / render_tree / to_dot
(procview.py:45-147) on fixed inputs (the reference tests' own traces plus
seeded random traces).  Run from the repo root after oracle/build_ref.sh:

    python scripts/make_golden_metrics.py
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

from xstrace.metrics import busy_fraction, sampled_utilization, summarize, utilization_samples  # noqa: E402
from xstrace.model import Category, Event, InvalidTraceError, ProcessMeta, Trace  # noqa: E402
from xstrace.overlap import compute_overlap  # noqa: E402
from xstrace.procview import build_process_tree, render_tree, to_dot  # noqa: E402
from xstrace.synth import (  # noqa: E402
    expand_leaf_trace,
    generate_workload,
    minigo_like_traces,
    preset_exact,
    random_trace,
    sparse_kernel_trace,
)

sys.path.insert(0, HERE)
from make_golden import enc_breakdown, enc_trace  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
G, B, H, O = Category.GPU, Category.BACKEND, Category.HIGH_LEVEL, Category.OPERATION


def guard(fn):
    try:
        return fn()
    except (ValueError, InvalidTraceError) as exc:
        return {"error": type(exc).__name__}


def metric_case(name, trace, periods):
    span = None
    if trace.events:
        span = max(e.end for e in trace.events) - min(e.start for e in trace.events)
    exp = {"busy": {int(c): guard(lambda c=c: busy_fraction(trace, c)) for c in Category}}
    exp["sampled"] = {}
    exp["samples"] = {}
    for p in periods:
        exp["sampled"][p] = guard(lambda p=p: sampled_utilization(trace, p))
        if span is not None and span // max(p, 1) <= 2000:
            s = guard(lambda p=p: utilization_samples(trace, p))
            exp["samples"][p] = s if isinstance(s, dict) else [[x.period_start, x.period_ns, x.utilized] for x in s]
    rows = guard(lambda: summarize(compute_overlap(trace)))
    exp["summarize"] = rows if isinstance(rows, dict) else [
        [r.pid, list(r.path), None if r.categories is None else sorted(int(c) for c in r.categories), r.ns, r.percent]
        for r in rows]
    return {"name": name, "trace": enc_trace(trace), "expect": exp}


def tree_case(name, traces):
    def build():
        t = build_process_tree(traces)
        return {
            "nodes": sorted([n.pid, n.name, n.span_ns, n.gpu_busy_ns, enc_breakdown(n.breakdown)]
                            for n in t.nodes.values()),
            "children": sorted([k, list(v)] for k, v in t.children.items()),
            "roots": list(t.roots), "warnings": list(t.warnings),
            "render": render_tree(t), "dot": to_dot(t),
        }
    return {"name": name, "traces": [enc_trace(t) for t in traces], "expect": guard(build)}


def main():
    P = [ProcessMeta(1, "p")]
    m_cases = []
    hand = {
        "no_gpu": [Event(1, 0, B, "x", 0, 1000)],
        "gpu_full": [Event(1, 9, G, "kernel", 0, 1000)],
        "clipped_tail": [Event(1, 0, B, "x", 5, 1003)],
        "half_span": [Event(1, 0, B, "x", 0, 100), Event(1, 9, G, "kernel", 0, 50)],
        "overlap_once": [Event(1, 0, H, "s", 0, 100), Event(1, 9, G, "a", 10, 30), Event(1, 10, G, "b", 20, 30)],
        "touching_gpu": [Event(1, 0, H, "s", 0, 100), Event(1, 9, G, "a", 10, 10), Event(1, 10, G, "b", 20, 10),
                         Event(1, 9, G, "z", 20, 0), Event(1, 9, G, "c", 95, 5)],
        "untracked": [Event(1, 0, B, "x", 0, 60), Event(1, 0, O, "op", 0, 100)],
        "zero_span": [Event(1, 0, B, "x", 7, 0)],
        "invalid": [Event(1, 0, B, "x", -1, 5)],
    }
    for k, ev in hand.items():
        m_cases.append(metric_case(k, Trace(1, ev, P), [1, 3, 7, 10, 100, 1000]))
    m_cases.append(metric_case("empty", Trace(1, [], []), [10]))
    m_cases.append(metric_case("empty_with_meta", Trace(1, [], P), [10]))
    m_cases.append(metric_case("expand_leaf", expand_leaf_trace(), [1000, 100_000, 333_333]))
    m_cases.append(metric_case("sparse_kernels", sparse_kernel_trace(), [166_666_667, 50_000_000, 999_999_937]))
    for seed in range(120):
        rng = random.Random(seed)
        tr = random_trace(rng, max_events=120, max_span=rng.choice([200, 5_000, 20_000, 1_000_000]),
                          pids=1 + seed % 3)
        lo = min(e.start for e in tr.events)
        span = max(e.end for e in tr.events) - lo
        periods = sorted({1 + seed % 5, max(1, span // 7), max(1, -(-span // 3)), max(1, span // 50), span + 1})
        m_cases.append(metric_case(f"random_{seed}", tr, periods))
    for seed in (13, 21):
        un, inst, _ = generate_workload(preset_exact(seed=seed, iterations=3))
        m_cases.append(metric_case(f"workload_un_{seed}", un, [1_000_000, 137_000]))
        m_cases.append(metric_case(f"workload_inst_{seed}", inst, [1_000_000]))

    t_cases = []
    two = Trace(1, [Event(1, 0, B, "x", 0, 100), Event(1, 9, G, "k", 10, 30)], P)
    t_cases.append(tree_case("single", [two]))
    t_cases.append(tree_case("duplicate_pid", [two, two]))
    t_cases.append(tree_case("clock_mismatch", [two, Trace(99, [Event(2, 0, B, "x", 0, 5)], [ProcessMeta(2, "q")])]))
    t_cases.append(tree_case("orphan", [two, Trace(1, [Event(5, 0, B, "x", 0, 5)],
                                                   [ProcessMeta(5, "lost", parent=404)])]))
    t_cases.append(tree_case("multi_pid_one_trace", [Trace(1, [Event(1, 0, H, "parent", 0, 100),
                                                              Event(2, 0, H, "child", 10, 50)],
                                                           [ProcessMeta(1, "root"),
                                                            ProcessMeta(2, "worker", parent=1, fork_ns=10,
                                                                        join_ns=60)])]))
    t_cases.append(tree_case("fork_outside", [Trace(1, [Event(1, 0, H, "parent", 0, 100),
                                                       Event(2, 0, H, "child", 10, 50)],
                                                    [ProcessMeta(1, "root"),
                                                     ProcessMeta(2, "worker", parent=1, fork_ns=500)])]))
    t_cases.append(tree_case("meta_without_events", [Trace(1, [Event(1, 0, H, "parent", 0, 100)],
                                                           [ProcessMeta(1, "root"),
                                                            ProcessMeta(3, "idle", parent=1)])]))
    t_cases.append(tree_case("minigo_3", minigo_like_traces(workers=3)))
    t_cases.append(tree_case("minigo_16", minigo_like_traces()))
    for seed in range(10):
        tr = random_trace(random.Random(1000 + seed), max_events=150, pids=3)
        t_cases.append(tree_case(f"random_{seed}", [tr]))

    with gzip.open(os.path.join(OUT, "metrics_cases.json.gz"), "wt", encoding="utf-8") as fh:
        json.dump({"metrics": m_cases, "trees": t_cases}, fh, separators=(",", ":"))
    print(len(m_cases), "metric cases,", len(t_cases), "tree cases")


if __name__ == "__main__":
    main()
