#!/usr/bin/env python3
"""Generate tests/golden/*.json.gz by running the REFERENCE (xstrace) here.

The reference cannot travel to the GPU box, so its outputs on a fixed set of
inputs are frozen into small fixtures that pin both the CPU oracle and the
CUDA path.  Run from the repo root:

    PYTHONPATH=baseline/_ref/src python scripts/make_golden.py

(``baseline/_ref`` is a build of /root/reference/pkg with the native Cython
sweep; /root/reference/pkg/src works too with the pure-Python kernel -- the
reference's own tests assert both kernels agree.)
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
from fractions import Fraction

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if not any("xstrace" in os.listdir(p) for p in sys.path if os.path.isdir(p)):
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref", "src"))

from xstrace import overlap as X_ov  # noqa: E402
from xstrace.calibration import CalibrationProfile, build_profile  # noqa: E402
from xstrace.correction import UncalibratedHookError, correct_trace  # noqa: E402
from xstrace.model import Category, Event, InvalidTraceError, ProcessMeta, Trace, validate_trace  # noqa: E402
from xstrace.synth import (  # noqa: E402
    brute_force_overlap,
    expand_leaf_trace,
    generate_calibration_ladder,
    generate_workload,
    minigo_like_traces,
    preset_exact,
    preset_inflation,
    preset_noisy,
    random_trace,
)

OUT = os.path.join(ROOT, "tests", "golden")
O, H, B, S, A, G = (Category.OPERATION, Category.HIGH_LEVEL, Category.BACKEND,
                    Category.SIMULATOR, Category.ACCEL_API, Category.GPU)


def enc_trace(trace):
    return {
        "clock_domain": trace.clock_domain,
        "events": [[e.pid, e.tid, int(e.category), e.name, e.start, e.duration, e.correlation]
                   for e in trace.events],
        "processes": [[m.pid, m.name, m.parent, m.fork_ns, m.join_ns] for m in trace.processes],
    }


def enc_breakdown(bd):
    return {
        "cells": sorted([k.pid, list(k.path), sorted(int(c) for c in k.categories), ns]
                        for k, ns in bd.cells.items()),
        "spans": sorted([pid, lo, hi] for pid, (lo, hi) in bd.spans.items()),
        "untracked": sorted([pid, v] for pid, v in bd.untracked.items()),
    }


def frac(v):
    v = Fraction(v)
    return [v.numerator, v.denominator]


def enc_profile(p):
    return {
        "annotation": frac(p.annotation_ns),
        "transition": frac(p.transition_ns),
        "api_interception": frac(p.api_interception_ns),
        "api_internal": {k: frac(v) for k, v in sorted(p.api_internal_ns.items())},
    }


def overlap_expect(trace, attribution):
    try:
        bd = X_ov.compute_overlap(trace, attribution)
    except InvalidTraceError as exc:
        return {"invalid": [[v.rule, v.message, list(v.event_indices)] for v in exc.violations]}
    return enc_breakdown(bd)


def transitions_expect(trace):
    index = {id(e): i for i, e in enumerate(trace.events)}
    sites = X_ov.transition_sites(trace)
    return {f"{int(s)}-{int(d)}": [index[id(e)] for e in sites[(s, d)]] for s, d in X_ov.TRANSITION_PAIRS}


def hand_traces():
    """Small hand-written traces covering each rule of the sweep (SURVEY.md
    section 8c lists the reference cases these mirror)."""
    P = [ProcessMeta(1, "p")]
    cases = {
        "single_event_under_op": [Event(1, 0, O, "a", 0, 10), Event(1, 0, H, "script", 0, 10)],
        "empty_path": [Event(1, 0, B, "call", 5, 10)],
        "set_semantics": [Event(1, 0, B, "x", 0, 10), Event(1, 1, B, "y", 5, 10)],
        "innermost_scoping": [Event(1, 0, O, "outer", 0, 100), Event(1, 0, O, "inner", 40, 20),
                              Event(1, 0, B, "call", 0, 100)],
        "zero_duration": [Event(1, 0, B, "x", 0, 10), Event(1, 0, A, "launch", 5, 0)],
        "adjacent_name_collapse": [Event(1, 0, O, "step", 0, 100), Event(1, 0, O, "step", 10, 50),
                                   Event(1, 0, H, "script", 0, 100)],
        "correlation_launch_site": [Event(1, 0, O, "launch_op", 0, 50), Event(1, 0, O, "other_op", 50, 100),
                                    Event(1, 0, A, "launch", 10, 10, 1), Event(1, 9, G, "kernel", 60, 30, 1)],
        "correlation_same_path": [Event(1, 0, O, "op", 0, 100), Event(1, 0, A, "launch", 0, 10, 1),
                                  Event(1, 9, G, "kernel", 5, 20, 1)],
        "duplicate_correlation": [Event(1, 0, O, "first_op", 0, 50), Event(1, 0, O, "second_op", 50, 50),
                                  Event(1, 0, A, "launch", 10, 5, 7), Event(1, 0, A, "launch", 60, 5, 7),
                                  Event(1, 9, G, "kernel", 80, 15, 7)],
        "cross_tid_path": [Event(1, 0, O, "A", 0, 100), Event(1, 1, O, "B", 10, 40), Event(1, 0, O, "C", 20, 10),
                           Event(1, 0, H, "script", 0, 100)],
        "span_includes_zero_duration": [Event(1, 0, O, "op", 0, 100), Event(1, 0, B, "b", 10, 20),
                                        Event(1, 1000, G, "k", 150, 0)],
        "transition_examples": [Event(1, 0, H, "script", 0, 100), Event(1, 0, B, "call", 10, 30),
                                Event(1, 0, A, "launch", 12, 5), Event(1, 0, A, "launch", 20, 5),
                                Event(1, 0, A, "memcpy", 27, 5)],
        "nested_same_category": [Event(1, 0, H, "script", 0, 100), Event(1, 0, B, "outer", 10, 50),
                                 Event(1, 0, B, "reentrant", 20, 10)],
        "transition_containing_start": [Event(1, 0, H, "script", 0, 10), Event(1, 0, B, "late", 10, 5),
                                        Event(1, 0, B, "inside", 9, 5)],
        "transition_tid_boundary": [Event(1, 0, H, "script", 0, 100), Event(1, 1, B, "other_thread", 10, 5)],
        "equal_ops_and_ties": [Event(1, 0, O, "x", 0, 50), Event(1, 0, O, "x", 0, 50), Event(1, 1, O, "a", 0, 50),
                               Event(1, 0, S, "x", 5, 10), Event(1, 0, B, "x", 5, 20), Event(1, 0, H, "h", 0, 60),
                               Event(1, 0, B, "x", 5, 20)],
        "touching_ops": [Event(1, 0, O, "a", 0, 10), Event(1, 0, O, "b", 10, 10), Event(1, 0, O, "c", 20, 0),
                         Event(1, 0, H, "s", 0, 30)],
        "clipped_rank_pitfall": [Event(1, 0, O, "zeta", 0, 100), Event(1, 1, O, "alpha", 50, 50),
                                 Event(1, 0, B, "b", 0, 100)],
        "invalid_partial_overlap": [Event(1, 0, O, "a", 0, 10), Event(1, 0, O, "b", 5, 10)],
        "invalid_negative": [Event(1, 0, B, "neg", -5, 10), Event(1, 0, B, "negd", 5, -1)],
        "invalid_dangling": [Event(1, 9, G, "kernel", 0, 10, 42), Event(1, 0, A, "launch", 0, 5, 41)],
    }
    out = [(k, Trace(1, v, P)) for k, v in cases.items()]
    out.append(("unknown_pid", Trace(1, [Event(2, 0, B, "x", 0, 5)], P)))
    out.append(("expand_leaf", expand_leaf_trace()))
    out.append(("empty", Trace(1, [], [])))
    out.append(("multi_pid_mixed", Trace(3, [Event(5, 0, B, "b", 0, 10), Event(2, 0, B, "b", 3, 10),
                                               Event(5, 0, O, "op", 2, 4)],
                                         [ProcessMeta(2, "x"), ProcessMeta(5, "y", parent=2, fork_ns=0, join_ns=10),
                                          ProcessMeta(7, "nometa-events")])))
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    overlap_cases = []
    transition_cases = []

    def add_overlap(name, trace, attributions=("instant", "correlation"), brute=False):
        exp = {}
        for a in attributions:
            attr = X_ov.Attribution(a)
            exp[a] = overlap_expect(trace, attr)
            if brute and "invalid" not in exp[a]:
                bf = brute_force_overlap(trace, 1, attr)
                assert enc_breakdown(bf) == exp[a], name
        overlap_cases.append({"name": name, "trace": enc_trace(trace), "expect": exp})
        if not validate_trace(trace):
            transition_cases.append({"name": name, "trace": enc_trace(trace), "expect": transitions_expect(trace)})

    for name, tr in hand_traces():
        add_overlap(name, tr)
    for seed in range(80):
        add_overlap(f"rand2pid_{seed}", random_trace(random.Random(seed), max_events=200, max_span=50_000, pids=2),
                    brute=seed < 20)
    for seed in range(40):
        add_overlap(f"randcorr_{seed}", random_trace(random.Random(1000 + seed), max_events=150, max_span=30_000),
                    brute=seed < 10)
    for seed in range(25):
        add_overlap(f"rand1000_{seed}", random_trace(random.Random(2000 + seed), max_events=1000,
                                                     max_span=1_000_000, max_depth=3, max_categories=4))
    for seed in range(25):
        add_overlap(f"randdeep_{seed}", random_trace(random.Random(3000 + seed), max_events=600,
                                                     max_span=200_000, max_depth=7, max_categories=5, pids=3))
    for seed in range(6):
        un, inst, _ = generate_workload(preset_exact(seed=seed, iterations=4, processes=1 + seed % 3))
        add_overlap(f"workload_un_{seed}", un)
        add_overlap(f"workload_inst_{seed}", inst)
    mg = minigo_like_traces(workers=3)
    add_overlap("minigo_merged", Trace(4, [e for t in mg for e in t.events], [m for t in mg for m in t.processes]),
                attributions=("instant",))

    # correction --------------------------------------------------------
    exact = CalibrationProfile(Fraction(4000), Fraction(1000), Fraction(1500),
                               {"launch": Fraction(3000), "memcpy": Fraction(1000)})
    corr_cases = []

    def add_corr(name, trace, profile, closure=None):
        case = {"name": name, "trace": enc_trace(trace), "profile": enc_profile(profile)}
        try:
            out, rep = correct_trace(trace, profile)
        except UncalibratedHookError as exc:
            case["expect"] = {"uncalibrated": str(exc)}
        except InvalidTraceError as exc:
            case["expect"] = {"invalid": [[v.rule, v.message, list(v.event_indices)] for v in exc.violations]}
        else:
            case["expect"] = {
                "start": [e.start for e in out.events],
                "dur": [e.duration for e in out.events],
                "processes": [[m.pid, m.name, m.parent, m.fork_ns, m.join_ns] for m in out.processes],
                "removed_ns": {str(k): v for k, v in rep.removed_ns.items()},
                "shortfall_ns": {str(k): v for k, v in rep.shortfall_ns.items()},
                "original_total_ns": rep.original_total_ns,
                "corrected_total_ns": rep.corrected_total_ns,
                "overlap_corrected": enc_breakdown(X_ov.compute_overlap(out)),
            }
            if closure is not None:
                case["expect"]["closure"] = [e.start for e in closure.events] == [e.start for e in out.events]
        corr_cases.append(case)

    for seed, procs in [(0, 1), (1, 1), (3, 2), (4, 3), (6, 2)]:
        spec = preset_exact(seed=seed, iterations=5, processes=procs)
        un, inst, _ = generate_workload(spec)
        add_corr(f"exact_{seed}", inst, exact, closure=un)
        add_corr(f"exact_ladder_{seed}", inst, build_profile(generate_calibration_ladder(spec).values()), closure=un)
    for seed in range(6):
        spec = preset_noisy(seed=seed, iterations=4, processes=1 + seed % 2)
        _, inst, _ = generate_workload(spec)
        add_corr(f"noisy_ladder_{seed}", inst, build_profile(generate_calibration_ladder(spec).values()))
    spec = preset_inflation(seed=0, iterations=8)
    _, inst, _ = generate_workload(spec)
    add_corr("inflation_ladder", inst, build_profile(generate_calibration_ladder(spec).values()))
    add_corr("zero_profile", generate_workload(preset_exact(seed=1, iterations=3))[1],
             CalibrationProfile.zero(("launch", "memcpy")))
    add_corr("uncalibrated", generate_workload(preset_exact(seed=2, iterations=2))[1],
             CalibrationProfile(Fraction(0), Fraction(0), Fraction(0), {"launch": Fraction(0)}))
    add_corr("shortfall", Trace(1, [Event(1, 0, O, "op", 0, 10), Event(1, 0, B, "tail", 20, 30)],
                                [ProcessMeta(1, "p")]),
             CalibrationProfile(Fraction(100), Fraction(0), Fraction(0), {}))
    rng = random.Random(99)
    for seed in range(40):
        tr = random_trace(random.Random(4000 + seed), max_events=300, max_span=100_000, pids=1 + seed % 3,
                          max_depth=4, max_categories=5)
        api_names = sorted({e.name for e in tr.events if e.category == A})
        prof = CalibrationProfile(Fraction(rng.randint(0, 3000), rng.randint(1, 7)),
                                  Fraction(rng.randint(0, 900), rng.randint(1, 5)),
                                  Fraction(rng.randint(0, 700), rng.randint(1, 3)),
                                  {n: Fraction(rng.randint(0, 5000), rng.randint(1, 11)) for n in api_names})
        add_corr(f"random_{seed}", tr, prof)
    add_corr("equal_ops_ties", dict(hand_traces())["equal_ops_and_ties"],
             CalibrationProfile(Fraction(7, 3), Fraction(5, 2), Fraction(1, 3), {}))
    add_corr("invalid", dict(hand_traces())["invalid_partial_overlap"], exact)

    for fname, data in (("overlap_cases.json.gz", overlap_cases), ("transition_cases.json.gz", transition_cases),
                        ("correction_cases.json.gz", corr_cases)):
        with gzip.open(os.path.join(OUT, fname), "wt", encoding="utf-8") as fh:
            json.dump(data, fh, separators=(",", ":"))
        print(fname, len(data))


if __name__ == "__main__":
    main()
