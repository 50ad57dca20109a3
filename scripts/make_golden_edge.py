#!/usr/bin/env python3
"""tests/golden/edge_cases.json.gz: reference outputs on REFERENCE-VALID
inputs at the edges of the device formulation:

* merged multi-tid operation stacks deeper than 256 (two tids nesting 150 and
  151 deep; 70 tids with a 4-deep stack each -- more than 64 active op tids);
* timelines too wide for one 64-bit key over all pids (300 pids, each spanning
  ~2^55 ns: pid bits + span bits + code bits > 64) and a single process
  spanning >= 2^61 ns;
* calibration profiles whose common denominator overflows int64 / int128
  (denominators ~2^70 and a product of coprime ~2^45 denominators).

Each case stores compute_overlap (INSTANT and CORRELATION) and, with its
profile, correct_trace + compute_overlap(corrected), in the formats of
scripts/make_golden.py.  Run after oracle/build_ref.sh:

    python scripts/make_golden_edge.py
"""
import gzip
import json
import os
import random
import sys
from fractions import Fraction

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, HERE)

from make_golden import enc_breakdown, enc_profile, enc_trace  # noqa: E402
from xstrace import overlap as X_ov  # noqa: E402
from xstrace.calibration import CalibrationProfile  # noqa: E402
from xstrace.correction import correct_trace  # noqa: E402
from xstrace.model import Category, Event, ProcessMeta, Trace  # noqa: E402

O, H, B, S, A, G = (Category.OPERATION, Category.HIGH_LEVEL, Category.BACKEND,
                    Category.SIMULATOR, Category.ACCEL_API, Category.GPU)
APIS = ("launch", "memcpy")


def resources(rng, pid, t0, t1, k, corr0, tid=0, gtid=1000):
    """k BACKEND calls with ACCEL_API launches and correlated GPU kernels in [t0, t1)."""
    ev, corr = [], corr0
    step = max(1, (t1 - t0) // (k + 1))
    for i in range(k):
        s = t0 + i * step
        ev.append(Event(pid, tid, B, "call", s, max(1, step // 2)))
        corr += 1
        a = s + 1
        ev.append(Event(pid, tid, A, rng.choice(APIS), a, max(1, step // 8), corr))
        ev.append(Event(pid, gtid, G, "kernel", a + 2, max(1, step // 3), corr))
    return ev, corr


def deep_two_tids():
    rng = random.Random(1)
    ev = [Event(1, 0, H, "script", 0, 100_000)]
    for i in range(150):
        ev.append(Event(1, 0, O, f"a{i:03d}", 10 * i, 100_000 - 20 * i))
    for i in range(151):
        ev.append(Event(1, 1, O, f"b{i:03d}", 10 * i + 5, 100_000 - 20 * i - 10))
    r, _ = resources(rng, 1, 3_000, 97_000, 40, 0)
    return Trace(1, ev + r, [ProcessMeta(1, "deep")])


def many_tids():
    rng = random.Random(2)
    ev = [Event(1, 0, H, "script", 0, 50_000)]
    for t in range(70):
        for d in range(4):
            ev.append(Event(1, t, O, f"t{t % 7}d{d}", 100 + 3 * t + d, 40_000 - 5 * t - 2 * d))
    r, _ = resources(rng, 1, 2_000, 38_000, 30, 0, tid=0)
    return Trace(1, ev + r, [ProcessMeta(1, "many_tids")])


def many_wide_pids():
    rng = random.Random(3)
    ev, procs = [], []
    span = 1 << 55
    for p in range(1, 301):
        base = rng.randrange(0, 1 << 40)
        ev.append(Event(p, 0, H, "script", base, span))
        ev.append(Event(p, 0, O, "step", base + 10, 1000))
        r, _ = resources(rng, p, base + 20, base + 900, 3, 0)
        ev += r
        ev.append(Event(p, 0, B, "late", base + span - (1 << 50), 1 << 40))
        procs.append(ProcessMeta(p, f"w{p}"))
    return Trace(1, ev, procs)


def wide_single_pid():
    rng = random.Random(4)
    top = (1 << 62) + (1 << 60)
    ev = [Event(1, 0, H, "script", 0, top)]
    ev.append(Event(1, 0, O, "early", 100, 10_000))
    r, c = resources(rng, 1, 200, 9_000, 5, 0)
    ev += r
    ev.append(Event(1, 0, O, "late", top - 50_000, 20_000))
    r, _ = resources(rng, 1, top - 49_000, top - 31_000, 5, c)
    ev += r
    ev.append(Event(1, 0, S, "sim", 1 << 61, 1 << 40))
    return Trace(1, ev, [ProcessMeta(1, "wide")])


def workload_trace():
    ev = []
    rng = random.Random(5)
    t = 0
    corr = 0
    for it in range(60):
        ev.append(Event(1, 0, O, "step", t, 5_000))
        r, corr = resources(rng, 1, t + 100, t + 4_900, 4, corr)
        ev += r
        t += 5_000
    ev.append(Event(1, 0, H, "script", 0, t + 10))
    return Trace(1, ev, [ProcessMeta(1, "w")])


def big_den_profile():
    d = (1 << 70) + 3
    return CalibrationProfile(Fraction(4000 * d + 7, d), Fraction(1000 * d - 5, d), Fraction(1500 * d + 1, d),
                              {"launch": Fraction(3000 * d + d // 3, d), "memcpy": Fraction(1000 * d + 11, d)})


def coprime_profile():
    ps = [(1 << 45) + k for k in (7, 9, 13, 19, 21)]  # pairwise coprime enough: L ~ 2^225
    return CalibrationProfile(Fraction(4000 * ps[0] + 1, ps[0]), Fraction(1000 * ps[1] + 3, ps[1]),
                              Fraction(1500 * ps[2] - 2, ps[2]),
                              {"launch": Fraction(3000 * ps[3] + 5, ps[3]), "memcpy": Fraction(999 * ps[4] + 4, ps[4])})


PLAIN = CalibrationProfile(Fraction(4001, 3), Fraction(999, 7), Fraction(1501, 2),
                           {"launch": Fraction(3001, 11), "memcpy": Fraction(997, 13)})

cases = []


def add(name, trace, profiles):
    case = {"name": name, "trace": enc_trace(trace), "overlap": {}}
    for attr in ("instant", "correlation"):
        a = X_ov.Attribution.INSTANT if attr == "instant" else X_ov.Attribution.CORRELATION
        case["overlap"][attr] = enc_breakdown(X_ov.compute_overlap(trace, a))
    case["corrections"] = []
    for prof in profiles:
        out, rep = correct_trace(trace, prof)
        case["corrections"].append({
            "profile": enc_profile(prof),
            "start": [e.start for e in out.events],
            "dur": [e.duration for e in out.events],
            "removed_ns": {str(k): v for k, v in rep.removed_ns.items()},
            "shortfall_ns": {str(k): v for k, v in rep.shortfall_ns.items()},
            "original_total_ns": rep.original_total_ns,
            "corrected_total_ns": rep.corrected_total_ns,
            "overlap_corrected": enc_breakdown(X_ov.compute_overlap(out)),
        })
    cases.append(case)
    print(name, len(trace.events), "events")


add("deep_merged_two_tids", deep_two_tids(), [PLAIN])
add("more_than_64_op_tids", many_tids(), [PLAIN])
add("many_pids_wide_spans", many_wide_pids(), [PLAIN])
add("single_pid_span_2e62", wide_single_pid(), [PLAIN])
add("denominator_2e70", workload_trace(), [big_den_profile()])
add("denominator_product_2e225", workload_trace(), [coprime_profile()])
with gzip.open(os.path.join(ROOT, "tests", "golden", "edge_cases.json.gz"), "wt") as fh:
    json.dump(cases, fh, separators=(",", ":"))
