#!/usr/bin/env python3
"""Generate tests/golden/traceio/: trace directories written by the REFERENCE
writer (traceio.write_trace) plus the reference reader's verdicts, including
corrupted variants and their exact error messages.  Run after
oracle/build_ref.sh:

    python scripts/make_golden_traceio.py
"""

from __future__ import annotations

import json
import os
import random
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

from xstrace import traceio as RT  # noqa: E402
from xstrace.model import Category, Event, ProcessMeta, Trace  # noqa: E402
from xstrace.synth import generate_workload, preset_exact, random_trace  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "traceio")


def events_of(trace):
    return [[e.pid, e.tid, int(e.category), e.name, e.start, e.duration, e.correlation] for e in trace.events]


def verdict(path):
    try:
        t = RT.read_trace(path)
    except ValueError as exc:
        return {"error": type(exc).__name__, "message": str(exc)}
    return {"clock_domain": t.clock_domain, "events": events_of(t),
            "processes": [[m.pid, m.name, m.parent, m.fork_ns, m.join_ns] for m in t.processes]}


def corrupt(src, dst, fn):
    shutil.copytree(src, dst)
    fn(dst)


def patch(path, offset, data):
    b = bytearray(open(path, "rb").read())
    b[offset: offset + len(data)] = data
    open(path, "wb").write(bytes(b))


def main():
    if os.path.exists(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    cases = {}
    demo = Trace(42, [Event(1, 0, Category.OPERATION, "step", 0, 120),
                      Event(1, 0, Category.BACKEND, "step_backend", 10, 60),
                      Event(1, 4, Category.GPU, "kernel", 40, 50, 1),
                      Event(1, 0, Category.ACCEL_API, "launch", 30, 20, 1)],
                 [ProcessMeta(1, "demo", None, fork_ns=0, join_ns=200)])
    good = {
        "golden_demo": (demo, 2**20),
        "empty": (Trace(3, [], [ProcessMeta(7, "idle", parent=3)]), 2**20),
        "random_small_chunks": (random_trace(random.Random(5), max_events=1500, pids=3), 4096),
        "random_unicode": (Trace(1, [Event(1, 0, Category.BACKEND, "naïve→ß", 0, 10),
                                     Event(1, 0, Category.HIGH_LEVEL, "ok", 0, 20)], [ProcessMeta(1, "pé")]), 2**20),
        "workload": (generate_workload(preset_exact(seed=3, iterations=20))[1], 16384),
    }
    for name, (trace, limit) in good.items():
        d = os.path.join(OUT, name)
        RT.write_trace(trace, d, chunk_limit_bytes=limit)
        cases[name] = {"limit": limit, "expect": verdict(d), "write": True}
    base = os.path.join(OUT, "golden_demo")
    bad = {
        "bad_magic": lambda d: patch(os.path.join(d, "trace.0.bin"), 0, b"XSTRACE9"),
        "bad_version": lambda d: patch(os.path.join(d, "trace.0.bin"), 8, b"\x02\x00"),
        "bad_meta_magic": lambda d: patch(os.path.join(d, "meta.bin"), 0, b"NOTTRACE"),
        "missing_meta": lambda d: os.remove(os.path.join(d, "meta.bin")),
        "missing_chunk": lambda d: os.remove(os.path.join(d, "trace.0.bin")),
        "wrong_index": lambda d: patch(os.path.join(d, "trace.0.bin"), 18, b"\x05\x00\x00\x00"),
        "clock_mismatch": lambda d: patch(os.path.join(d, "trace.0.bin"), 10, b"\x07"),
        "truncated_record": lambda d: open(os.path.join(d, "trace.0.bin"), "r+b").truncate(200),
        "truncated_header": lambda d: open(os.path.join(d, "trace.0.bin"), "r+b").truncate(20),
        "bad_category": lambda d: patch(os.path.join(d, "trace.0.bin"), 74 + 20, b"\x09"),
        "bad_name_index": lambda d: patch(os.path.join(d, "trace.0.bin"), 74 + 21, b"\x63\x00\x00\x00"),
        "bad_corr_flag": lambda d: patch(os.path.join(d, "trace.0.bin"), 74 + 41, b"\x07"),
        "short_body": lambda d: patch(os.path.join(d, "trace.0.bin"), 74, b"\x10\x00\x00\x00"),
        "bad_utf8": lambda d: patch(os.path.join(d, "trace.0.bin"), 34, b"\xff"),
        "bad_meta_flag": lambda d: patch(os.path.join(d, "meta.bin"), 42, b"\x05"),
    }
    for name, fn in bad.items():
        d = os.path.join(OUT, name)
        corrupt(base, d, fn)
        cases[name] = {"expect": verdict(d), "write": False}
    with open(os.path.join(OUT, "cases.json"), "w") as fh:
        json.dump(cases, fh, indent=0)
    print(len(cases), "cases")
    for k, v in cases.items():
        if "error" in v["expect"]:
            print(k, v["expect"]["message"])


if __name__ == "__main__":
    main()
