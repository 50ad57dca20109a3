#!/usr/bin/env python3
"""tests/golden/sweep_pid_cases.json.gz: the inputs the REFERENCE's
compute_overlap hands its kernel plugin (overlap.py:171-174) and the pure-
Python kernel's outputs (_sweep_py.sweep_pid), recorded on seeded random
traces (INSTANT).  Cells are stored with paths decoded to name-id tuples so
any path-id assignment compares.  Run after oracle/build_ref.sh."""
import gzip
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

from xstrace import _sweep_py  # noqa: E402
from xstrace.overlap import Attribution, compute_overlap  # noqa: E402
from xstrace.synth import generate_workload, preset_exact, random_trace  # noqa: E402

cases = []


class Recorder:
    @staticmethod
    def sweep_pid(starts, ends, cats, ranks, fixed_paths, add_order, rem_order, rank_name_ids, path_table):
        cells, tracked = _sweep_py.sweep_pid(starts, ends, cats, ranks, fixed_paths, add_order, rem_order,
                                             rank_name_ids, path_table)
        dec = sorted([list(path_table.paths[k >> 6]), k & 63, v] for k, v in cells.items())
        case = {"args": [list(starts), list(ends), list(cats), list(ranks), list(fixed_paths),
                         list(add_order), list(rem_order), list(rank_name_ids)],
                "cells": dec, "tracked": tracked}
        if any(fp >= 0 for fp in fixed_paths):  # CORRELATION: the table the fixed path ids refer to
            case["paths"] = [list(p) for p in path_table.paths]
        cases.append(case)
        return cells, tracked


for seed in range(40):
    compute_overlap(random_trace(random.Random(seed), max_events=200, max_span=50_000, pids=2), kernel=Recorder)
compute_overlap(generate_workload(preset_exact(seed=5, iterations=10))[1], kernel=Recorder)
# CORRELATION: GPU events pinned to their launch-site paths (fixed_paths >= 0)
for seed in range(40, 60):
    compute_overlap(random_trace(random.Random(seed), max_events=200, max_span=50_000, pids=2),
                    Attribution.CORRELATION, kernel=Recorder)
compute_overlap(generate_workload(preset_exact(seed=6, iterations=10))[1], Attribution.CORRELATION, kernel=Recorder)
with gzip.open(os.path.join(ROOT, "tests", "golden", "sweep_pid_cases.json.gz"), "wt") as fh:
    json.dump(cases, fh, separators=(",", ":"))
print(len(cases), "sweep_pid calls recorded")
