"""Loading of the reference-generated golden fixtures (scripts/make_golden.py)."""

import gzip
import json
import os
from fractions import Fraction

from paper_2102_04285_b200.calibration import CalibrationProfile
from paper_2102_04285_b200.model import Category, Event, ProcessMeta, Trace

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with gzip.open(os.path.join(GOLDEN, name), "rt", encoding="utf-8") as fh:
        return json.load(fh)


def dec_trace(d):
    events = [Event(p, t, Category(c), n, s, du, k) for p, t, c, n, s, du, k in d["events"]]
    procs = [ProcessMeta(*m) for m in d["processes"]]
    return Trace(d["clock_domain"], events, procs)


def dec_profile(d):
    f = lambda v: Fraction(v[0], v[1])  # noqa: E731
    return CalibrationProfile(f(d["annotation"]), f(d["transition"]), f(d["api_interception"]),
                              {k: f(v) for k, v in d["api_internal"].items()})


def enc_cells(cells):
    """{(pid, path, cats): ns} with int categories -> sorted golden list form."""
    return sorted([pid, list(path), sorted(int(c) for c in cats), ns] for (pid, path, cats), ns in cells.items())


def enc_breakdown(bd):
    """A Breakdown (ours) -> golden form."""
    return {
        "cells": sorted([k.pid, list(k.path), sorted(int(c) for c in k.categories), ns] for k, ns in bd.cells.items()),
        "spans": sorted([pid, lo, hi] for pid, (lo, hi) in bd.spans.items()),
        "untracked": sorted([pid, v] for pid, v in bd.untracked.items()),
    }
