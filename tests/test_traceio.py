"""Trace I/O: the native XSTRACE1 decoder and the
vectorised writer against directories and verdicts produced by the REFERENCE
(tests/golden/traceio, scripts/make_golden_traceio.py): decoded events in
read_trace order, exact error classes and messages on corrupted input, and
byte-identical writer output.  Host code only: runs without a GPU."""

import json
import os

import numpy as np
import pytest

from paper_2102_04285_b200 import synth, traceio
from paper_2102_04285_b200.model import Category, Event, ProcessMeta, Trace

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "traceio")
GEN_ROOT = "/root/repo/tests/golden/traceio"  # where the fixtures were generated (messages embed it)
CASES = json.load(open(os.path.join(GOLD, "cases.json")))


def _events(t):
    return [[e.pid, e.tid, int(e.category), e.name, e.start, e.duration, e.correlation] for e in t.events]


@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_matches_reference(name):
    exp = CASES[name]["expect"]
    path = os.path.join(GOLD, name)
    if "error" in exp:
        with pytest.raises(getattr(traceio, exp["error"])) as ei:
            traceio.read_trace_columnar(path)
        assert str(ei.value) == exp["message"].replace(GEN_ROOT, GOLD)
        return
    t = traceio.read_trace(path)
    assert t.clock_domain == exp["clock_domain"]
    assert _events(t) == exp["events"]
    assert [[m.pid, m.name, m.parent, m.fork_ns, m.join_ns] for m in t.processes] == exp["processes"]


@pytest.mark.parametrize("name", sorted(k for k, v in CASES.items() if v["write"]))
def test_writer_bytes_match_reference(name, tmp_path):
    src = os.path.join(GOLD, name)
    t = traceio.read_trace(src)
    n = traceio._write_unchecked(t, tmp_path, CASES[name]["limit"])
    files = sorted(f for f in os.listdir(src))
    assert sorted(os.listdir(tmp_path)) == files and n == len(files) - 1
    for f in files:
        assert open(os.path.join(src, f), "rb").read() == open(os.path.join(tmp_path, f), "rb").read(), f


def test_columnar_roundtrip_large(tmp_path):
    ct = synth.ddpg_trace(6000, processes=2, outer_op="iteration", second_tid_ops=True)
    n = traceio._write_unchecked(ct, tmp_path, 1 << 20)
    assert n > 1
    back = traceio.read_trace_columnar(tmp_path, workers=4)
    order = np.lexsort((np.where(ct.has_corr == 1, ct.corr, -1), ct.name, ct.group_tid[ct.tid], ct.pids[ct.pid],
                        ct.cat, ct.start + ct.dur, ct.start))
    for f in ("start", "dur", "cat", "corr", "has_corr"):
        assert np.array_equal(getattr(back, f), getattr(ct, f)[order]), f
    assert np.array_equal(back.pids[back.pid], ct.pids[ct.pid][order])
    assert np.array_equal(back.group_tid[back.tid], ct.group_tid[ct.tid][order])
    assert [back.names[i] for i in back.name[:100]] == [ct.names[i] for i in ct.name[order][:100]]


def test_unsorted_writer_input_is_sorted_on_read(tmp_path):
    # a foreign writer may emit any order: read_trace sorts by Event.sort_key
    t = Trace(5, [Event(1, 0, Category.BACKEND, "b", 50, 5), Event(1, 0, Category.BACKEND, "a", 10, 5, 3),
                  Event(1, 0, Category.BACKEND, "a", 10, 5)], [ProcessMeta(1, "p")])
    traceio._write_unchecked(t, tmp_path)
    ct = traceio.read_trace_columnar(tmp_path)
    assert ct.start.tolist() == [10, 10, 50] and ct.has_corr.tolist() == [0, 1, 0]


def test_chunk_limit_floor():
    with pytest.raises(ValueError):
        traceio.write_trace(Trace(1, [], []), "/tmp/unused_xs", chunk_limit_bytes=100)
