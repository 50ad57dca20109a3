"""GPU parity: correct_trace / transition_sites / analyze through the C ABI
vs reference golden vectors, the CPU oracle and the closure property."""

from fractions import Fraction

import numpy as np
import pytest

import oracle
from golden_util import dec_profile, dec_trace, enc_breakdown, load
from paper_2102_04285_b200 import (
    CalibrationProfile,
    ColumnarTrace,
    InvalidTraceError,
    UncalibratedHookError,
    analyze_columnar,
    compute_overlap,
    correct_trace,
    correct_trace_columnar,
    count_transitions,
    synth,
    transition_sites,
)
from paper_2102_04285_b200.overlap import TRANSITION_PAIRS, transition_site_indices

pytestmark = pytest.mark.gpu

CORR = load("correction_cases.json.gz")
TRANS = load("transition_cases.json.gz")


@pytest.mark.parametrize("case", TRANS, ids=[c["name"] for c in TRANS])
def test_transition_sites_match_reference(case):
    trace = dec_trace(case["trace"])
    got = transition_site_indices(trace, 0xF)
    for (s, d), lst in got.items():
        assert lst == case["expect"][f"{int(s)}-{int(d)}"], (s, d)
    counts = count_transitions(trace)
    for s, d in TRANSITION_PAIRS:
        assert counts.get(s, d) == len(case["expect"][f"{int(s)}-{int(d)}"])


def test_transition_sites_return_events():
    trace = dec_trace(TRANS[0]["trace"])
    sites = transition_sites(trace)
    for pair, evs in sites.items():
        for e in evs:
            assert e in trace.events


@pytest.mark.parametrize("case", CORR, ids=[c["name"] for c in CORR])
def test_correction_matches_reference(case, monkeypatch):
    trace = dec_trace(case["trace"])
    prof = dec_profile(case["profile"])
    exp = case["expect"]
    if "invalid" in exp:
        with pytest.raises(InvalidTraceError) as ei:
            correct_trace(trace, prof)
        assert [[v.rule, v.message, list(v.event_indices)] for v in ei.value.violations] == exp["invalid"]
        return
    if "uncalibrated" in exp:
        with pytest.raises(UncalibratedHookError) as ei:
            correct_trace(trace, prof)
        assert str(ei.value) == exp["uncalibrated"]
        return
    out, rep = correct_trace(trace, prof)
    assert [e.start for e in out.events] == exp["start"]
    assert [e.duration for e in out.events] == exp["dur"]
    assert [[m.pid, m.name, m.parent, m.fork_ns, m.join_ns] for m in out.processes] == exp["processes"]
    assert {str(k): v for k, v in rep.removed_ns.items()} == exp["removed_ns"]
    assert {str(k): v for k, v in rep.shortfall_ns.items()} == exp["shortfall_ns"]
    assert rep.original_total_ns == exp["original_total_ns"]
    assert rep.corrected_total_ns == exp["corrected_total_ns"]
    assert enc_breakdown(compute_overlap(out)) == exp["overlap_corrected"]
    # one-call analyze path (correct + overlap(corrected)) gives the same,
    # with the overlap pass launched speculatively reusing the original's
    # operation stage (default), speculatively with its own operation stage,
    # or after a sync
    for mode in ("reuse", "spec", "sync"):
        if mode == "spec":
            monkeypatch.setenv("XS_NO_REUSE_OPS", "1")
        if mode == "sync":
            monkeypatch.setenv("XS_NO_SPECULATE", "1")
        s, d, rep2, bd = analyze_columnar(ColumnarTrace.from_trace(trace), prof)
        assert s.cpu().numpy().tolist() == exp["start"]
        assert d.cpu().numpy().tolist() == exp["dur"]
        assert {str(k): v for k, v in rep2.removed_ns.items()} == exp["removed_ns"]
        assert rep2.original_total_ns == exp["original_total_ns"]
        assert rep2.corrected_total_ns == exp["corrected_total_ns"]
        assert enc_breakdown(bd) == exp["overlap_corrected"]


def _frac_profile():
    return CalibrationProfile(Fraction(4001, 3), Fraction(999, 7), Fraction(1501, 2),
                              {"launch": Fraction(3001, 11), "memcpy": Fraction(997, 13)})


@pytest.mark.parametrize("iters,procs,outer,tid2", [(1500, 1, None, False), (300, 3, "iteration", True)])
def test_correction_synthetic_vs_oracle(iters, procs, outer, tid2):
    un, inst = synth.ddpg_trace(iters, processes=procs, outer_op=outer, second_tid_ops=tid2, both=True)
    for prof in (synth.exact_profile(), _frac_profile()):
        out, rep = correct_trace_columnar(inst, prof)
        s, d, orep, _ = oracle.correct(inst, prof)
        assert np.array_equal(out.start, s) and np.array_equal(out.dur, d)
        assert rep.removed_ns == orep["removed_ns"] and rep.shortfall_ns == orep["shortfall_ns"]
        assert rep.original_total_ns == orep["original_total_ns"]
        assert rep.corrected_total_ns == orep["corrected_total_ns"]


def test_correction_closure_1m():
    """Size-independent property: the exact profile undoes the instrumentation."""
    un, inst = synth.ddpg_trace(27027, both=True)
    out, rep = correct_trace_columnar(inst, synth.exact_profile())
    assert np.array_equal(out.start, un.start)
    assert np.array_equal(out.dur, un.dur)
    assert rep.original_total_ns - sum(sum(v.values()) for v in rep.removed_ns.values()) == rep.corrected_total_ns


def test_repeated_calls_replay_captured_graphs():
    """1st call eager, 2nd captures a CUDA graph, later calls replay it: all
    must give the oracle's answer (and the closure) every time."""
    un, inst = synth.ddpg_trace(800, processes=2, both=True)
    prof = synth.exact_profile()
    ref_cells, _, _ = oracle.overlap(un, 0)
    for _ in range(4):
        s, d, rep, bd = analyze_columnar(inst, prof)
        assert np.array_equal(s.cpu().numpy(), un.start) and np.array_equal(d.cpu().numpy(), un.dur)
        cells = {(k.pid, k.path, frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items()}
        assert cells == ref_cells
    for _ in range(3):
        out, rep2 = correct_trace_columnar(inst, _frac_profile())
        s2, d2, orep, _ = oracle.correct(inst, _frac_profile())
        assert np.array_equal(out.start, s2) and np.array_equal(out.dur, d2)
        assert rep2.removed_ns == orep["removed_ns"]


def test_stage_profiling_survives_graph_replay():
    """Per-stage timing events recorded inside a captured segment are replayed
    with it; reading them must neither fail nor leak an error into later calls."""
    from paper_2102_04285_b200 import _engine
    un, inst = synth.ddpg_trace(300, processes=2, both=True)
    prof = synth.exact_profile()
    ref_cells, _, _ = oracle.overlap(un, 0)
    eng = _engine.get(0)
    eng.lib.xs_profile_enable(eng.ctx, 1)
    try:
        for _ in range(5):
            _, _, _, bd = analyze_columnar(inst, prof)
            cells = {(k.pid, k.path, frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items()}
            assert cells == ref_cells
        ms = np.zeros(32)
        calls = np.zeros(32, np.int64)
        n = eng.lib.xs_profile_read(eng.ctx, ms.ctypes.data, calls.ctypes.data, 32)
        assert n > 0 and calls[:n].sum() > 0 and np.all(ms[:n] >= 0)
    finally:
        eng.lib.xs_profile_enable(eng.ctx, 0)


def _stretched(ct, gap):
    """Append one short OPERATION far after the trace: the time span grows by
    `gap`, so the real records crowd into a few fine buckets of the bucketed
    sorts (dense-bucket radix branch, or chunk overflow -> CUB re-run)."""
    import dataclasses
    i = int(np.flatnonzero(ct.cat == 0)[0])
    t_end = int((ct.start + ct.dur).max())
    add = lambda a, v: np.concatenate([a, np.asarray([v], dtype=a.dtype)])  # noqa: E731
    return dataclasses.replace(
        ct, start=add(ct.start, t_end + gap), dur=add(ct.dur, 10), pid=add(ct.pid, ct.pid[i]),
        tid=add(ct.tid, ct.tid[i]), cat=add(ct.cat, 0), name=add(ct.name, ct.name[i]), corr=add(ct.corr, 0),
        has_corr=add(ct.has_corr, 0), _source=None)


@pytest.mark.parametrize("gap", [2**24, 2**30, 2**36, 2**42])
def test_correction_dense_buckets_vs_oracle(gap):
    _, inst = synth.ddpg_trace(2500, processes=1, second_tid_ops=True, both=True)
    ct = _stretched(inst, gap)
    for prof in (synth.exact_profile(), _frac_profile()):
        out, rep = correct_trace_columnar(ct, prof)
        s, d, orep, _ = oracle.correct(ct, prof)
        assert np.array_equal(out.start, s) and np.array_equal(out.dur, d)
        assert rep.removed_ns == orep["removed_ns"]
    s2, d2, _, bd = analyze_columnar(ct, synth.exact_profile())
    s, d, _, _ = oracle.correct(ct, synth.exact_profile())
    assert np.array_equal(s2.cpu().numpy(), s) and np.array_equal(d2.cpu().numpy(), d)
    cells = {(k.pid, k.path, frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items()}
    ref_cells, _, _ = oracle.overlap(dataclasses_replace_times(ct, s, d), 0)
    assert cells == ref_cells


def dataclasses_replace_times(ct, start, dur):
    import dataclasses
    return dataclasses.replace(ct, start=np.ascontiguousarray(start), dur=np.ascontiguousarray(dur), _source=None)


def test_analyze_to_host_pinned_matches_device_outputs():
    """xs_analyze_to_host: the corrected columns land in pinned host buffers
    (copy overlapped with the overlap pass) and equal xs_analyze's."""
    import torch
    from paper_2102_04285_b200 import analyze_columnar

    un, inst = synth.ddpg_trace(3000, processes=2, outer_op="iteration", both=True)
    s, d, rep, bd = analyze_columnar(inst, synth.exact_profile())
    wide = inst.pinned(packed=False)
    assert wide._pinned["start"].is_pinned() and np.array_equal(wide.start, inst.start)
    packed = inst.pinned()
    assert packed._pinned["_block"].is_pinned() and packed._pinned["_block"].numel() < 20 * inst.n
    for pin in (wide, packed):
        for _ in range(3):  # eager, capture, replay
            hs = torch.empty(inst.n, dtype=torch.int64).pin_memory()
            hd = torch.empty(inst.n, dtype=torch.int64).pin_memory()
            s2, d2, rep2, bd2 = analyze_columnar(pin, synth.exact_profile(), out=(hs, hd))
            assert s2 is hs and np.array_equal(hs.numpy(), s.cpu().numpy()) and np.array_equal(hd.numpy(), un.dur)
            assert bd2.cells == bd.cells and rep2.removed_ns == rep.removed_ns


def test_pipelined_analyze_equals_one_call():
    """analyze_columnar_pipelined (pid batches, next upload overlapping the
    current analysis) returns exactly analyze_columnar's results."""
    import torch
    from paper_2102_04285_b200 import analyze_columnar, analyze_columnar_pipelined

    for ct, prof in ((synth.config3_trace(processes=7, events_per_pid=30_000), synth.exact_profile()),
                     (synth.adversarial_trace(150_000, pids=12), synth.adversarial_profile())):
        s0, d0, rep0, bd0 = analyze_columnar(ct, prof)
        for pin, workers in ((ct.pinned(), 2), (ct.pinned(), 1), (ct.pinned(), 3), (ct.pinned(packed=False), 2),
                             (ct, 2)):
            hs = torch.empty(ct.n, dtype=torch.int64).pin_memory()
            hd = torch.empty(ct.n, dtype=torch.int64).pin_memory()
            s1, d1, rep1, bd1 = analyze_columnar_pipelined(pin, prof, out=(hs, hd), batches=4, workers=workers)
            assert np.array_equal(hs.numpy(), s0.cpu().numpy()) and np.array_equal(hd.numpy(), d0.cpu().numpy())
            assert rep1.removed_ns == rep0.removed_ns and rep1.shortfall_ns == rep0.shortfall_ns
            assert rep1.original_total_ns == rep0.original_total_ns
            assert rep1.corrected_total_ns == rep0.corrected_total_ns
            assert bd1 == bd0


def test_to_host_copies_follow_graph_replays():
    """The corrected-column D2H waits on the event node inside the captured
    graph: the same device buffers refilled with different data between
    calls (same graph key -> replay) read back each call's own result, for
    xs_analyze_to_host and the async variant."""
    import torch

    from paper_2102_04285_b200 import _engine

    eng = _engine.get(0)
    un, inst = synth.ddpg_trace(2000, processes=2, outer_op="iteration", both=True)
    sc = synth.exact_profile().scaled(inst.names)
    shifted = dataclasses_replace_times(inst, inst.start + 12345, inst.dur)
    want = {}
    for k, ct in (("a", inst), ("b", shifted)):
        raw = eng.correct(_engine.DeviceTrace(ct, 0), sc, analyze_attribution=0)
        want[k] = (raw.start.cpu().numpy(), raw.dur.cpu().numpy())
    assert not np.array_equal(want["a"][0], want["b"][0])
    dt = _engine.DeviceTrace(inst, 0)
    src = {"a": torch.from_numpy(inst.start).cuda(), "b": torch.from_numpy(shifted.start).cuda()}
    dev_out = (torch.empty(inst.n, dtype=torch.int64, device="cuda"),
               torch.empty(inst.n, dtype=torch.int64, device="cuda"))
    for i in range(8):
        k = "ab"[i % 2]
        dt.start.copy_(src[k])
        hs = torch.zeros(inst.n, dtype=torch.int64).pin_memory()
        hd = torch.zeros(inst.n, dtype=torch.int64).pin_memory()
        async_copy = i >= 4
        eng.correct(dt, sc, analyze_attribution=0, host_out=(hs, hd), dev_out=dev_out, async_copy=async_copy)
        if async_copy:
            eng.host_copy_wait()
        assert np.array_equal(hs.numpy(), want[k][0]) and np.array_equal(hd.numpy(), want[k][1]), (i, k)


def test_pipelined_errors_surface_after_copies_drain():
    """A batch that fails validation (a negative duration in one pid) or
    lacks a calibrated hook raises the reference's exception from the
    pipelined multi-context path, after every in-flight read-back drained;
    the next call on the same contexts is unaffected."""
    import dataclasses

    import torch

    from paper_2102_04285_b200 import analyze_columnar, analyze_columnar_pipelined

    ct = synth.config3_trace(processes=6, events_per_pid=20_000)
    prof = synth.exact_profile()
    rows = np.flatnonzero(ct.pid == 4)
    bad = dataclasses.replace(ct, dur=np.where(np.arange(ct.n) == rows[100], -7, ct.dur).astype(np.int64),
                              _source=None)
    hs = torch.empty(ct.n, dtype=torch.int64).pin_memory()
    hd = torch.empty(ct.n, dtype=torch.int64).pin_memory()
    with pytest.raises(InvalidTraceError):
        analyze_columnar_pipelined(bad.pinned(), prof, out=(hs, hd), batches=5, workers=3)
    thin = dataclasses.replace(prof, api_internal_ns={})
    with pytest.raises(UncalibratedHookError):
        analyze_columnar_pipelined(ct.pinned(), thin, out=(hs, hd), batches=5, workers=3)
    s0, d0, r0, b0 = analyze_columnar(ct, prof)
    analyze_columnar_pipelined(ct.pinned(), prof, out=(hs, hd), batches=5, workers=3)
    assert np.array_equal(hs.numpy(), s0.cpu().numpy()) and np.array_equal(hd.numpy(), d0.cpu().numpy())


def test_pipelined_mixed_errors_follow_trace_order():
    """Errors of different batches resolve like the reference's whole-trace
    order: an invalid event in a LATE batch wins over an uncalibrated hook in
    an early one (require_valid runs first, correction.py:121), and among
    uncalibrated hooks in several batches the first row in trace order names
    the hook (collect_sites walks events in order, correction.py:86-100)."""
    import dataclasses

    import torch

    from paper_2102_04285_b200 import analyze_columnar, analyze_columnar_pipelined

    ct = synth.config3_trace(processes=6, events_per_pid=20_000)
    prof = synth.exact_profile()
    api = [i for i, nm in enumerate(ct.names) if nm in prof.api_internal_ns]
    other = [i for i, nm in enumerate(ct.names) if nm not in prof.api_internal_ns]
    assert api and other
    is_api = (ct.cat == 4) & np.isin(ct.name, api)

    def rename(name_col, pid, new):
        r = np.flatnonzero(is_api & (ct.pid == pid))[50]
        name_col[r] = new
        return r

    name = ct.name.copy()
    rename(name, 1, other[0])  # uncalibrated in the first batch
    late = np.flatnonzero(ct.pid == 5)[100]
    mixed = dataclasses.replace(ct, name=name, _source=None,
                                dur=np.where(np.arange(ct.n) == late, -7, ct.dur).astype(np.int64))
    hs = torch.empty(ct.n, dtype=torch.int64).pin_memory()
    hd = torch.empty(ct.n, dtype=torch.int64).pin_memory()
    for workers in (1, 3):
        with pytest.raises(InvalidTraceError):
            analyze_columnar_pipelined(mixed.pinned(), prof, out=(hs, hd), batches=5, workers=workers)
    name = ct.name.copy()
    rename(name, 5, other[-1])
    rename(name, 2, other[0])  # earlier in trace order: this one is reported
    two = dataclasses.replace(ct, name=name, _source=None)
    with pytest.raises(UncalibratedHookError) as one_call:
        analyze_columnar(two, prof)
    for workers in (1, 3):
        with pytest.raises(UncalibratedHookError) as piped:
            analyze_columnar_pipelined(two.pinned(), prof, out=(hs, hd), batches=5, workers=workers)
        assert str(piped.value) == str(one_call.value) and repr(ct.names[other[0]]) in str(piped.value)
    s0, d0, r0, b0 = analyze_columnar(ct, prof)
    analyze_columnar_pipelined(ct.pinned(), prof, out=(hs, hd), batches=5, workers=3)
    assert np.array_equal(hs.numpy(), s0.cpu().numpy()) and np.array_equal(hd.numpy(), d0.cpu().numpy())
