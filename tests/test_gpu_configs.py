"""GPU parity on the BASELINE.json configurations beyond config 1/2
(SURVEY.md 8d): config 3 (multi-process, multi-phase, nested ops on two tids,
all six categories) and config 5 (adversarial: Zipf-skewed pids, recursive
ops to depth 64, 256 GPU streams of long concurrent kernels, 1% zero-duration
events, 10% duplicate correlation ids, coarse timestamp grid).

Every comparison is bit-exact against the C oracle (oracle/xs_oracle.c, itself
pinned to the reference's outputs in tests/test_oracle_golden.py): cells,
spans and untracked of compute_overlap; corrected start/duration columns and
the CorrectionReport of correct_trace; transition site lists.
"""

import numpy as np
import pytest

import oracle
from paper_2102_04285_b200 import Attribution, analyze_columnar, compute_overlap_columnar, synth
from paper_2102_04285_b200 import CalibrationProfile, correct_trace_columnar
from paper_2102_04285_b200.overlap import transition_site_indices

pytestmark = pytest.mark.gpu


def _ours(bd):
    cells = {(k.pid, k.path, frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items()}
    return cells, bd.spans, bd.untracked


def _check_correction(ct, prof):
    out, rep = correct_trace_columnar(ct, prof)
    s, d, orep, _ = oracle.correct(ct, prof)
    assert np.array_equal(out.start, s) and np.array_equal(out.dur, d)
    assert rep.removed_ns == orep["removed_ns"] and rep.shortfall_ns == orep["shortfall_ns"]
    assert rep.original_total_ns == orep["original_total_ns"]
    assert rep.corrected_total_ns == orep["corrected_total_ns"]
    return out


@pytest.fixture(scope="module")
def cfg3():
    return synth.config3_trace(processes=6, events_per_pid=150_000, both=True, workers=6)


@pytest.fixture(scope="module")
def cfg5():
    return synth.adversarial_trace(400_000, pids=16, workers=8)


def test_config3_overlap_vs_oracle(cfg3):
    for ct in cfg3:
        assert _ours(compute_overlap_columnar(ct)) == oracle.overlap(ct, 0)


def test_config3_correlation_vs_oracle(cfg3):
    ct = cfg3[1]
    assert _ours(compute_overlap_columnar(ct, Attribution.CORRELATION)) == oracle.overlap(ct, 1)


def test_config3_correction_closure_and_oracle(cfg3):
    un, inst = cfg3
    out = _check_correction(inst, synth.exact_profile())
    assert np.array_equal(out.start, un.start) and np.array_equal(out.dur, un.dur)


def test_config3_analyze_one_call(cfg3):
    un, inst = cfg3
    s, d, rep, bd = analyze_columnar(inst, synth.exact_profile())
    assert np.array_equal(s.cpu().numpy(), un.start) and np.array_equal(d.cpu().numpy(), un.dur)
    assert _ours(bd) == oracle.overlap(un, 0)


def test_config5_overlap_vs_oracle(cfg5):
    assert _ours(compute_overlap_columnar(cfg5)) == oracle.overlap(cfg5, 0)


def test_config5_correlation_vs_oracle():
    # the reference's CORRELATION cost is O(events x concurrent fixed paths):
    # keep the oracle side to seconds
    ct = synth.adversarial_trace(60_000, pids=6, streams=64)
    assert _ours(compute_overlap_columnar(ct, Attribution.CORRELATION)) == oracle.overlap(ct, 1)


def test_config5_correction_vs_oracle(cfg5):
    for prof in (synth.adversarial_profile(),
                 CalibrationProfile(1000, 500, 250, {"launch": 3000, "memcpy": 1000, "sync": 20})):
        _check_correction(cfg5, prof)


def test_config5_transition_sites_vs_oracle(cfg5):
    got = transition_site_indices(cfg5, 0xF)
    exp = oracle.transition_sites(cfg5, 0xF)
    assert {(int(a), int(b)): list(v) for (a, b), v in got.items()} == exp


def test_config5_analyze_vs_oracle(cfg5):
    prof = synth.adversarial_profile()
    s, d, rep, bd = analyze_columnar(cfg5, prof)
    os_, od, _, _ = oracle.correct(cfg5, prof)
    assert np.array_equal(s.cpu().numpy(), os_) and np.array_equal(d.cpu().numpy(), od)
    from paper_2102_04285_b200 import ColumnarTrace
    c = cfg5
    corrected = ColumnarTrace(c.clock_domain, os_, od, c.pid, c.tid, c.cat, c.name, c.corr, c.has_corr, c.pids,
                              c.group_pid, c.group_tid, c.names, c.processes, c.pid_has_meta)
    assert _ours(bd) == oracle.overlap(corrected, 0)


@pytest.mark.slow
def test_config5_full_10m_overlap_vs_oracle():
    ct = synth.adversarial_trace(10_000_000, pids=64, workers=16)
    assert _ours(compute_overlap_columnar(ct)) == oracle.overlap(ct, 0)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_config5_window_split_shards_on_device(world):
    """The multi-GPU plan (giant pids cut into operation-free windows, LPT
    packing) run shard by shard on this GPU: the merged Breakdown equals the
    single-call one bit for bit."""
    from paper_2102_04285_b200 import _engine
    from paper_2102_04285_b200.distributed import merge_raw_list, plan_shards, shard_trace

    ct = synth.adversarial_trace(400_000, pids=16, workers=8)
    whole = compute_overlap_columnar(ct)
    eng = _engine.get(0)
    parts = []
    for sh in plan_shards(ct, world, 2):
        local = shard_trace(ct, sh)
        parts.append((local, eng.overlap(_engine.DeviceTrace(local, 0), 0)))
    bd = merge_raw_list(parts)
    assert bd.cells == whole.cells and bd.spans == whole.spans and bd.untracked == whole.untracked


def test_analyze_sharded_single_rank_equals_analyze():
    """analyze_sharded (no process group: world 1) returns analyze_columnar's
    report, Breakdown and corrected columns."""
    from paper_2102_04285_b200.distributed import analyze_sharded

    ct = synth.adversarial_trace(120_000, pids=9, workers=4)
    prof = synth.adversarial_profile()
    s0, d0, rep0, bd0 = analyze_columnar(ct, prof)
    rows, s1, d1, rep1, bd1 = analyze_sharded(ct, prof, gather_columns=True)
    assert np.array_equal(s1, s0.cpu().numpy()) and np.array_equal(d1, d0.cpu().numpy())
    assert rep1 == rep0 and bd1 == bd0
