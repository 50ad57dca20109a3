"""GPU parity of the window-split correction (distributed.analyze_sharded with
``split``): giant processes cut into time windows corrected by one device
call each with the window carries (xs_profile_t.residue_in / span_end_in),
overlapped with the clipped GPU pieces, merged -- vs the C oracle on the
whole trace, bit for bit (correction.py:115-186, overlap.py:106-188).  One
GPU: every window runs on this rank, the carry protocol is the same."""

import numpy as np
import pytest
import torch

from paper_2102_04285_b200 import synth
from paper_2102_04285_b200.distributed import (
    DeviceWindowRunner,
    _analyze_windows,
    analyze_sharded,
    plan_correction_shards,
)
from test_window_correction import _check, _profiles, _trace, _whole

pytestmark = pytest.mark.gpu


def _runner():
    from paper_2102_04285_b200 import _engine

    return DeviceWindowRunner(_engine.get(0))


@pytest.mark.parametrize("kind", ["ddpg", "ddpg1", "c3"])
@pytest.mark.parametrize("prof", ["exact", "ladder", "frac"])
def test_device_windows_instant(kind, prof):
    ct = _trace(kind)
    profile = _profiles()[prof]
    plan = plan_correction_shards(ct, 1, 4)
    assert any(a is not None for sh in plan for _, a, _ in sh)
    out = _analyze_windows(ct, profile, 0, torch.device("cuda", 0), 1, 0, 4, _runner())
    assert out is not None
    _check(ct, out, _whole(ct, profile, 0))


@pytest.mark.parametrize("kind", ["ddpg", "ddpg1"])
@pytest.mark.parametrize("attr", [0, 1])
def test_analyze_sharded_split_public(kind, attr):
    """The public entry point (window path, or the whole-pid fallback for a
    correlated kernel crossing a mapped cut) equals the whole-trace oracle."""
    ct = _trace(kind)
    profile = _profiles()["ladder"]
    out = analyze_sharded(ct, profile, attribution=("instant", "correlation")[attr], split=8)
    _check(ct, out, _whole(ct, profile, attr))


def test_many_windows_multiword_profile():
    """16 windows of one process with a profile whose common denominator
    needs 2 words (the residue carry in multiword form)."""
    from fractions import Fraction

    from paper_2102_04285_b200.calibration import CalibrationProfile

    ct = _trace("ddpg1")
    den = (1 << 70) + 3
    profile = CalibrationProfile(Fraction(4000 * den + 17, den), Fraction(999 * den + 5, den),
                                 Fraction(1500 * den + 1, den),
                                 {"launch": Fraction(3000 * den + 7, den), "memcpy": Fraction(1000)})
    assert profile.scaled(ct.names).words == 2
    out = _analyze_windows(ct, profile, 0, torch.device("cuda", 0), 1, 0, 16, _runner())
    assert out is not None
    # the whole-process device path (pinned to the reference's 2^70-denominator
    # goldens in test_gpu_edge.py) is the comparison: the oracle is int64-scaled
    rows, s, d, rep, bd = out
    wr, ws, wd, wrep, wbd = analyze_sharded(ct, profile, split=0, gather_columns=True)
    assert np.array_equal(s, ws[rows]) and np.array_equal(d, wd[rows])
    assert rep.removed_ns == wrep.removed_ns and rep.shortfall_ns == wrep.shortfall_ns
    assert rep.original_total_ns == wrep.original_total_ns and rep.corrected_total_ns == wrep.corrected_total_ns
    assert bd.cells == wbd.cells and bd.spans == wbd.spans and bd.untracked == wbd.untracked


def test_config5_dominant_process_windows():
    """Config-5 shape (Zipf process sizes, depth-64 operations, 256 streams):
    the dominant process is split; results equal the whole-trace oracle."""
    ct = synth.adversarial_trace(400_000, pids=8, streams=32)
    profile = synth.adversarial_profile()
    counts = np.bincount(ct.pid)
    assert counts.max() > ct.n // 4
    out = _analyze_windows(ct, profile, 0, torch.device("cuda", 0), 1, 0, 4, _runner())
    if out is None:
        pytest.skip("no window check passed on this shape (whole-pid fallback)")
    _check(ct, out, _whole(ct, profile, 0))
