"""Full-scale parity in the driver-run GPU suite (BASELINE.json configs at
their stated sizes):

* config 2: the 1M-event DDPG-style trace corrected with the reference's own
  fractional ladder profile (build_profile(generate_calibration_ladder(
  preset_noisy(seed=1234, iterations=2000))), tests/golden/ladder_profile_*)
  -- whole trace vs the C oracle and vs the reference itself;
* config 3: 100M events (100 pids x 1M, nested ops on two tids, six
  categories), one analyze call, with the integer profile (closure against
  the uninstrumented twin) and with the ladder profile -- EVERY pid vs the C
  oracle, 4 sampled pids vs the reference;
* config 5: the full 10M adversarial trace (Zipf pids, depth-64 recursion,
  256 GPU streams, zero-duration events, duplicate correlations), one analyze
  call -- every pid vs the C oracle, 4 sampled pids vs the reference.

Each check covers the corrected start/duration columns, the CorrectionReport
rows and compute_overlap(corrected) cells / spans / untracked, bit for bit
(correction.py:115-186, overlap.py:106-188).
"""

import os

import numpy as np
import pytest

from fullscale_util import have_reference, oracle_check, pid_bounds, reference_check
from paper_2102_04285_b200 import CalibrationProfile, analyze_columnar, synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
WORKERS = os.cpu_count() or 1


def ladder_profile() -> CalibrationProfile:
    with open(os.path.join(GOLDEN, "ladder_profile_noisy1234_2000.txt")) as fh:
        return CalibrationProfile.from_text(fh.read())


def _analyze(ct, prof):
    s, d, rep, bd = analyze_columnar(ct, prof)
    return s.cpu().numpy(), d.cpu().numpy(), rep, bd


def _sample_pids(ct, k=4, lo=100_000, hi=1_100_000):
    sizes = np.diff(pid_bounds(ct))
    cand = [p for p in range(ct.n_pids) if lo <= sizes[p] <= hi]
    step = max(1, len(cand) // k)
    return cand[::step][:k]


needs_ref = pytest.mark.skipif(not have_reference(), reason="oracle/_ref (the built reference) not present")


@pytest.fixture(scope="module")
def cfg2_ladder():
    ct = synth.ddpg_trace(27027)
    prof = ladder_profile()
    return (ct, prof) + _analyze(ct, prof)


def test_config2_ladder_profile_whole_trace(cfg2_ladder):
    ct, prof, s, d, rep, bd = cfg2_ladder
    assert oracle_check(ct, bd, prof, s, d, rep) == []
    assert rep.original_total_ns > rep.corrected_total_ns


@needs_ref
def test_config2_ladder_profile_vs_reference(cfg2_ladder):
    ct, prof, s, d, rep, bd = cfg2_ladder
    errs, n = reference_check(ct, bd, [0], prof, s, d, rep)
    assert errs == [] and n == ct.n


@pytest.fixture(scope="module")
def cfg3_100m():
    return synth.config3_trace(processes=100, events_per_pid=1_000_000, both=True, workers=WORKERS)


def test_config3_100m_integer_profile_every_pid(cfg3_100m):
    un, inst = cfg3_100m
    assert inst.n >= 99_000_000 and inst.n_pids == 100
    prof = synth.exact_profile()
    s, d, rep, bd = _analyze(inst, prof)
    assert np.array_equal(s, un.start) and np.array_equal(d, un.dur)  # closure
    assert oracle_check(inst, bd, prof, s, d, rep, workers=WORKERS) == []


@pytest.fixture(scope="module")
def cfg3_ladder(cfg3_100m):
    _, inst = cfg3_100m
    prof = ladder_profile()
    return (inst, prof) + _analyze(inst, prof)


def test_config3_100m_ladder_profile_every_pid(cfg3_ladder):
    inst, prof, s, d, rep, bd = cfg3_ladder
    assert oracle_check(inst, bd, prof, s, d, rep, workers=WORKERS) == []


@needs_ref
def test_config3_100m_ladder_profile_vs_reference(cfg3_ladder):
    inst, prof, s, d, rep, bd = cfg3_ladder
    pids = _sample_pids(inst)
    errs, n = reference_check(inst, bd, pids, prof, s, d, rep)
    assert errs == [] and len(pids) == 4 and n >= 4 * 900_000


@pytest.fixture(scope="module")
def cfg5_full():
    ct = synth.adversarial_trace(10_000_000, pids=64, workers=WORKERS)
    prof = synth.adversarial_profile()
    return (ct, prof) + _analyze(ct, prof)


def test_config5_full_10m_analyze_every_pid(cfg5_full):
    ct, prof, s, d, rep, bd = cfg5_full
    assert ct.n >= 10_000_000
    assert oracle_check(ct, bd, prof, s, d, rep, workers=WORKERS) == []


@needs_ref
def test_config5_full_10m_analyze_vs_reference(cfg5_full):
    ct, prof, s, d, rep, bd = cfg5_full
    pids = _sample_pids(ct, lo=50_000, hi=1_100_000)
    errs, n = reference_check(ct, bd, pids, prof, s, d, rep)
    assert errs == [] and len(pids) == 4
