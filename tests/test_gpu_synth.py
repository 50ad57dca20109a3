"""Device synthetic generator (csrc/xs_synth.cu): the
generated twins are valid traces, correct back to each other exactly
(through the C oracle and through the device pipeline: InsertionMap then
RemovalMap with the same constant amounts, _timeline.py:3-19), and match the
host generator's shape (synth.py:246-375): identical per-iteration CPU event
structure and the same duration / kernel-probability statistics."""

import numpy as np
import pytest

import oracle
from paper_2102_04285_b200 import _engine, synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gen():
    return synth.device_ddpg_trace(300, processes=3, outer_op="iteration", second_tid_ops=True)


def test_device_generator_twins_valid_and_close_exactly(gen):
    un, inst = gen.columnar("un"), gen.columnar("inst")
    assert un.n == inst.n and un.n > 300 * 3 * 30
    assert oracle.validate_count(un) == 0 and oracle.validate_count(inst) == 0
    s, d, rep, _ = oracle.correct(inst, synth.exact_profile())
    assert np.array_equal(s, un.start) and np.array_equal(d, un.dur)
    assert rep["original_total_ns"] > rep["corrected_total_ns"]
    # the device pipeline on the resident columns (no host round trip)
    eng = _engine.get(0)
    raw = eng.correct(gen.device_trace("inst"), synth.exact_profile().scaled(inst.names), analyze_attribution=0)
    assert np.array_equal(raw.start.cpu().numpy(), un.start) and np.array_equal(raw.dur.cpu().numpy(), un.dur)


def test_device_generator_matches_host_generator_shape(gen):
    dev, dev_i = gen.columnar("un"), gen.columnar("inst")
    host, host_i = synth.ddpg_trace(300, processes=3, outer_op="iteration", second_tid_ops=True, both=True)
    for p in range(3):
        dc = np.bincount(dev.cat[dev.pid == p], minlength=6)
        hc = np.bincount(host.cat[host.pid == p], minlength=6)
        assert np.array_equal(dc[:5], hc[:5])                      # CPU structure: identical counts
        n_api = dc[4]
        assert abs(dc[5] - 0.7 * n_api) < 5 * np.sqrt(n_api * 0.21)  # kernel probability 0.7
    for d, h in ((dev, host), (dev_i, host_i)):  # both twins
        for cat in (2, 3, 4, 5):
            dm = d.dur[d.cat == cat].mean()
            hm = h.dur[h.cat == cat].mean()
            assert abs(dm - hm) / hm < 0.03, (cat, dm, hm)
    names = [dev.names[i] for i in np.unique(dev.name)]
    assert sorted(names) == sorted(host.names[i] for i in np.unique(host.name))


def test_device_generator_pid_blocks_regenerate_the_same_processes():
    a = synth.device_ddpg_trace(50, processes=4, first_pid=1).columnar("inst")
    b = synth.device_ddpg_trace(50, processes=2, first_pid=3).columnar("inst")
    ra = a.pid >= 2
    assert np.array_equal(a.start[ra], b.start) and np.array_equal(a.dur[ra], b.dur)
    assert np.array_equal(a.cat[ra], b.cat) and np.array_equal(a.corr[ra], b.corr)
