"""The hashed global overlap histogram (csrc/xs_overlap.cu, GHist) used when
the dense [pid][node][32] layout is too large: forced on at small sizes in a
subprocess (XS_HIST_DENSE_MAX_LOG2=0) and compared bit-exactly with the
oracle, INSTANT and CORRELATION, plus one analyze call."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys
sys.path[:0] = [{root!r}, {root!r} + "/oracle"]
import numpy as np, oracle
from paper_2102_04285_b200 import Attribution, analyze_columnar, compute_overlap_columnar, synth, ColumnarTrace

def ours(bd):
    return ({{(k.pid, k.path, frozenset(int(c) for c in k.categories)): v for k, v in bd.cells.items()}},
            bd.spans, bd.untracked)

ct = synth.adversarial_trace(80_000, pids=8, streams=32)
assert ours(compute_overlap_columnar(ct)) == oracle.overlap(ct, 0), "instant"
assert ours(compute_overlap_columnar(ct, Attribution.CORRELATION)) == oracle.overlap(ct, 1), "correlation"
un, inst = synth.config3_trace(processes=3, events_per_pid=20_000, both=True)
s, d, rep, bd = analyze_columnar(inst, synth.exact_profile())
assert np.array_equal(s.cpu().numpy(), un.start)
assert ours(bd) == oracle.overlap(un, 0), "analyze"
print("hashed ok")
'''


def test_hashed_histogram_vs_oracle():
    env = dict(os.environ, XS_HIST_DENSE_MAX_LOG2="0")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "hashed ok" in r.stdout, r.stdout + r.stderr
