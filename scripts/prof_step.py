"""One short workload for ncu captures: N xs_analyze calls on the bench trace."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2102_04285_b200 import _engine, synth  # noqa: E402

iters = int(os.environ.get("XS_ITERS", "27027"))
calls = int(os.environ.get("XS_CALLS", "2"))
ct = synth.ddpg_trace(iters)
eng = _engine.get(0)
dt = _engine.DeviceTrace(ct, 0)
scaled = synth.exact_profile().scaled(ct.names)
for _ in range(calls):
    eng.correct(dt, scaled, analyze_attribution=0)
print("events", ct.n)
