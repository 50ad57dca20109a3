"""One short workload for ncu captures: N xs_analyze calls on a bench trace.

    XS_CONFIG=2 (default): the config-2 DDPG trace (XS_ITERS iterations)
    XS_CONFIG=3: config 3 with XS_EVENTS events (100 pids of 1M by default)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2102_04285_b200 import _engine, synth  # noqa: E402

cfg = int(os.environ.get("XS_CONFIG", "2"))
calls = int(os.environ.get("XS_CALLS", "2"))
if cfg == 5:
    ct = synth.adversarial_trace(int(os.environ.get("XS_EVENTS", "10000000")), pids=64, workers=os.cpu_count())
elif cfg == 3:
    ev = int(os.environ.get("XS_EVENTS", "100000000"))
    procs = max(1, ev // 1_000_000)
    ct = synth.config3_trace(processes=procs, events_per_pid=ev // procs, workers=os.cpu_count())
else:
    ct = synth.ddpg_trace(int(os.environ.get("XS_ITERS", "27027")))
eng = _engine.get(0)
dt = _engine.DeviceTrace(ct, 0)
scaled = (synth.adversarial_profile() if cfg == 5 else synth.exact_profile()).scaled(ct.names)
for _ in range(calls):
    eng.correct(dt, scaled, analyze_attribution=0)
print("events", ct.n)
