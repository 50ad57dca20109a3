"""Diagnose a device 'invalid trace' verdict the oracle does not share:
validate the whole trace, then each pid alone, then bisect the failing pid's
OPERATION events by time."""
import os
import sys
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle  # noqa: E402
from paper_2102_04285_b200 import _engine, synth  # noqa: E402

n = int(os.environ.get("XS_N", "10000000"))
ct = synth.adversarial_trace(n, pids=64, workers=16)
eng = _engine.get(0)
print("whole:", eng.validate(_engine.DeviceTrace(ct, 0)), "oracle:", oracle.validate_count(ct), flush=True)
bad = []
for p in range(ct.n_pids):
    sub = ct.select_pids([p])
    nb = eng.validate(_engine.DeviceTrace(sub, 0))
    if nb:
        bad.append(p)
        print("pid", p, "events", sub.n, "device n_bad", nb, "oracle", oracle.validate_count(sub), flush=True)
print("bad pids", bad)
if bad:
    sub = ct.select_pids([bad[0]])
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", "bad_pid.npz"), start=sub.start, dur=sub.dur, pid=sub.pid,
                        tid=sub.tid, cat=sub.cat, name=sub.name, corr=sub.corr, has_corr=sub.has_corr)
