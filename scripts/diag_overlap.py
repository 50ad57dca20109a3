"""Find the pid (and event subset) on which xs_overlap reports a violation the
oracle does not see (config 5 at 10M)."""
import os
import sys
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from paper_2102_04285_b200 import _engine, synth  # noqa: E402

n = int(os.environ.get("XS_N", "10000000"))
ct = synth.adversarial_trace(n, pids=64, workers=16)
eng = _engine.get(0)


def ov(c):
    try:
        eng.overlap(_engine.DeviceTrace(c, 0), 0)
        return "ok"
    except _engine.XsError as e:
        return str(e)


print("whole:", ov(ct), flush=True)
bad = []
for p in range(ct.n_pids):
    r = ov(ct.select_pids([p]))
    if r != "ok":
        bad.append(p)
        print("pid", p, int((ct.pid == p).sum()), r, flush=True)
print("bad pids", bad, flush=True)
for p in bad[:1]:
    sub = ct.select_pids([p])
    for cat in range(6):
        keep = sub.cat != cat
        if cat == 4:
            keep &= True
        s2 = sub.__class__(sub.clock_domain, sub.start[keep], sub.dur[keep], sub.pid[keep], sub.tid[keep],
                           sub.cat[keep], sub.name[keep], sub.corr[keep], sub.has_corr[keep], sub.pids,
                           sub.group_pid, sub.group_tid, sub.names, sub.processes, sub.pid_has_meta)
        if cat == 4:  # dropping APIs makes GPU correlations dangle: drop their ids too
            s2.has_corr[s2.cat == 5] = 0
        print("without cat", cat, ov(s2), flush=True)
