"""Per-stage device times (xs_profile_*) of a few xs_analyze calls on a config-2/3 trace."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2102_04285_b200 import _engine, synth  # noqa: E402

cfg = int(os.environ.get("XS_CONFIG", "2"))
if cfg == 3:
    ev = int(os.environ.get("XS_EVENTS", "30000000"))
    ct = synth.config3_trace(processes=ev // 1_000_000, events_per_pid=1_000_000, workers=os.cpu_count())
elif cfg == 5:
    ct = synth.adversarial_trace(int(os.environ.get("XS_EVENTS", "10000000")), pids=64, workers=os.cpu_count())
else:
    ct = synth.ddpg_trace(27027)
eng = _engine.get(0)
dt = _engine.DeviceTrace(ct, 0)
sc = (synth.adversarial_profile() if cfg == 5 else synth.exact_profile()).scaled(ct.names)
for _ in range(3):
    eng.correct(dt, sc, analyze_attribution=0)
torch.cuda.synchronize()
tt = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.correct(dt, sc, analyze_attribution=0)
    e1.record()
    e1.synchronize()
    tt.append(e0.elapsed_time(e1))
print("step ms", " ".join(f"{t:.3f}" for t in tt), "events", ct.n)
eng.lib.xs_profile_enable(eng.ctx, 1)
K = 5
for _ in range(K):
    eng.correct(dt, sc, analyze_attribution=0)
torch.cuda.synchronize()
ms = np.zeros(32)
calls = np.zeros(32, np.int64)
nst = eng.lib.xs_profile_read(eng.ctx, ms.ctypes.data, calls.ctypes.data, 32)
print(os.environ.get("XS_LIB_PATH", "default"), " ".join(
    f"{eng.lib.xs_profile_stage_name(i).decode()}={ms[i] / K:.3f}" for i in range(nst) if calls[i]))
