"""Device timeline of one analyze step (config 2 by default): every kernel's
start/end on its stream, from CUPTI activity records via torch.profiler
(graph-launched kernels included).  Prints the kernels in start order with
their offset from the step's first kernel, duration, stream, and the gaps on
the critical stream.  XS_CONFIG=3 XS_EVENTS=N for the config-3 shape."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2102_04285_b200 import _engine, synth  # noqa: E402

cfg = int(os.environ.get("XS_CONFIG", "2"))
if cfg == 3:
    ev = int(os.environ.get("XS_EVENTS", "30000000"))
    ct = synth.config3_trace(processes=ev // 1_000_000, events_per_pid=1_000_000, workers=os.cpu_count())
else:
    ct = synth.ddpg_trace(27027)
eng = _engine.get(0)
dt = _engine.DeviceTrace(ct, 0)
sc = synth.exact_profile().scaled(ct.names)
for _ in range(4):
    eng.correct(dt, sc, analyze_attribution=0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        eng.correct(dt, sc, analyze_attribution=0)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs if "xs::" in e.name or "k_" in e.name])
# the second step: from the second k_init_stats-like first kernel
firsts = [i for i, k in enumerate(ks) if "k_init_stats" in k[2]]
start = firsts[len(firsts) // 2] if len(firsts) >= 2 else 0
ks = ks[start:]
t0 = ks[0][0]
end = max(k[1] for k in ks)
print(f"kernels {len(ks)}  span {end - t0:.1f} us")
busy = 0.0
cur_end = t0
for s, e, n in ks:
    if s > cur_end:
        busy += 0
    short = n.split("(")[0].replace("void ", "")[:60]
    print(f"{s - t0:8.1f} {e - t0:8.1f} {e - s:7.1f}  {short}")
# idle time: union of kernel intervals vs span
iv = sorted((s, e) for s, e, _ in ks)
u = 0.0
cs, ce = iv[0]
for s, e in iv[1:]:
    if s > ce:
        u += ce - cs
        cs, ce = s, e
    else:
        ce = max(ce, e)
u += ce - cs
print(f"device busy (union of kernels) {u:.1f} us of {end - t0:.1f} us")
