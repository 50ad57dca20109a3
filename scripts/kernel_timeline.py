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
import json  # noqa: E402
import tempfile  # noqa: E402

path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
tr = json.load(open(path))
acts = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
ks = sorted((float(e["ts"]), float(e["ts"]) + float(e.get("dur", 0)), e["name"], e.get("args", {}).get("stream", -1),
             e["cat"]) for e in acts)
# the second step starts at the second-to-last k_init_stats pair: take the last third of the list
firsts = [i for i, k in enumerate(ks) if "k_init_stats" in k[2]]
start = firsts[len(firsts) // 2] if len(firsts) >= 2 else 0
ks = ks[start:]
t0 = ks[0][0]
end = max(k[1] for k in ks)
print(f"activities {len(ks)}  span {end - t0:.1f} us")
for s_, e_, n, st, cat in ks:
    short = n.split("(")[0].replace("void ", "")[:60]
    print(f"{s_ - t0:8.1f} {e_ - t0:8.1f} {e_ - s_:7.1f}  s{st:<3} {'M ' if cat != 'kernel' else '  '}{short}")
iv = sorted((s_, e_) for s_, e_, _, _, _ in ks)
u = 0.0
cs, ce = iv[0]
for s_, e_ in iv[1:]:
    if s_ > ce:
        u += ce - cs
        cs, ce = s_, e_
    else:
        ce = max(ce, e_)
u += ce - cs
print(f"device busy (union of activities) {u:.1f} us of {end - t0:.1f} us")
