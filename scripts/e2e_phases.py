"""Host-side phases of one config-2 e2e step (analyze_columnar on the packed
pinned trace): upload+unpack, xs_analyze_to_host, fetch, decode."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2102_04285_b200 import _engine, synth  # noqa: E402
from paper_2102_04285_b200.overlap import decode_breakdown  # noqa: E402

ct = synth.ddpg_trace(27027)
pin = ct.pinned()
prof = synth.exact_profile()
eng = _engine.get(0)
sc = prof.scaled(ct.names)
hs = torch.empty(ct.n, dtype=torch.int64).pin_memory()
hd = torch.empty(ct.n, dtype=torch.int64).pin_memory()
rows = []
for it in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dt = _engine.DeviceTrace(pin, 0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    raw = eng.correct(dt, sc, 0, host_out=(hs, hd))
    t2 = time.perf_counter()
    ov = eng.fetch_overlap()
    t3 = time.perf_counter()
    decode_breakdown(pin, ov)
    t4 = time.perf_counter()
    rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3))
r = np.median(np.array(rows[10:]), axis=0) * 1e3
print(f"upload+unpack {r[0]:.3f} ms  analyze_to_host {r[1]:.3f} ms  fetch {r[2]:.3f} ms  decode {r[3]:.3f} ms")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
dt = _engine.DeviceTrace(pin, 0)
ts = []
for it in range(20):
    torch.cuda.synchronize()
    e0.record()
    eng.correct(dt, sc, 0, host_out=(hs, hd))
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ts2 = []
for it in range(20):
    torch.cuda.synchronize()
    e0.record()
    eng.correct(dt, sc, 0)
    e1.record()
    e1.synchronize()
    ts2.append(e0.elapsed_time(e1))
print(f"device: analyze_to_host {np.median(ts[5:]):.3f} ms  analyze {np.median(ts2[5:]):.3f} ms")
