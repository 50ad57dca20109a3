"""Host-side phases of one from-numpy config-2 e2e step (analyze_columnar on
ordinary numpy columns): staging (native pack into page-locked memory + DMA
+ unpack), the analysis to host buffers, fetch + decode -- and the whole
public call."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2102_04285_b200 import _engine, analyze_columnar, synth  # noqa: E402
from paper_2102_04285_b200.overlap import decode_breakdown  # noqa: E402

ct = synth.ddpg_trace(27027)
prof = synth.exact_profile()
eng = _engine.get(0)
hs = torch.empty(ct.n, dtype=torch.int64).pin_memory()
hd = torch.empty(ct.n, dtype=torch.int64).pin_memory()
rows = []
for it in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sc = prof.scaled(ct.names)
    t1 = time.perf_counter()
    staged = eng.stage_packed(ct)
    t2 = time.perf_counter()
    eng.staged_upload_done() if hasattr(eng, "staged_upload_done") else None
    dt = _engine.DeviceTrace(ct, 0)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    raw = eng.correct(dt, sc, 0, host_out=(hs, hd))
    t4 = time.perf_counter()
    bd = decode_breakdown(ct, eng.fetch_overlap())
    t5 = time.perf_counter()
    rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4))
r = np.median(np.array(rows[10:]), axis=0) * 1e3
print(f"profile.scaled {r[0]:.3f}  stage_packed {r[1]:.3f}  DeviceTrace(stage+DMA+unpack) {r[2]:.3f}  "
      f"analyze_to_host {r[3]:.3f}  fetch+decode {r[4]:.3f} ms")
ts = []
for it in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    analyze_columnar(ct, prof, out=(hs, hd))
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"analyze_columnar(numpy ct, out=pinned): {np.median(ts[10:]) * 1e3:.3f} ms")
