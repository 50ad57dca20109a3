"""e2e of analyze_columnar_pipelined on config 3 (100M events) vs batch count."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2102_04285_b200 import analyze_columnar_pipelined, synth  # noqa: E402

ev = int(os.environ.get("XS_EVENTS", "100000000"))
ct = synth.config3_trace(processes=ev // 1_000_000, events_per_pid=1_000_000, workers=os.cpu_count())
pin = ct.pinned()
prof = synth.exact_profile()
hs = torch.empty(ct.n, dtype=torch.int64).pin_memory()
hd = torch.empty(ct.n, dtype=torch.int64).pin_memory()
W = int(os.environ.get("XS_WORKERS", "2"))
for b in [int(x) for x in os.environ.get("XS_BATCHES", "4,8,16,32").split(",")]:
    for _ in range(3):
        analyze_columnar_pipelined(pin, prof, out=(hs, hd), batches=b, workers=W)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        analyze_columnar_pipelined(pin, prof, out=(hs, hd), batches=b, workers=W)
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"workers {W} batches {b}: ms {[round(t, 1) for t in ts]}  ev/s {ct.n / (min(ts) / 1e3) / 1e9:.3f} G", flush=True)
