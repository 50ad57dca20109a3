"""Host-side profile of one analyze_columnar step (the bench's e2e path)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2102_04285_b200 import analyze_columnar, synth  # noqa: E402

if os.environ.get("XS_CONFIG") == "5":
    ct = synth.adversarial_trace(10_000_000, pids=64, workers=os.cpu_count())
    prof = synth.adversarial_profile()
else:
    ct = synth.ddpg_trace(27027)
    prof = synth.exact_profile()
pin = ct.pinned(packed=os.environ.get("XS_PACKED", "1") == "1")
hs = torch.empty(ct.n, dtype=torch.int64).pin_memory()
hd = torch.empty(ct.n, dtype=torch.int64).pin_memory()
for _ in range(2 if os.environ.get("XS_CONFIG") == "5" else 5):
    analyze_columnar(pin, prof, out=(hs, hd))
torch.cuda.synchronize()
ts = []
R = 2 if os.environ.get("XS_CONFIG") == "5" else 10
for _ in range(R):
    t0 = time.perf_counter()
    analyze_columnar(pin, prof, out=(hs, hd))
    ts.append((time.perf_counter() - t0) * 1e3)
print("analyze_columnar(out=pinned) ms:", [round(t, 3) for t in ts])
pr = cProfile.Profile()
pr.enable()
for _ in range(R):
    analyze_columnar(pin, prof, out=(hs, hd))
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
