"""Device time of the first calls on a new trace shape (eager sizing, capture, replays)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2102_04285_b200 import _engine, synth  # noqa: E402

ev = int(os.environ.get("XS_EVENTS", "30000000"))
ct = synth.config3_trace(processes=ev // 1_000_000, events_per_pid=1_000_000, workers=os.cpu_count())
eng = _engine.get(0)
dt = _engine.DeviceTrace(ct, 0)
sc = synth.exact_profile().scaled(ct.names)
for i in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.correct(dt, sc, analyze_attribution=0)
    torch.cuda.synchronize()
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
