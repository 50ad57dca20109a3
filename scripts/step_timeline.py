"""Host-side timeline of one analyse step: wall time of each public call with
and without graphs, against the device time of the same step (CUDA events)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2102_04285_b200 import _engine, synth  # noqa: E402

ct = synth.ddpg_trace(int(os.environ.get("XS_ITERS", "27027")))
eng = _engine.get(0)
dt = _engine.DeviceTrace(ct, 0)
scaled = synth.exact_profile().scaled(ct.names)


def timeit(fn, k=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev, host = [], []
    for _ in range(k):
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        host.append((time.perf_counter() - t0) * 1e3)
        dev.append(e0.elapsed_time(e1))
    dev.sort()
    host.sort()
    return dev[k // 2], host[k // 2]


for name, fn in [
    ("validate", lambda: eng.validate(dt) if hasattr(eng, "validate") else None),
    ("overlap", lambda: eng.overlap(dt, 0)),
    ("correct", lambda: eng.correct(dt, scaled)),
    ("analyze", lambda: eng.correct(dt, scaled, analyze_attribution=0)),
]:
    try:
        d, h = timeit(fn)
        print(f"{name:10s} device {d:.3f} ms  host {h:.3f} ms")
    except Exception as e:  # noqa: BLE001
        print(name, "skipped:", e)
