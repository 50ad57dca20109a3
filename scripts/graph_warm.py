"""Which segments are eager / captured / replayed on each of the first calls
(XS_DEBUG_GRAPH=1 prints misses and workspace growth to stderr)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2102_04285_b200 import _engine, synth  # noqa: E402

ct = synth.ddpg_trace(27027)
eng = _engine.get(0)
dt = _engine.DeviceTrace(ct, 0)
sc = synth.exact_profile().scaled(ct.names)
raw = None  # (held across calls like bench.py: output buffers alternate between two addresses)
for i in range(6):
    print(f"--- call {i}", file=sys.stderr, flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    raw = eng.correct(dt, sc, analyze_attribution=0)
    e1.record()
    torch.cuda.synchronize()
    print(f"--- call {i} {e0.elapsed_time(e1):.3f} ms", file=sys.stderr, flush=True)
