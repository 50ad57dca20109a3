import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
from paper_2102_04285_b200 import _engine, synth
ct = synth.ddpg_trace(27027)
eng = _engine.get(0)
dev = torch.device("cuda", 0)
for it in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lay, block, st = eng.stage_packed(ct)
    t1 = time.perf_counter()
    nb = max(lay.total, 16)
    d = st.get("_dev_cache")
    dblock = d[1] if d is not None else torch.empty(nb, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    dblock[:nb].copy_(block[:nb], non_blocking=True)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    dt = _engine.DeviceTrace(ct, 0)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    if it > 4:
        print(f"stage {1e3*(t1-t0):.3f} dma {1e3*(t3-t2):.3f} ({nb/1e6:.1f} MB, pinned={block.is_pinned()}) DeviceTrace {1e3*(t4-t3):.3f} ms")
