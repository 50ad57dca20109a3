"""Host packing cost (xs_pack_plan / xs_pack_fill) of the config-2 trace into
a reused page-locked block, per thread count: the staging half of the
from-numpy e2e path."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2102_04285_b200 import _lib, synth  # noqa: E402
from paper_2102_04285_b200.columnar import _host_events  # noqa: E402

ct = synth.ddpg_trace(27027)
lib = _lib.load()
print("cpus", os.cpu_count())
block = None
for threads in (0, 1, 2, 4, 8, 16):
    best = [1e9, 1e9]
    for _ in range(8):
        ev, keep = _host_events(ct)
        nat = _lib.XsPackLayout()
        t0 = time.perf_counter()
        lib.xs_pack_plan(C.byref(ev), threads, C.byref(nat))
        t1 = time.perf_counter()
        if block is None or block.numel() < nat.total:
            block = torch.empty(int(nat.total) + 1024, dtype=torch.uint8).pin_memory()
        t2 = time.perf_counter()
        lib.xs_pack_fill(C.byref(ev), C.byref(nat), block.data_ptr(), block.numel())
        t3 = time.perf_counter()
        best = [min(best[0], t1 - t0), min(best[1], t3 - t2)]
    print(f"threads {threads} ({nat.n_threads}): plan {best[0] * 1e3:.2f} ms fill {best[1] * 1e3:.2f} ms")
