"""PCIe upload rate of one pinned column block and the analyze_columnar e2e time (config 2)."""
import sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2102_04285_b200 import analyze_columnar, synth
ct = synth.ddpg_trace(27027); pin = ct.pinned(); prof = synth.exact_profile()
hs = torch.empty(ct.n, dtype=torch.int64).pin_memory(); hd = torch.empty(ct.n, dtype=torch.int64).pin_memory()
blk = pin._pinned["_block"]
for _ in range(5): analyze_columnar(pin, prof, out=(hs, hd))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts=[]
for _ in range(10):
    e0.record(); d = blk.to('cuda', non_blocking=True); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
print("H2D block ms", min(ts), "GB/s", blk.numel()/min(ts)/1e6)
ts=[]
for _ in range(10):
    torch.cuda.synchronize(); t0=time.perf_counter(); analyze_columnar(pin, prof, out=(hs, hd)); ts.append((time.perf_counter()-t0)*1e3)
print("e2e ms", sorted(ts)[:5])
