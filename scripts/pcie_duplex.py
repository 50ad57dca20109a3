"""PCIe ceiling for the pipelined e2e: H2D alone, D2H alone, both at once (pinned, 1.6 GB each)."""
import time

import torch

n = 1_600_000_000
h_up = torch.empty(n, dtype=torch.uint8).pin_memory()
h_dn = torch.empty(n, dtype=torch.uint8).pin_memory()
d_up = torch.empty(n, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(up, dn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if up:
        with torch.cuda.stream(s1):
            d_up.copy_(h_up, non_blocking=True)
    if dn:
        with torch.cuda.stream(s2):
            h_dn.copy_(d_dn, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


for _ in range(2):
    a, b, c = run(True, False), run(False, True), run(True, True)
print(f"H2D {a:.1f} ms ({n / a / 1e6:.1f} GB/s)  D2H {b:.1f} ms ({n / b / 1e6:.1f} GB/s)  both {c:.1f} ms")
