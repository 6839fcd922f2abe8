"""Isolated vs back-to-back launch times of the fp32 path (n = 2^14 and 2^15, 2^28 elements):
one launch between synchronizations (cold start, as ncu serializes) and 10 back-to-back."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_08832_b200 as hc

elems = 1 << 28
x = torch.randn(elems, device="cuda")
y = torch.empty_like(x)
scrub = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
for n in (16384, 32768):
    a, b = x.view(-1, n), y.view(-1, n)
    for _ in range(3):
        hc.hadacore_fwht(a, out=b)
    iso = []
    for _ in range(5):
        scrub.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hc.hadacore_fwht(a, out=b)
        e1.record()
        torch.cuda.synchronize()
        iso.append(e0.elapsed_time(e1) * 1e3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        hc.hadacore_fwht(a, out=b)
    e1.record()
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) * 1e3 / 10
    print(f"n={n} isolated_us={[round(t, 1) for t in iso]} back_to_back_us={b2b:.1f} "
          f"GBps_iso={8 * elems / min(iso) / 1e3:.0f} GBps_b2b={8 * elems / b2b / 1e3:.0f}")
