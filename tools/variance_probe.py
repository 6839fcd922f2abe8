"""Batch-to-batch variance of one (n, dtype) configuration (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_08832_b200 as hc

elems = 1 << 28
x = torch.randn(elems, device="cuda").half()
o = torch.empty_like(x)
for n, dt in [(32768, torch.float16), (16384, torch.bfloat16), (128, torch.float16), (4096, torch.float16)]:
    xv, ov = x.view(torch.int16).view(dt).view(-1, n), o.view(torch.int16).view(dt).view(-1, n)
    for _ in range(3):
        hc.hadacore_fwht(xv, out=ov)
    vals = []
    for b in range(24):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            hc.hadacore_fwht(xv, out=ov)
        e1.record()
        e1.synchronize()
        vals.append(4.0 * elems / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e9)
    print(n, dt, " ".join(f"{v:.0f}" for v in vals), flush=True)
    # single launches individually timed
    single = []
    for b in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        hc.hadacore_fwht(xv, out=ov)
        e1.record()
        e1.synchronize()
        single.append(4.0 * elems / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    print("   single:", " ".join(f"{v:.0f}" for v in single), flush=True)
