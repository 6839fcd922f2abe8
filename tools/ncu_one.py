"""One launch per (dtype, n) at 2^28 elements, after one warm-up pass (for ncu captures:
use -k regex:fwht_kernel -s <18 or 2*len(ns)> -c <2*len(ns)>)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_08832_b200 as hc

ns = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128,256,512,1024,2048,4096,8192,16384,32768").split(",")]
elems = 1 << 28
src = torch.randn(elems, device="cuda").to(torch.float16)
dst = torch.empty_like(src)
for _ in range(2):
    for dt in (torch.float16, torch.bfloat16):
        for n in ns:
            hc.hadacore_fwht(src.view(torch.int16).view(dt).view(-1, n), out=dst.view(torch.int16).view(dt).view(-1, n))
torch.cuda.synchronize()
