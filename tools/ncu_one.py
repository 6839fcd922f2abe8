"""One launch per (dtype, n) at 2^28 elements, after one warm-up pass (for ncu captures:
use -k regex:fwht_kernel -s <len(dtypes)*len(ns)> -c <len(dtypes)*len(ns)>).

    python tools/ncu_one.py [ns] [dtypes: f16,bf16 (default) | f32]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_08832_b200 as hc

ns = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128,256,512,1024,2048,4096,8192,16384,32768").split(",")]
dts = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}
dtypes = [dts[d] for d in (sys.argv[2] if len(sys.argv) > 2 else "f16,bf16").split(",")]
elems = 1 << 28
src = {dt: torch.randn(elems, device="cuda").to(dt) for dt in dtypes}
dst = {dt: torch.empty_like(src[dt]) for dt in dtypes}
for _ in range(2):
    for dt in dtypes:
        for n in ns:
            hc.hadacore_fwht(src[dt].view(-1, n), out=dst[dt].view(-1, n))
torch.cuda.synchronize()
