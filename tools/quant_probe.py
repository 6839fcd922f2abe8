"""Launch the fused quantization for a few n (for ncu captures; dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_08832_b200 as hc

ns = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [128, 4096]
qt = sys.argv[2] if len(sys.argv) > 2 else "e4m3"
elems = 1 << 28
x = torch.randn(elems, device="cuda").to(torch.bfloat16)
q = torch.empty(elems, dtype=hc.QTYPES[qt][1], device="cuda")
s = torch.empty(elems // 128, dtype=torch.float32, device="cuda")
for _ in range(2):
    for n in ns:
        hc.hadacore_fwht_quant(x.view(-1, n), qtype=qt, out=q.view(-1, n), row_scale=s[: elems // n])
torch.cuda.synchronize()
