"""One fused FWHT+quantization launch per (dtype, n) at 2^28 elements after one warm-up
pass (ncu captures: -k regex:fwht -s <2*len(ns)> -c <2*len(ns)>).

    python tools/ncu_quant.py [ns] [e4m3|int8|int4]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_08832_b200 as hc  # noqa: E402

ns = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128,256,512,1024,2048,4096,8192,16384,32768").split(",")]
qtype = sys.argv[2] if len(sys.argv) > 2 else "e4m3"
elems = 1 << 28
src = torch.randn(elems, device="cuda").to(torch.float16)
q = torch.empty(elems, dtype=hc.QTYPES[qtype][1], device="cuda")
sc = torch.empty(elems // 128, dtype=torch.float32, device="cuda")
for _ in range(2):
    for dt in (torch.float16, torch.bfloat16):
        for n in ns:
            x = src.view(torch.int16).view(dt).view(-1, n)
            hc.hadacore_fwht_quant(x, qtype=qtype, out=q[: elems // (2 if qtype == "int4" else 1)].view(
                -1, n // 2 if qtype == "int4" else n), row_scale=sc[: x.shape[0]])
torch.cuda.synchronize()
