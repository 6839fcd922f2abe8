"""One Q/K-heads rotate+quantize launch (hadacore_fwht_quant_strided) and one contiguous
fused quantization launch of the same rows, fp16, for ncu comparison:
    ncu -k regex:fwht -s 2 -c 2 python tools/ncu_qk.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_08832_b200 as hc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
H = max(1, 4096 // n)
T = (1 << 28) // (3 * H * n)
qkv = torch.randn(T, 3, H, n, device="cuda").to(torch.float16)
qk = qkv[:, 0:2]
flat = qk.contiguous()
for _ in range(2):
    q, s = hc.hadacore_fwht_quant_strided(qk, "e4m3")
    q2, s2 = hc.hadacore_fwht_quant(flat.view(-1, n), "e4m3")
torch.cuda.synchronize()
