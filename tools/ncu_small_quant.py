"""ncu: fused quantization n = 64 fp16, E4M3 then INT4 (ncu -k regex:fwht -s 2 -c 2)."""
import sys, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2412_08832_b200 as hc
x = torch.randn(1 << 28, device="cuda").to(torch.float16).view(-1, 64)
for _ in range(2):
    for q in ("e4m3", "int4"):
        hc.hadacore_fwht_quant(x, q)
torch.cuda.synchronize()
