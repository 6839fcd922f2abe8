import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2412_08832_b200 as hc
x = torch.randn(8192, 32768, device="cuda"); y = torch.empty_like(x)
for _ in range(2): hc.hadacore_fwht(x, out=y)
torch.cuda.synchronize()
