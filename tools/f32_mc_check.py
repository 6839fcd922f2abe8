"""Quick check of the fp32 n = 2^15 kernel (dev tool): a few row counts vs the fp64 oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2412_08832_b200 as hc  # noqa: E402
import synthetic  # noqa: E402

for m in (1, 2, 3, 149, 1000):
    x = synthetic.generate(m, 32768, torch.float32, 77 + m).cuda()
    y = hc.hadacore_fwht(x)
    torch.cuda.synchronize()
    k = min(m, 6)
    ref = oracle.fwht(x[:k].cpu().double().numpy())
    err = (np.linalg.norm(y[:k].cpu().double().numpy() - ref, axis=1) / np.linalg.norm(ref, axis=1)).max()
    print(m, f"{err:.2e}", flush=True)
