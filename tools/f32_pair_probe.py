"""Timing probe of the fp32 n = 2^15 path (2-CTA cluster kernel): full 2^28-element
launch, and launch time vs m (rows) to expose the co-resident cluster count."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_08832_b200 as hc  # noqa: E402


def t_ms(x, y, reps=5):
    hc.hadacore_fwht(x, out=y)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        hc.hadacore_fwht(x, out=y)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


x = torch.randn(8192, 32768, device="cuda")
y = torch.empty_like(x)
ms = t_ms(x, y)
print(f"n=32768 fp32 m=8192: {ms:.4f} ms, {8 * x.numel() / ms / 1e6:.1f} GB/s")
for m in [1, 2, 8, 16, 32, 48, 64, 70, 72, 74, 76, 96, 128, 148, 222, 296]:
    print(f"m={m:4d}: {1e3 * t_ms(x[:m], y[:m], 20):8.2f} us")
