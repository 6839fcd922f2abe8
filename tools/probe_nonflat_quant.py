"""n = 128 fused quantization: flat (contiguous) vs non-flat (row-grid) kernel instantiations on the SAME
contiguous bytes, and a true Q/K strided view -- to separate code cost from memory layout."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_08832_b200 as hc  # noqa: E402


def gbps(fn, elems, reps=20):
    fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return (3.0 * elems + 4.0 * elems / 128) * reps / (s.elapsed_time(e) * 1e-3) / 1e9


n, H = 128, 32
E = 1 << 28
x = torch.randn(E, device="cuda").to(torch.float16)
q = torch.empty(E, dtype=torch.float8_e4m3fn, device="cuda")
sc = torch.empty(E // n, dtype=torch.float32, device="cuda")
flat = x.view(-1, n)
print("flat contiguous     ", round(gbps(lambda: hc.hadacore_fwht_quant(flat, "e4m3", out=q.view(-1, n), row_scale=sc), E)))
grid = x.view(-1, 2 * H, n)  # contiguous bytes, but a 2-level grid (m_inner = 64) -> non-flat kernel
print("grid on contiguous  ", round(gbps(lambda: hc.hadacore_fwht_quant_strided(grid, "e4m3", out=q.view(-1, n), row_scale=sc), E)))
T = E // (3 * H * n)
qkv = x[: T * 3 * H * n].view(T, 3, H, n)[:, 0:2]
e2 = qkv.numel()
print("Q/K strided view    ", round(gbps(lambda: hc.hadacore_fwht_quant_strided(qkv, "e4m3", out=q[:e2], row_scale=sc[: e2 // n]), e2)))
