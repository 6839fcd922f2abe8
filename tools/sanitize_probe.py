"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
fwht_kernel (n = 128, 256), fwht_rows_kernel (n = 512, 4096, 32768), strided rows, fused quantization
(E4M3 / INT8 / INT4, the register epilogues and the tcgen05 kernel: n = 4096 INT4, 16384, 32768,
contiguous and row grids, ragged last tiles), fwht_small_kernel (n = 2..64, ragged totals), the fp32 kernels
(incl. the 2-CTA cluster n = 2^15) and the quant-lab kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_08832_b200 as hc  # noqa: E402

torch.manual_seed(0)
dev = "cuda"
for dt in (torch.float16, torch.bfloat16):
    for n, m in ((128, 67), (256, 33), (512, 19), (4096, 5), (32768, 3), (2, 7), (4, 5), (8, 9), (16, 3), (64, 130)):
        x = torch.randn(m, n, device=dev).to(dt)
        y = hc.hadacore_fwht(x)
        hc.hadacore_fwht(x, out=x)
        if n >= 128:
            for q in ("e4m3", "int8", "int4"):
                hc.hadacore_fwht_quant(y, q)
    qkv = torch.randn(5, 3, 4, 128, device=dev).to(dt)
    hc.hadacore_fwht_strided(qkv[:, 0:2], out=qkv[:, 0:2])
for dt in (torch.float16, torch.bfloat16):  # row grids n = 8..64 (GRID small kernel), quantized grids, small-n quant
    for n in (8, 16, 64, 128, 1024):
        qkv = torch.randn(7, 3, 5, n, device=dev).to(dt)
        hc.hadacore_fwht_strided(qkv[:, 0:2], out=qkv[:, 0:2])
        for q in ("e4m3", "int8", "int4"):
            hc.hadacore_fwht_quant_strided(qkv[:, 0:2], q)
    for n, m in ((2, 7), (4, 5), (8, 3), (64, 33)):
        for q in ("e4m3", "int8", "int4"):
            hc.hadacore_fwht_quant(torch.randn(m, n, device=dev).to(dt), q)
for n, m in ((2, 5), (64, 9), (2048, 3), (16384, 2), (32768, 3)):
    x = torch.randn(m, n, device=dev)
    hc.hadacore_fwht(x)
    hc.fake_quant(x, "int4", per_tensor=True)
    hc.row_sq_error(x, x)
x = torch.randn(160, 32768, device=dev)  # fp32 ring kernel: some CTAs take 2 rows, so chunk slots are reused
hc.hadacore_fwht(x)
hc.hadacore_fwht(x, out=x)
for dt in (torch.float16, torch.bfloat16):  # the tcgen05 fused quantization: ragged tiles, row grids
    for n, m in ((16384, 5), (32768, 2), (8192, 9)):
        x = torch.randn(m, n, device=dev).to(dt)
        for q in ("e4m3", "int8", "int4"):
            hc.hadacore_fwht_quant(x, q)
    qkv = torch.randn(3, 3, 2, 16384, device=dev).to(dt)
    for q in ("e4m3", "int4"):
        hc.hadacore_fwht_quant_strided(qkv[:, 0:2], q)
torch.cuda.synchronize()
print("sanitize probe done")
