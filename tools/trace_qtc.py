"""Pipeline timeline of fwht_quant_tc_kernel from an HC_TRACE build (dev tool):
    python tools/trace_qtc.py lib_trace.so 8192 [e4m3|int8|int4]
Events per tile (us from the CTA's first load): load issued, phase A start/done (first
phase-A warp), MMA: phase A seen / issued (after the TMEM buffer is free), epilogue (warp 0):
TMEM full seen, row max done, buffer released."""
import ctypes
import sys

import numpy as np
import torch

lib = ctypes.CDLL(sys.argv[1])
n = int(sys.argv[2])
qt = {"e4m3": 0, "int8": 1, "int4": 2}[sys.argv[3] if len(sys.argv) > 3 else "e4m3"]
f = lib.hadacore_fwht_quant
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
              ctypes.c_int, ctypes.c_float, ctypes.c_void_p]
elems = 1 << 28
x = torch.randn(elems, device="cuda").half()
q = torch.empty(elems, dtype=torch.uint8, device="cuda")
sc = torch.empty(elems // n, dtype=torch.float32, device="cuda")
for _ in range(3):
    assert f(x.data_ptr(), q.data_ptr(), sc.data_ptr(), elems // n, n, 0, qt, n ** -0.5, None) == 0
torch.cuda.synchronize()
buf = np.zeros((4, 48, 8), dtype=np.uint64)
assert lib.hadacore_trace_read(buf.ctypes.data, buf.nbytes) == 0
names = ["load", "A_start", "A_done", "mma_issue", "E_start", "E_max", "E_done", "mma_seenA"]
order = [0, 1, 2, 7, 3, 4, 5, 6]
for cta in range(2):
    t0 = int(buf[cta, 0, 0])
    print(f"CTA {cta} (us from first load)")
    for it in range(0, 20):
        row = buf[cta, it]
        print(f"  tile {it:2d}: " + "  ".join(f"{names[e]}={(int(row[e]) - t0) / 1000:7.2f}" for e in order if row[e]))
    d = buf[cta, 2:40].astype(np.int64)
    ok = (d > 0).all(axis=1)
    d = d[ok]
    med = lambda a, b: np.median(d[:, b] - d[:, a]) / 1000  # noqa: E731
    print(f"  median us: load->A_start {med(0, 1):.2f}, A {med(1, 2):.2f}, A_done->mma_seen {med(2, 7):.2f}, "
          f"mma_seen->issue {med(7, 3):.2f}, issue->E_start {med(3, 4):.2f}, E pass1+max {med(4, 5):.2f}, "
          f"E pass2 {med(5, 6):.2f}; periods: load {np.median(np.diff(d[:, 0]))/1000:.2f} A {np.median(np.diff(d[:, 1]))/1000:.2f} "
          f"E {np.median(np.diff(d[:, 4]))/1000:.2f}")
