"""Pipeline timeline of fwht_rows_kernel from an HC_TRACE build (dev tool).
    python tools/trace_pipeline.py build/tune/libhc_tuned_trace.so 32768"""
import ctypes
import sys

import numpy as np
import torch

lib = ctypes.CDLL(sys.argv[1])
n = int(sys.argv[2])
f = lib.hadacore_fwht
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_void_p]
elems = 1 << 28
x = torch.randn(elems, device="cuda").half()
y = torch.empty_like(x)
for _ in range(3):
    f(x.data_ptr(), y.data_ptr(), elems // n, n, 0, 1.0, None)
torch.cuda.synchronize()
buf = np.zeros((4, 48, 8), dtype=np.uint64)
assert lib.hadacore_trace_read(buf.ctypes.data, buf.nbytes) == 0
names = ["load_issue", "done_seen(prod)", "store_issued", "", "full_seen(cons)", "phase1_done", "phase2_done", ""]
for cta in range(2):
    t0 = buf[cta, 0, 0]
    print(f"CTA {cta} (us from first load issue)")
    for it in range(0, 24):
        row = buf[cta, it]
        vals = {names[e]: (int(row[e]) - int(t0)) / 1000 for e in (0, 4, 5, 6, 1, 2) if row[e]}
        print(f"  tile {it:2d}: " + "  ".join(f"{k}={v:7.2f}" for k, v in vals.items()))
    d = buf[cta, 1:40]
    full = d[:, 4].astype(np.int64); p1 = d[:, 5].astype(np.int64); p2 = d[:, 6].astype(np.int64)
    ld = d[:, 0].astype(np.int64)
    print(f"  median: load->full {np.median(full - ld)/1000:.2f} us, full->p1 {np.median(p1 - full)/1000:.2f}, "
          f"p1->p2 {np.median(p2 - p1)/1000:.2f}, tile period {np.median(np.diff(full))/1000:.2f} us")

span = np.zeros((1024, 3), dtype=np.uint64)
assert lib.hadacore_span_read(span.ctypes.data, span.nbytes) == 0
grid = int((span[:, 1] > 0).sum())
t0 = span[:grid, 0].astype(np.int64).min()
start = (span[:grid, 0].astype(np.int64) - t0) / 1000
end = (span[:grid, 1].astype(np.int64) - t0) / 1000
tiles = span[:grid, 2].astype(np.int64)
per = (end - start) / tiles
print(f"CTAs {grid}: start max {start.max():.2f} us; end min {end.min():.1f} median {np.median(end):.1f} max {end.max():.1f} us; "
      f"tiles {tiles.min()}..{tiles.max()}; us/tile min {per.min():.2f} median {np.median(per):.2f} max {per.max():.2f}")
order = np.argsort(per)
print("slowest CTAs:", [(int(i), round(float(per[i]), 2)) for i in order[-8:]])
print("fastest CTAs:", [(int(i), round(float(per[i]), 2)) for i in order[:8]])
