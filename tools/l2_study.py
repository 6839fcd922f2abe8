"""NEXT-2: in-place vs out-of-place FWHT across element counts on
B200's 126 MB L2 -- the paper's App. B effect (in-place helped at 8M
elements on A100 / 16M on H100, whose L2 is 40/50 MB).  Repeated launches on the
same buffers, so a working set that fits in L2 stays there; GB/s is algorithmic
(4 B/element) and can exceed the HBM roofline when L2-resident."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_08832_b200 as hc


def gbs(fn, elems, reps=50):
    """Replays `reps` launches captured in one CUDA graph: no host overhead between them
    (the C ABI is graph-capturable: no allocation, no synchronisation)."""
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    return 4.0 * elems / (a.elapsed_time(b) / reps * 1e-3) / 1e9


res = {}
# BASELINE configs[0]: fp16, m = 1024, n = 256 (L2-resident, latency-bound): per-launch time
x = torch.randn(1024, 256, device="cuda").half()
y = torch.empty_like(x)
g = gbs(lambda: hc.hadacore_fwht(x, out=y), x.numel(), reps=200)
res["C1_us_per_launch_graph"] = round(4.0 * x.numel() / (g * 1e9) * 1e6, 3)
print(f"C1 (fp16 1024x256): {res['C1_us_per_launch_graph']} us per launch in a CUDA graph ({g:.0f} GB/s)", flush=True)
for n in (256, 4096):
    for k in range(20, 29):
        e = 1 << k
        x = torch.randn(e, device="cuda").half().view(-1, n)
        y = torch.empty_like(x)
        oop = gbs(lambda: hc.hadacore_fwht(x, out=y), e)
        inp = gbs(lambda: hc.hadacore_fwht(x, out=x), e)
        res[f"n{n}_2^{k}"] = {"elements": e, "MB_in": 2 * e / 1e6, "out_of_place_GBps": round(oop), "in_place_GBps": round(inp),
                              "in_place_speedup": round(inp / oop, 3)}
        print(f"n={n:5d} elems=2^{k} ({2*e/1e6:7.1f} MB) out-of-place {oop:8.0f} GB/s  in-place {inp:8.0f} GB/s  x{inp/oop:.2f}",
              flush=True)
json.dump(res, open(os.path.join("gpurun_out", "l2_study.json"), "w"), indent=1)
