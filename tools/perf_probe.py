"""Quick per-(n, dtype) timing of the CUDA path at 2^28 elements (dev tool)."""
import argparse
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2412_08832_b200 as hc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=1 << 28)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--ns", default="128,256,512,1024,2048,4096,8192,16384,32768")
    ap.add_argument("--inplace", action="store_true")
    a = ap.parse_args()
    buf_in = torch.randn(a.elems, device="cuda").to(torch.float16)
    buf_out = torch.empty_like(buf_in)
    res = {}
    for dt in (torch.float16, torch.bfloat16):
        x0 = buf_in.view(torch.int16).view(dt)
        for n in map(int, a.ns.split(",")):
            x = x0.view(-1, n)
            o = x if a.inplace else buf_out.view(torch.int16).view(dt).view(-1, n)
            for _ in range(3):
                hc.hadacore_fwht(x, out=o)
            torch.cuda.synchronize()
            ts = []
            for _ in range(3):  # back-to-back launches so host overhead is hidden
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.reps):
                    hc.hadacore_fwht(x, out=o)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) / a.reps)
            ts.sort()
            med = ts[len(ts) // 2]
            gbs = 4.0 * a.elems / (med * 1e-3) / 1e9
            res[f"{str(dt)[6:]}_{n}"] = round(gbs, 1)
            print(f"{str(dt):15s} n={n:6d}  {med*1e3:8.1f} us  {gbs:7.1f} GB/s  ({gbs/6538*100:5.1f}% of measured copy)",
                  flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
