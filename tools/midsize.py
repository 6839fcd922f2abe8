"""Mid-size element counts (the paper's size sweep varies the element
count): GB/s of prebuilt libhadacore variants at n x 2^k elements, warm (50
launches replayed from one CUDA graph on the same buffers: L2-resident below ~2^24) and cold
(a 2 x L2 write before each event-timed launch).  Variants are interleaved, medians of
`--repeats` passes.

    python tools/midsize.py --libs a.so,b.so [--ns 256,512,4096] [--ks 22,23,24,25,26] [--repeats 3]
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


def load(path):
    lib = ctypes.CDLL(os.path.abspath(path))
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    lib.hadacore_fwht.argtypes = [vp, vp, i64, i64, ctypes.c_int, ctypes.c_float, vp]
    lib.hadacore_fwht.restype = ctypes.c_int
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--ns", default="256,512,1024,2048,4096,8192,16384,32768")
    ap.add_argument("--ks", default="22,23,24,25,26")
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--dtype", default="fp16")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    libs = {os.path.basename(p): load(p) for p in a.libs.split(",")}
    ns = [int(v) for v in a.ns.split(",")]
    ks = [int(v) for v in a.ks.split(",")]
    dt = {"fp16": torch.float16, "bf16": torch.bfloat16}[a.dtype]
    code = {"fp16": 0, "bf16": 1}[a.dtype]
    big = 1 << max(ks)
    x = torch.randn(big, device="cuda").to(dt)
    y = torch.empty_like(x)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size or 126000000
    scrub = torch.empty(2 * l2, dtype=torch.uint8, device="cuda")
    res = {}
    s = torch.cuda.Stream()
    for rep in range(a.repeats):
        for n in ns:
            for k in ks:
                e = 1 << k
                m = e // n
                for name, lib in libs.items():
                    def call(stream):
                        rc = lib.hadacore_fwht(x.data_ptr(), y.data_ptr(), m, n, code, 1.0 / n ** 0.5, stream)
                        assert rc == 0, rc
                    # warm: graph of 50 launches
                    with torch.cuda.stream(s):
                        for _ in range(3):
                            call(s.cuda_stream)
                        torch.cuda.synchronize()
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, stream=s):
                            for _ in range(50):
                                call(s.cuda_stream)
                        g.replay()
                        torch.cuda.synchronize()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(s)
                        g.replay()
                        e1.record(s)
                        torch.cuda.synchronize()
                        warm = 4.0 * e * 50 / (e0.elapsed_time(e1) * 1e-3) / 1e9
                        cold = []
                        for _ in range(5):
                            scrub.fill_(rep & 1)
                            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                            c0.record(s)
                            call(s.cuda_stream)
                            c1.record(s)
                            torch.cuda.synchronize()
                            cold.append(4.0 * e / (c0.elapsed_time(c1) * 1e-3) / 1e9)
                    res.setdefault((name, n, k), {"warm": [], "cold": []})
                    res[(name, n, k)]["warm"].append(warm)
                    res[(name, n, k)]["cold"].append(statistics.median(cold))
    out = []
    for (name, n, k), v in sorted(res.items(), key=lambda t: (t[0][1], t[0][2], t[0][0])):
        w, c = statistics.median(v["warm"]), statistics.median(v["cold"])
        out.append({"lib": name, "n": n, "log2_elems": k, "warm_GBps": round(w), "cold_GBps": round(c)})
        print(f"n={n:6d} 2^{k} {name:32s} warm {w:7.0f}  cold {c:7.0f} GB/s", flush=True)
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
