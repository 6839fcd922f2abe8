"""Launch-configuration sweep (dev tool): build libhadacore variants with different
HC_* macros (NT compute warps, tile KiB, ring stages, unroll U) and time each
(n, dtype) at 2^28 elements on the GPU.

    python tools/tune.py build  "8,32,4,2" "16,32,4,2" ...   # here (nvcc)
    python tools/tune.py run                                  # on the GPU box
"""
import ctypes
import glob
import json
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "build", "tune")
NS = [1 << k for k in range(7, 16)]


def build_one(spec):
    """spec: "nt,tile_kb,stages,u[,ctas]" or "tuned" / "tuned-nocompute" (per-n table)."""
    base = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC", "-shared"]
    if spec.startswith("tuned"):
        name = spec.replace("-", "_")
        extra = (["-DHC_NOCOMPUTE"] if "nocompute" in spec else []) + (["-DHC_SIMT"] if "simt" in spec else []) + \
            (["-DHC_SEG"] if "-seg" in spec else []) + (["-DHC_STG_OUT"] if "stgout" in spec else []) + \
            (["-DHC_NO_PDL"] if "nopdl" in spec else []) + \
            (["-DHC_TRACE"] if "trace" in spec else []) + \
            (["-DHC_STATIC_SCHED"] if "static" in spec else [])
    else:
        nt, tkb, st, u, ctas = (spec.split(",") + ["1"])[:5]
        name = f"nt{nt}_t{tkb}_s{st}_u{u}_c{ctas}"
        extra = ["-DHC_TUNE", f"-DHC_CTAS={ctas}", f"-DHC_NT={nt}", f"-DHC_TILE_KB={tkb}", f"-DHC_STAGES={st}",
                 f"-DHC_U={u}"]
    so = os.path.join(OUT, f"libhc_{name}.so")
    cmd = base + extra + ["-o", so, os.path.join(ROOT, "paper_2412_08832_b200", "csrc", "hadacore.cu")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return name, r.returncode, r.stderr[-2000:]


def build(specs):
    os.makedirs(OUT, exist_ok=True)
    with ThreadPoolExecutor(max_workers=8) as ex:
        for name, rc, err in ex.map(build_one, specs):
            print(name, "ok" if rc == 0 else f"FAILED\n{err}")


def run(reps=15, ns=None, repeats=3):
    """Times every built variant; the whole sweep is repeated `repeats` times
    (variants interleaved) and the median per (variant, dtype, n) is reported."""
    import statistics

    import torch
    libs = sorted(glob.glob(os.path.join(OUT, "libhc_*.so")))
    elems = 1 << 28
    src = torch.randn(elems, device="cuda").to(torch.float16)
    dst = torch.empty_like(src)
    st = torch.cuda.current_stream().cuda_stream

    def batch_ms(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / reps

    # TUNE_QT=e4m3|int8: time the fused quantization entry instead (3 B/element + 4 B/row)
    qt = {"": None, "e4m3": 0, "int8": 1}[os.environ.get("TUNE_QT", "")]
    qbuf = torch.empty(elems, dtype=torch.uint8, device="cuda") if qt is not None else None
    sbuf = torch.empty(elems // 128, dtype=torch.float32, device="cuda") if qt is not None else None
    fns = {}
    for path in libs:
        lib = ctypes.CDLL(path)
        if qt is None:
            f = lib.hadacore_fwht
            f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                          ctypes.c_float, ctypes.c_void_p]
        else:
            fq = lib.hadacore_fwht_quant
            fq.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                           ctypes.c_int, ctypes.c_int, ctypes.c_float, ctypes.c_void_p]

            def f(i, o, m, n, dt, sc, stream, fq=fq):  # o is ignored: codes/scales go to qbuf/sbuf
                return fq(i, qbuf.data_ptr() if o == dst.data_ptr() else o, sbuf.data_ptr(), m, n, dt, qt, sc, stream)
        fns[os.path.basename(path)[6:-3]] = f
    samples = {}
    mem = []
    # bench-like paired design: each variant runs whole C3 steps (18 different launches
    # back to back, each timed with its own events, as bench.py does); variants
    # alternate step by step so slow drifts of the box affect all of them alike
    pairs = [(dt, n) for dt in (0, 1) for n in (ns or NS)]
    for rep in range(repeats):
        mem.append(4.0 * elems / (batch_ms(lambda: dst.copy_(src)) * 1e-3) / 1e9)
        for name, f in fns.items():
            for _ in range(2):  # 1 warm-up step + 1 timed step per repeat
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in pairs]
                for (dt, n), (a, b) in zip(pairs, evs):
                    a.record()
                    f(src.data_ptr(), dst.data_ptr(), elems // n, n, dt, 1.0, st)
                    b.record()
                torch.cuda.synchronize()
            for (dt, n), (a, b) in zip(pairs, evs):
                nbytes = 4.0 * elems if qt is None else 3.0 * elems + 4.0 * elems / n
                samples.setdefault(name, {}).setdefault(f"{'f16' if dt == 0 else 'bf16'}_{n}", []).append(
                    nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    base = sorted(fns)[0] if "tuned" not in fns else "tuned"
    for name in fns:
        rel = {k: statistics.median([a / b for a, b in zip(v, samples[base][k])]) for k, v in samples[name].items()}
        agg = statistics.median([len(pairs) / sum(1.0 / samples[name][k][i] for k in samples[name])
                                 for i in range(repeats)])
        print(f"paired ratio vs {base}: {name} step-GB/s={agg:.0f} " + " ".join(f"{k}={r:.3f}" for k, r in rel.items()),
              flush=True)
    print(f"memcpy(copy_) back-to-back: median {statistics.median(mem):.0f} GB/s  samples {[round(v) for v in mem]}")
    # each variant must agree with the parity-tested default library (nocompute excluded)
    sys.path.insert(0, ROOT)
    import paper_2412_08832_b200 as hc
    small = torch.randn(1 << 20, device="cuda")
    for name, f in fns.items():
        if "nocompute" in name or qt is not None:
            continue
        worst = 0.0
        for dt, tdt in ((0, torch.float16), (1, torch.bfloat16)):
            x = small.to(tdt)
            for n in (ns or NS):
                xv = x.view(-1, n)
                ref = hc.hadacore_fwht(xv).float()
                o = torch.empty_like(xv)
                assert f(xv.data_ptr(), o.data_ptr(), xv.shape[0], n, dt, 1.0 / n ** 0.5, st) == 0
                err = ((o.float() - ref).norm(dim=1) / ref.norm(dim=1)).max().item()
                worst = max(worst, err)
        print(f"agreement {name}: max rel-L2 vs default library {worst:.2e}")
    if qt is not None:
        x = small.to(torch.bfloat16)
        for name, f in fns.items():
            bad = 0
            for n in (ns or NS):
                xv = x.view(-1, n)
                q_ref, s_ref = hc.hadacore_fwht_quant(xv, qtype=["e4m3", "int8"][qt])
                o = torch.empty(xv.numel(), dtype=torch.uint8, device="cuda")
                assert f(xv.data_ptr(), o.data_ptr(), xv.shape[0], n, 1, 1.0 / n ** 0.5, st) == 0
                bad += int((o.view(-1, n) != q_ref.view(torch.uint8)).sum())
            print(f"agreement {name}: quant codes differing from the default library: {bad}")
    results = {nm: {k: round(statistics.median(v)) for k, v in d.items()} for nm, d in samples.items()}
    spread = {nm: {k: round(max(v) - min(v)) for k, v in d.items()} for nm, d in samples.items()}
    for nm, res in results.items():
        print(nm, " ".join(f"{k}={v}" for k, v in res.items()), flush=True)
    keys = list(next(iter(results.values())).keys())
    best = {k: max(results, key=lambda nm: results[nm][k]) for k in keys}
    print("BEST", json.dumps({k: (best[k], results[best[k]][k], spread[best[k]][k]) for k in keys}))
    json.dump({"median": results, "spread": spread, "memcpy": mem}, open(os.path.join(ROOT, "gpurun_out", "tune.json"), "w"),
              indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        ns = [int(v) for v in os.environ["TUNE_NS"].split(",")] if os.environ.get("TUNE_NS") else None
        run(ns=ns, repeats=int(os.environ.get("TUNE_REPEATS", "3")))
