#!/usr/bin/env python
"""Benchmark of the B200-native batched normalized FWHT (HadaCore hot path).

Metric (BASELINE.json): FWHT HBM GB/s vs n = 2^7..2^15 (bf16/fp16) at 1/2/4/8
B200; % of 8 TB/s.  One STEP = the paper's size sweep (config C3): for each
dtype in {fp16, bf16} and each n in 2^7..2^15, one hadacore_fwht call over a
resident 2^28-element matrix (512 MiB in, 512 MiB out, out-of-place) -- 18
kernel launches.  value = algorithmic bytes (read + write, 4 B/element) of all
ranks / max-over-ranks device time, in GB/s.  Inputs (512 MiB per launch) are
larger than the 126 MB L2, so no flush is needed between launches.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {hadacore,reference}]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Rank 0 prints ONE JSON line.  --impl reference times the fp64 CPU oracle (the
only reference that exists for this paper) on a bounded sample of the same
workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FWHT HBM GB/s vs n=2^7..2^15 (bf16/fp16) at 1/2/4/8 B200; % of 8 TB/s"
NS = [1 << k for k in range(7, 16)]
SMALL_NS = [1 << k for k in range(1, 7)]  # NEXT-2: rows shorter than the paper's 2^7 floor
ELEMS = 1 << 28
C5_ELEMS = 1 << 33  # BASELINE config C5: bf16 n = 2^15, 2^33 elements in total
NOMINAL_HBM_GBS = 8000.0
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["hadacore", "reference"], default="hadacore")
    ap.add_argument("--elems", type=int, default=ELEMS, help="elements per (n, dtype) launch per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--inplace", action="store_true",
                    help="transform the resident input in place (P:264-274 App. B) instead of out of place")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--ns", default=None, help="comma-separated n list overriding the workload's sweep "
                                               "(e.g. --workload quant-e4m3 --ns 2,4,8,16,32,64)")
    ap.add_argument("--check-rows", type=int, default=4,
                    help="output rows per rank per launch gathered to rank 0 for the oracle and bitwise checks")
    ap.add_argument("--misshard", action="store_true",
                    help="negative control of the multi-rank check: rank 1 (rank 0 at N=1) generates its rows "
                         "one base row off; the sampled-row check must then fail (exit code 3)")
    ap.add_argument("--workload", choices=["fwht", "quant-e4m3", "quant-int8", "quant-int4", "qk-rotate", "qk-quant", "small", "f32", "c5",
                             "c1", "c2", "c4", "lab"], default="fwht",
                    help="fwht = the metric's C3 sweep (default); quant-* = the fused FWHT + per-row "
                         "quantization row (NEXT-1) on the same inputs; small = n=2^1..2^6 (NEXT-2); "
                         "f32 = the fp32 path over n=2^1..2^15 (NEXT-2); c5 = BASELINE config C5: bf16 "
                         "n=2^15, 2^33 elements row-sharded over the ranks (strong scaling); c1 = BASELINE config "
                         "C1 (fp16 m=1024 n=256): microseconds per launch, warm (CUDA graph) and cold (L2 flushed); "
                         "c2 = BASELINE config C2 (bf16 n=128, m=2^20: Llama-3 8B Q/K head_dim rotation); c4 = "
                         "BASELINE config C4 (fp16 n=4096, m=16384: QuaRot Llama-2 7B online rotation), L2 scrubbed "
                         "before every launch")
    return ap.parse_args()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def measured_hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str = "fwht"):
    """Per-launch DRAM bytes from the committed ncu --set full capture of this workload's
    launches (profiles/ncu_traffic.json for the C3 sweep, ncu_traffic_<workload>.json for
    the others), if present."""
    name = "ncu_traffic.json" if workload == "fwht" else f"ncu_traffic_{workload}.json"
    p = os.path.join(ROOT, "profiles", name)
    try:
        return json.load(open(p))
    except Exception:
        return None


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled while the timed region runs: NVML
    polled every ~2 ms from a thread (a 3 ms step still gets samples), falling back to
    `nvidia-smi -lms 20` when NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (time, sm_mhz, sm_max_mhz, reasons)
        self.proc = None
        self.stop = threading.Event()
        self.t0 = self.t1 = None
        self.source = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.physical_index())
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((time.time(), float(sm), float(smax),
                                          {nm for nm, b in bits.items() if r & b}))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.reader = threading.Thread(target=poll, daemon=True)
            self.reader.start()
            self.source = "NVML, 2 ms polling"
            time.sleep(0.05)
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "20", "-i", str(self.physical_index())], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.reader = threading.Thread(target=self._read, daemon=True)
            self.reader.start()
            self.source = "nvidia-smi -lms 20"
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def physical_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[self.index])
            except (ValueError, IndexError):
                pass
        return self.index

    def _read(self):
        for line in self.proc.stdout:
            f = [v.strip() for v in line.strip().split(",")]
            try:
                self.rows.append((time.time(), float(f[0]), float(f[1]),
                                  {nm for nm, v in zip(self.NAMES, f[4:8]) if v.lower() == "active"}))
            except Exception:
                continue

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        inside = [r for r in self.rows if self.t0 is not None and self.t0 <= r[0] <= (self.t1 or r[0])]
        use = inside if inside else self.rows
        sm = [r[1] for r in use]
        reasons = set().union(*[r[3] for r in use])
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[2] for r in use),
                "reasons": sorted(reasons), "samples": len(use), "samples_in_timed_region": len(inside),
                "source": self.source}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL communicator INIT lines (nranks, transports) in the log, so a scaling run
        # shows which communicator the ranks formed
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        ndev = torch.cuda.device_count()
        dev = local % ndev
        torch.cuda.set_device(dev)
        if ndev >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:  # more ranks than GPUs (code-path check only): NCCL forbids sharing a GPU
            dist.init_process_group("gloo")
        return rank, world, dev, dist
    torch.cuda.set_device(0)
    return 0, 1, 0, None


def barrier(dist, torch):
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(v: float, dist, torch):
    if dist is None:
        return v
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_oracle_sample(inputs, sample_elems, threads):
    """Time the fp64 oracle on the first rows of each (dtype, n) input: returns
    (seconds, elements)."""
    import numpy as np
    import oracle
    tot_t, tot_e = 0.0, 0
    for (dt, n), x in inputs.items():
        rows = max(1, sample_elems // n)
        xs = x[:rows]
        a = xs.cpu().double().numpy() if hasattr(xs, "cpu") else xs
        a = np.ascontiguousarray(a)
        t0 = time.perf_counter()
        oracle.fwht(a, threads=threads)
        tot_t += time.perf_counter() - t0
        tot_e += a.size
    return tot_t, tot_e


def reference_arm(args, rank, world):
    """--impl reference: the fp64 CPU oracle (as it stands) on host cores, rank 0 only."""
    if rank != 0:
        return None
    import torch
    import oracle
    import synthetic
    oracle.build()
    threads = oracle.default_threads()
    sample = 1 << 22  # elements per (dtype, n) per step; bounded so K+W steps finish in minutes
    inputs = {}
    for dt in (torch.float16, torch.bfloat16):
        for n in NS:
            m = sample // n
            inputs[(str(dt), n)] = synthetic.generate(m, n, dt, synthetic.seed_for(2, dt)).double().numpy()
    for _ in range(args.warmup):
        run_oracle_sample(inputs, sample, threads)
    t_all, e_all = 0.0, 0
    for _ in range(args.steps):
        t, e = run_oracle_sample(inputs, sample, threads)
        t_all += t
        e_all += e
    gbs = 4.0 * e_all / t_all / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t_all / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (oracle)",
        "data": "synthetic", "config": config_block(args, world),
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{sample} elements per (dtype, n) per step = {sample // (1 << 20)}Mi of the "
                                   f"{args.elems >> 20}Mi-element C3 matrices, 18 (dtype, n) pairs; fp64 "
                                   "listing (oracle/fwht_oracle.c), widening excluded"},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


def config_block(args, world):
    wl = ("C3 size sweep: n=2^7..2^15 x {fp16, bf16}, 2^28 elements per (n, dtype) per GPU, "
          "out-of-place, normalized (scale=1/sqrt(n))")
    ns = SMALL_NS if getattr(args, "workload", "fwht") == "small" else NS
    if getattr(args, "workload", "fwht") == "f32":
        ns = SMALL_NS + NS
        wl = ("NEXT-2 fp32 path: n=2^1..2^15 fp32, 2^28 elements (1 GiB in, 1 GiB out) per n per GPU, "
              "out-of-place, normalized (scale=1/sqrt(n))")
    if getattr(args, "workload", "fwht") == "c5":
        ns = [32768]
        wl = ("C5: bf16 n=2^15, 2^33 elements (262144 rows, 16 GiB in + 16 GiB out) row-sharded across the "
              "ranks, no collective on the hot path, out-of-place, normalized")
    if getattr(args, "ns", None):
        ns = [int(v) for v in args.ns.split(",")]
        wl = f"{getattr(args, 'workload', 'fwht')} over n in {ns} (--ns), 2^28 elements per (n, dtype) per GPU"
    if getattr(args, "workload", "fwht") == "small" and not getattr(args, "ns", None):
        wl = ("NEXT-2 small sizes: n=2^1..2^6 x {fp16, bf16}, 2^28 elements per (n, dtype) per GPU, "
              "out-of-place, normalized (scale=1/sqrt(n))")
    w = getattr(args, "workload", "fwht")
    if w.startswith("quant-") and not getattr(args, "ns", None):
        wl = (f"NEXT-1 fused FWHT + per-row {w[6:].upper()} quantization: n=2^7..2^15 x {{fp16, bf16}}, 2^28 "
              "elements per (n, dtype) per GPU, codes + fp32 row scales out, normalized (scale=1/sqrt(n))")
    nrange = f"n in {ns}" if getattr(args, "ns", None) else "n=2^7..2^15"
    if w == "qk-rotate":
        wl = (f"QK rotation: {nrange} x {{fp16, bf16}}; a 2^28-element QKV buffer viewed as [T, 3, H, n], "
              "H = max(1, 4096/n); the Q and K heads (2/3 of it) transformed in place, normalized")
    if w == "qk-quant":
        wl = (f"QK rotation + FP8-E4M3 quantization: {nrange} x {{fp16, bf16}}; a 2^28-element QKV buffer viewed "
              "as [T, 3, H, n], H = max(1, 4096/n); the Q and K heads read strided, codes and row scales written "
              "contiguously (hadacore_fwht_quant_strided), normalized")
    if w == "c2":
        ns = [128]
        wl = ("C2: Llama-3 8B FP8-attention Q/K rotation, bf16 n=128 (head_dim), m=8x32x4096=2^20 rows per GPU, "
              "normalized")
    if w == "c4":
        ns = [4096]
        wl = "C4: QuaRot Llama-2 7B online rotation, fp16 n=4096, m=16384 tokens per GPU, normalized"
    if getattr(args, "inplace", False):
        wl = wl.replace("out-of-place", "in place (out = in, P:264-274)")
        if "in place" not in wl:
            wl += "; in place (out = in, P:264-274)"
    elif w in ("c2", "c4"):
        wl += "; out-of-place"
    mib_in = args.elems * (4 if w == "f32" else 2) >> 20
    if w == "c5":
        l2 = "no flush: each rank's launch reads 16/N GiB and writes 16/N GiB (> 126 MB L2)"
    elif w == "c4":
        l2 = ("flushed: a 2 x L2-size buffer is written before every timed launch, outside its CUDA events "
              f"(each launch reads {mib_in} MiB and writes {mib_in} MiB, about the size of the 126 MB L2); value = "
              "bytes / sum of the per-launch event times")
    elif w in ("qk-rotate", "qk-quant"):
        l2 = (f"no flush: every launch reads the {mib_in * 2 // 3} MiB of Q and K heads (> 126 MB L2) and writes "
              + ("them back in place" if w == "qk-rotate" else f"{args.elems * 2 // 3 >> 20} MiB of codes"))
    elif w.startswith("quant-"):
        codes = args.elems // (2 if w == "quant-int4" else 1) >> 20
        l2 = f"no flush: every launch reads a {mib_in} MiB input and writes {codes} MiB of codes (> 126 MB L2)"
    else:
        l2 = f"no flush: every launch reads a {mib_in} MiB input and writes a {mib_in} MiB output (> 126 MB L2)"
    return {"workload": wl,
            "elements_per_launch": args.elems, "ns": ns,
            "dtypes": {"f32": ["fp32"], "c5": ["bf16"], "c2": ["bf16"], "c4": ["fp16"]}.get(w, ["fp16", "bf16"]),
            "launches_per_step": (1 if w in ("f32", "c5", "c2", "c4") else 2) * len(ns), "path": w,
            "inplace": bool(getattr(args, "inplace", False)),
            "l2": l2,
            "parallelism": f"row-sharded x{world}, no collective on the hot path" if world > 1 else "single GPU"}


def run_c1(args, rank, world, dist):
    """BASELINE configs[0] (C1: fp16, m = 1024, n = 256, 1 MiB of traffic): a launch-latency-bound,
    L2-resident problem, reported in microseconds per launch -- warm (100 launches captured in one CUDA
    graph, replayed) and cold (L2 flushed by a 2 x 126 MB write before each timed launch)."""
    import torch
    import paper_2412_08832_b200 as hc
    import synthetic
    hc._load()
    dev = torch.device("cuda", torch.cuda.current_device())
    x = synthetic.generate(1024, 256, torch.float16, synthetic.seed_for(0, torch.float16)).to(dev)
    y = torch.empty_like(x)
    stream = torch.cuda.Stream(dev)
    R = 100
    with torch.cuda.stream(stream):
        for _ in range(3):
            hc.hadacore_fwht(x, out=y, stream=stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(R):
                hc.hadacore_fwht(x, out=y, stream=stream)
        for _ in range(args.warmup):
            g.replay()
        barrier(dist, torch)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # at least ~0.5 s of replays so nvidia-smi samples the timed region (20 ms period)
        reps = max(args.steps, 3000)
        with ClockSampler(torch.cuda.current_device()) as cs:
            cs.mark_start()
            e0.record(stream)
            for _ in range(reps):
                g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            cs.mark_end()
        clocks = cs.summary()
        warm_us = max_over_ranks(e0.elapsed_time(e1) * 1e3 / (reps * R), dist, torch)
        flush = torch.empty(2 * 126 * 1000 * 1000, dtype=torch.uint8, device=dev)
        cold = []
        for _ in range(max(3, args.steps)):
            flush.fill_(1)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            hc.hadacore_fwht(x, out=y, stream=stream)
            c1.record(stream)
            torch.cuda.synchronize()
            cold.append(c0.elapsed_time(c1) * 1e3)
    cold_us = sorted(cold)[len(cold) // 2]
    bytes_ = 4.0 * x.numel()
    if rank != 0:
        return None
    return {"metric": "C1 latency: microseconds per hadacore_fwht launch, fp16 m=1024 n=256 (warm, CUDA graph)",
            "value": round(warm_us, 3), "unit": "us", "n_gpus": world, "steps": reps, "warmup": args.warmup,
            "ms_per_step": round(warm_us * R / 1e3, 4), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp16 (fp32 last-stage accumulate)", "data": "synthetic (synthetic/)",
            "config": {"workload": "C1: fp16 m=1024 n=256 (1 MiB traffic), 100 launches per CUDA graph replay; "
                                   "cold = one launch after a 252 MB L2-flushing write", "l2": "warm: L2-resident by "
                                   "design (C1 is launch-bound); cold: flushed", "parallelism": "single GPU"},
            "cold_us": round(cold_us, 3), "warm_GBps": round(bytes_ / (warm_us * 1e-6) / 1e9, 1),
            "roofline": {"bound": "hbm", "achieved": round(bytes_ / (cold_us * 1e-6) / 1e9, 1),
                         "peak": measured_hbm_peak()[0], "unit": "GB/s",
                         "frac": round(bytes_ / (cold_us * 1e-6) / 1e9 / measured_hbm_peak()[0], 4),
                         "traffic": None, "note": "1 MiB per launch: launch-latency-bound, not bandwidth-bound; "
                                                  "achieved from the cold launch time"},
            "gpu_launches": int(reps * R), "cpu_baseline": None, "e2e": None, "clocks": clocks,
            "graph_replays": reps}


def run_lab(args, rank, world):
    """NEXT-4 quantization lab (SPEC quant_lab): rotated vs plain per-row INT4 error on the SPEC's
    default outlier matrices (64 x 1024, rate 1e-3 x 100 sigma), 100 trials -- every step on the GPU
    (hadacore_fwht fp32 rotations, hadacore_fake_quant, hadacore_row_sq_error)."""
    import torch
    from paper_2412_08832_b200 import quant_lab
    spec = quant_lab.OutlierSpec(rows=64, cols=1024, outlier_rate=1e-3, outlier_scale=100.0, seed=1 + rank)
    for _ in range(max(1, args.warmup)):
        quant_lab.run_experiment(spec, "int4", "row", trials=5)
    torch.cuda.synchronize()
    rep = quant_lab.run_experiment(spec, "int4", "row", trials=100)
    a = rep["aggregate"]
    if rank != 0:
        return None
    return {"metric": "INT4 per-row quantization MSE, rotated / plain (SPEC quant_lab outlier matrices, 100 trials)",
            "value": round(a["mse_rotated"] / a["mse_plain"], 4), "unit": "ratio", "n_gpus": world, "steps": 100,
            "warmup": args.warmup, "ms_per_step": round(1e3 * rep["seconds"] / 100, 3), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32 rotations, INT4 codes", "data": "synthetic OutlierSpec",
            "config": {"workload": "NEXT-4 lab: 64 x 1024 fp32, outlier rate 1e-3, scale 100, INT4 per row"},
            "win_rate": a["win_rate"], "mse_plain": a["mse_plain"], "mse_rotated": a["mse_rotated"],
            "max_abs_plain": a["max_abs_plain"], "max_abs_rotated": a["max_abs_rotated"],
            "roofline": None, "cpu_baseline": None, "e2e": None, "gpu_launches": None}


# ---------------------------------------------------------------- resident inputs and the sampled check
# Every workload's data is a slice of one global seeded matrix generated at a base width W
# (synthetic/ keys its generator on the global element index): rank r's
# resident buffer holds global elements [flat0_r, flat0_r + elems), and the row of width n
# at local index i is global row flat0_r / n + i.  So any rank -- and rank 0 when it checks
# the others -- can regenerate any global row without communication.
WORKLOADS = {
    # workload: (config index for the seed, base width W, dtypes, ns)
    "fwht": (2, 256, ("fp16", "bf16"), NS),
    "small": (2, 256, ("fp16", "bf16"), SMALL_NS),
    "f32": (2, 256, ("fp32",), SMALL_NS + NS),
    "c2": (1, 128, ("bf16",), [128]),
    "c4": (3, 4096, ("fp16",), [4096]),
    "c5": (5, 32768, ("bf16",), [32768]),
}
C2_ROWS, C4_ROWS, C5_ROWS = 8 * 32 * 4096, 16384, C5_ELEMS // 32768


def torch_dtype(name):
    import torch
    return {"fp16": torch.float16, "bf16": torch.bfloat16, "fp32": torch.float32}[name]


def dtype_name(dt):
    import torch
    return {torch.float16: "fp16", torch.bfloat16: "bf16", torch.float32: "fp32"}[dt]


def seed_of(workload, dt):
    import synthetic
    idx = WORKLOADS.get(workload, WORKLOADS["fwht"])[0]  # C5: 5, the parity tests' seed
    return synthetic.seed_for(idx, dt)


def gen_rows(workload, dt, n, g0, count, device, shift_elems=0):
    """Rows [g0, g0 + count) of width n of the workload's global matrix (fresh from synthetic/)."""
    import synthetic
    w = WORKLOADS.get(workload, WORKLOADS["fwht"])[1]
    start = g0 * n + shift_elems
    end = start + count * n
    r0, r1 = start // w, -(-end // w)
    blk = synthetic.generate(r1 - r0, w, dt, seed_of(workload, dt), row0=r0, device=device).view(-1)
    return blk[start - r0 * w: end - r0 * w].view(count, n)


def rank_layout(workload, rank, world, elems):
    """(flat0, elems) of this rank's slice of the global matrix, and the global element count."""
    from paper_2412_08832_b200.shard import row_range
    if workload == "c5":
        lo, hi = row_range(C5_ROWS, rank, world)
        return lo * 32768, (hi - lo) * 32768, C5_ELEMS
    if workload == "c2":
        return rank * C2_ROWS * 128, C2_ROWS * 128, world * C2_ROWS * 128
    if workload == "c4":
        return rank * C4_ROWS * 4096, C4_ROWS * 4096, world * C4_ROWS * 4096
    return rank * elems, elems, world * elems


def fill_resident(buf, workload, dt, flat0, shift_elems=0):
    """buf (1-D, numel multiple of W) <- global elements [flat0, flat0 + numel) (+ shift)."""
    import synthetic
    w = WORKLOADS.get(workload, WORKLOADS["fwht"])[1]
    start = flat0 + shift_elems
    assert start % w == 0 and buf.numel() % w == 0
    synthetic.generate(buf.numel() // w, w, dt, seed_of(workload, dt), row0=start // w, out=buf.view(-1, w))


def sample_local_rows(n, dt, rank, m_loc, k):
    """The local row indices rank `rank` contributes to the check: its first and last row and
    k - 2 seeded random rows (the same list on every rank, so rank 0 can rebuild it)."""
    import torch
    g = torch.Generator().manual_seed(1000003 * n + 7919 * rank + (17 if dt == torch.bfloat16 else 0) +
                                      (29 if dt == torch.float32 else 0))
    extra = torch.randint(0, m_loc, (max(0, k - 2),), generator=g).tolist() if m_loc > 0 else []
    return ([0, m_loc - 1] + extra)[:max(k, 1)]


def gather_sample(y, n, dt, rank, world, k, dist):
    """This rank's sampled output rows (sample_local_rows) gathered to rank 0 with
    shard.gather_rows (NCCL; CPU tensors over gloo): [k * world, n] on rank 0, None elsewhere."""
    from paper_2412_08832_b200.shard import gather_rows
    loc = y[sample_local_rows(n, dt, rank, y.shape[0], k)].contiguous()
    if dist is None:
        return loc
    if dist.get_backend() != "nccl":
        loc = loc.cpu()
    return gather_rows(loc, k * world, dist)


def sampled_rows_check(results, workload, world, elems, k, dist, transform, device):
    """Rank 0's half of the multi-rank result check (north_star "NCCL only to
    gather results for checking").  `results[(dt, n)]` is the [k * world, n] block gathered from
    every rank (rank order; rank r's rows are sample_local_rows(...)).  Each row is compared with
    (a) the fp64 oracle on the regenerated global input (north_star tolerances) and (b) bitwise
    with rank 0's own transform of the same global rows (a 16-row aligned block regenerated on
    rank 0's GPU): sharding invariance, ambiguity 17."""
    import numpy as np
    import torch
    import oracle
    tol = {"fp16": 2e-3, "bf16": 1.6e-2, "fp32": 1e-5}
    dev = device
    worst, mism, checked, bad_rows = {}, 0, 0, []
    for (dt, n), got in results.items():
        got = got.to("cpu")
        rows_global = []
        for r in range(world):
            flat0, el, total = rank_layout(workload, r, world, elems)
            m_loc = el // n
            rows_global += [flat0 // n + i for i in sample_local_rows(n, dt, r, m_loc, k)]
        m_global = total // n
        x = torch.cat([gen_rows(workload, dt, n, g, 1, "cpu") for g in rows_global])
        ref = oracle.fwht(x.double().numpy())
        g64 = got.double().numpy()
        err = np.linalg.norm(g64 - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-300)
        name = dtype_name(dt)
        worst[name] = max(worst.get(name, 0.0), float(err.max()))
        for j, g in enumerate(rows_global):
            b = min(g - g % 16, max(0, m_global - 16))
            cnt = min(16, m_global - b)
            y = transform(gen_rows(workload, dt, n, b, cnt, dev))
            iv = torch.int32 if dt == torch.float32 else torch.int16
            same = torch.equal(y[g - b].cpu().view(iv), got[j].view(iv))
            checked += 1
            if not same or err[j] > tol[name]:
                mism += int(not same)
                if len(bad_rows) < 8:
                    bad_rows.append({"dtype": name, "n": n, "row": int(g), "rel_err": float(f"{err[j]:.3e}"),
                                     "bitwise_equal": bool(same)})
    ok_oracle = all(worst[nm] <= tol[nm] for nm in worst)
    return {"ranks": world, "rows_per_rank_per_launch": k, "rows_checked": checked,
            "gather": ("NCCL" if dist is not None and dist.get_backend() == "nccl" else
                       ("gloo" if dist is not None else "none (1 rank)")) + " gather of sampled output rows to rank 0",
            "oracle_max_rel_err": {nm: float(f"{v:.3e}") for nm, v in worst.items()},
            "tolerance": {nm: tol[nm] for nm in worst}, "oracle_pass": ok_oracle,
            "bitwise_mismatches_vs_rank0_recompute": mism, "bitwise_pass": mism == 0,
            "pass": ok_oracle and mism == 0, "failing_rows": bad_rows}


def main():
    args = parse()
    if args.impl == "reference":
        # CPU oracle on host cores; under torchrun only rank 0 works, the others exit 0
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        line = reference_arm(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    import torch
    rank, world, local, dist = dist_setup(args)
    if args.workload in ("c1", "lab"):
        line = run_c1(args, rank, world, dist) if args.workload == "c1" else run_lab(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        if dist is not None:
            dist.destroy_process_group()
        return

    import paper_2412_08832_b200 as hc
    hc._load()  # fails loudly without the CUDA library
    dev = torch.device("cuda", local)
    wl = args.workload
    src_wl = wl if wl in WORKLOADS else "fwht"  # quant-* / qk-*: the C3 matrices
    c5, f32, scrub = wl == "c5", wl == "f32", wl == "c4"
    flat0, args.elems, _ = rank_layout(src_wl, rank, world, args.elems)
    # negative control (--misshard): the last rank (rank 0 at N = 1) generates its slice one
    # base row off, so its outputs belong to other global rows than it reports
    shift = WORKLOADS[src_wl][1] if (args.misshard and rank == world - 1) else 0
    dtypes = [torch_dtype(d) for d in WORKLOADS[src_wl][2]]
    xin = {}
    for dt in dtypes:
        xin[dt] = torch.empty(args.elems, dtype=dt, device=dev)
        fill_resident(xin[dt], src_wl, dt, flat0, shift)
    obuf = torch.empty(args.elems, dtype=torch.float32 if f32 else torch.float16, device=dev)
    stream = torch.cuda.current_stream(dev)
    ns = list(WORKLOADS[src_wl][3])
    if args.ns:
        ns = [int(v) for v in args.ns.split(",")]
    pairs = [(dt, n) for dt in dtypes for n in ns]
    quant = wl.startswith("quant")
    qtype = wl.split("-")[1] if quant else None
    if quant:
        qbuf = torch.empty(args.elems // (2 if qtype == "int4" else 1), dtype=hc.QTYPES[qtype][1], device=dev)
        sbuf = torch.empty(args.elems // min(ns), dtype=torch.float32, device=dev)
    qb = 0.5 if qtype == "int4" else 1.0  # code bytes per element

    rotate = wl in ("qk-rotate", "qk-quant")
    qkq = wl == "qk-quant"  # Q/K heads rotated + FP8-quantized in one pass (FP8 attention)
    if qkq:
        qbuf = torch.empty(args.elems, dtype=torch.float8_e4m3fn, device=dev)
        sbuf = torch.empty(args.elems // min(ns), dtype=torch.float32, device=dev)
    qk = {}
    if rotate:
        # fused QKV activations [T, 3, H, n] (H = max(1, 4096 / n) heads); the Q and K
        # heads are rotated in place through the strided entry (2 row dims: T x 2H)
        for dt in xin:
            for n in ns:
                h = max(1, 4096 // n)
                t = args.elems // (3 * h * n)
                qk[(dt, n)] = xin[dt][: t * 3 * h * n].view(t, 3, h, n)[:, 0:2]
    elems_of = {(dt, n): (qk[(dt, n)].numel() if rotate else args.elems) for dt, n in pairs}

    def out_view(dt, n):
        return obuf.view(-1, n) if f32 else obuf.view(torch.int16).view(dt).view(-1, n)

    def launch(dt, n):
        if rotate:
            v = qk[(dt, n)]
            if qkq:
                hc.hadacore_fwht_quant_strided(v, qtype="e4m3", out=qbuf[: v.numel()], row_scale=sbuf[: v.numel() // n],
                                               stream=stream)
            else:
                hc.hadacore_fwht_strided(v, out=v, stream=stream)
            return
        x = xin[dt].view(-1, n)
        if quant:
            hc.hadacore_fwht_quant(x, qtype=qtype, out=qbuf.view(-1, n // 2 if qtype == "int4" else n),
                                   row_scale=sbuf[: x.shape[0]],
                                   stream=stream)
            return
        hc.hadacore_fwht(x, out=x if args.inplace else out_view(dt, n), stream=stream)

    # C4 (about the L2's size): a 2 x L2 write before every timed launch, outside its events
    l2_bytes = getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 * 1000 * 1000) or 126000000
    scrub_buf = torch.empty(2 * l2_bytes, dtype=torch.uint8, device=dev) if scrub else None

    # warm-up
    for _ in range(args.warmup):
        for dt, n in pairs:
            if scrub:
                scrub_buf.fill_(1)
            launch(dt, n)
    barrier(dist, torch)

    def timed_region(steps, per_launch_events):
        # The timed region has no events between launches: an event record between two
        # kernels breaks programmatic dependent launch (the next grid's prologue and
        # first loads no longer overlap the previous grid's tail), which measured -5 %
        # on the sweep (tools/gap_probe.py, profiles/r01_gap_probe.txt). The per-(dtype,
        # n) breakdown comes from a separate pass with per-launch events.  With an L2
        # scrub (C4) every launch has its own events and the region's time is their sum.
        ple = per_launch_events or scrub
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps * len(pairs) if ple else 0)]
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(dist, torch)
        torch.cuda.synchronize()
        g0.record(stream)
        i = 0
        for _ in range(steps):
            for dt, n in pairs:
                if scrub:
                    scrub_buf.fill_(1)
                if ple:
                    evs[i][0].record(stream)
                launch(dt, n)
                if ple:
                    evs[i][1].record(stream)
                i += 1
        g1.record(stream)
        torch.cuda.synchronize()
        per = [a.elapsed_time(b) for a, b in evs]
        total_ms = sum(per) if scrub else g0.elapsed_time(g1)
        barrier(dist, torch)
        return total_ms, per

    with ClockSampler(torch.cuda.current_device() if world == 1 else local) as cs:
        cs.mark_start()
        total_ms, _ = timed_region(args.steps, False)
        cs.mark_end()
    clocks = cs.summary()
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    remeasured = False
    if bad & set(clocks.get("reasons", [])):
        with ClockSampler(local) as cs:
            cs.mark_start()
            total_ms, _ = timed_region(args.steps, False)
            cs.mark_end()
        clocks = cs.summary()
        remeasured = True
    # per-launch breakdown: a separate pass after the timed region
    _, per = timed_region(max(3, min(args.steps, 10)), True)
    # per-(dtype, n) rate: back-to-back launches of one (dtype, n) between two events (the
    # per-launch events above break programmatic dependent launch, so they understate a
    # kernel's rate inside a run of launches, most for the shortest launches)
    per_pair_ms = {}
    per_pair_clocks = None
    if not scrub:
        reps = max(3, min(args.steps, 20))
        cs_pp = ClockSampler(torch.cuda.current_device() if world == 1 else local)
        cs_pp.__enter__()
        cs_pp.mark_start()
        for dt, n in pairs:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            launch(dt, n)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(reps):
                launch(dt, n)
            e1.record(stream)
            torch.cuda.synchronize()
            per_pair_ms[(dt, n)] = e0.elapsed_time(e1) / reps
        cs_pp.mark_end()
        cs_pp.__exit__(None, None, None)
        per_pair_clocks = cs_pp.summary()

    # output checks outside the timed regions, on every rank:
    # (1) a property that holds at any size: the normalized transform preserves
    #     every row's norm -- every row of every (dtype, n) launch, max over ranks;
    # (2) sampled rows: every rank's first, last and k-2 random rows of every launch are gathered
    #     to rank 0 (NCCL; gloo when ranks share a GPU) and checked there against the fp64 oracle
    #     and bitwise against rank 0's own transform of the same global rows.
    # In-place runs regenerate the input first (the timed launches transformed it repeatedly).
    check = None
    if not quant and not rotate:
        worst, by_dt = 0.0, {}
        tol_of = {torch.float16: 2e-3, torch.bfloat16: 1.6e-2, torch.float32: 1e-5}
        gathered = {}
        for dt, n in pairs:
            if args.inplace:
                fill_resident(xin[dt], src_wl, dt, flat0, shift)
                xcopy = out_view(dt, n)
                xcopy.view(-1).copy_(xin[dt])
            launch(dt, n)
            x = (xcopy if args.inplace else xin[dt].view(-1, n))
            y = (xin[dt].view(-1, n) if args.inplace else out_view(dt, n))[: x.shape[0]]
            for r0 in range(0, x.shape[0], max(1, (1 << 26) // n)):
                nx = torch.linalg.vector_norm(x[r0:r0 + (1 << 26) // n].float(), dim=1)
                ny = torch.linalg.vector_norm(y[r0:r0 + (1 << 26) // n].float(), dim=1)
                e = ((ny - nx).abs() / nx.clamp_min(1e-30)).max().item()
                by_dt[dt] = max(by_dt.get(dt, 0.0), e)
            gathered[(dt, n)] = gather_sample(y, n, dt, rank, world, args.check_rows, dist)
        errs = {dtype_name(dt): float(f"{max_over_ranks(e, dist, torch):.3e}") for dt, e in by_dt.items()}
        check = {"property": "row-norm preservation of the normalized transform, every row of every launch "
                             "(north_star tolerances per dtype)" + ("; input regenerated, one in-place launch"
                                                                    if args.inplace else ""),
                 "max_rel_err": errs, "tolerance": {dtype_name(dt): tol_of[dt] for dt in by_dt}}
        check["norm_pass"] = all(errs[dtype_name(dt)] <= tol_of[dt] for dt in by_dt)
        if rank == 0:
            mr = sampled_rows_check(gathered, src_wl, world, args.elems, args.check_rows, dist, hc.hadacore_fwht, dev)
            check["multi_rank"] = mr
        ok = torch.tensor([1.0 if (rank != 0 or check["multi_rank"]["pass"]) else 0.0], dtype=torch.float64)
        if dist is not None:
            okd = ok.to(dev) if dist.get_backend() == "nccl" else ok
            dist.broadcast(okd, src=0)
            ok = okd.cpu()
        check["pass"] = bool(check["norm_pass"] and ok.item() == 1.0)

    # same-run D2D copy of the same byte count ("% of achievable copy"): cudaMemcpyAsync
    # of one input buffer into the output buffer, event-timed on the same stream
    src_b = next(iter(xin.values())).view(torch.uint8)
    dst_b = obuf.view(torch.uint8)[: src_b.numel()]
    for _ in range(3):
        dst_b.copy_(src_b)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    c0.record(stream)
    for _ in range(10):
        dst_b.copy_(src_b)
    c1.record(stream)
    torch.cuda.synchronize()
    copy_gbps = 2.0 * src_b.numel() * 10 / (c0.elapsed_time(c1) * 1e-3) / 1e9

    t_max = max_over_ranks(total_ms, dist, torch)
    # algorithmic bytes: 2 B read + 2 B written per element (fwht); 2 + 1 B plus one fp32
    # scale per row for the fused quantization (per-n average over the sweep)
    esize = 4 if f32 else 2
    bytes_per_launch = 2.0 * esize * args.elems if not quant else \
        sum((2.0 + qb) * args.elems + 4.0 * (args.elems // n) for n in ns) / len(ns)
    if rotate:
        bytes_per_launch = sum(4.0 * e for e in elems_of.values()) / len(pairs)
    if qkq:  # 2 B read + 1 B code per element + a 4-byte scale per row
        bytes_per_launch = sum(3.0 * e + 4.0 * e / n for (dt, n), e in elems_of.items()) / len(pairs)
    total_bytes = bytes_per_launch * len(pairs) * args.steps * world
    if c5:  # strong scaling: the whole 2^33-element job per step, whatever the rank count
        total_bytes = 4.0 * C5_ELEMS * args.steps
    value = total_bytes / (t_max * 1e-3) / 1e9

    # per-launch device times of the per-launch pass: p10 / p50 / p90
    srt = sorted(per)
    launch_pct = [round(1e3 * srt[int(q * (len(srt) - 1))], 2) for q in (0.1, 0.5, 0.9)] if srt else None

    # per-(dtype, n) breakdown and the roofline of the kernel (device time per launch)
    per_n = {}
    for k, (dt, n) in enumerate(pairs):
        ts = sorted(per[k::len(pairs)])
        med = per_pair_ms.get((dt, n), ts[len(ts) // 2])
        b_n = 2.0 * esize * elems_of[(dt, n)] if not quant else (2.0 + qb) * args.elems + 4.0 * (args.elems // n)
        if qkq:
            b_n = 3.0 * elems_of[(dt, n)] + 4.0 * elems_of[(dt, n)] / n
        per_n.setdefault(dtype_name(dt), {})[str(n)] = round(b_n / (med * 1e-3) / 1e9, 1)
    # roofline over the timed region: every launch of the step is the same transform
    # (one per (dtype, n)), so the kernel's average launch duration is the region time
    # over the launches in it (per-(dtype, n) values: per_n_GBps)
    avg_launch_ms = t_max / (args.steps * len(pairs))
    peak, peak_src = measured_hbm_peak()
    achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
    traffic = ncu_traffic(wl)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_source": peak_src,
                "frac_of_8TBps": round(achieved / NOMINAL_HBM_GBS, 4),
                "algorithmic_bytes_per_launch": int(bytes_per_launch),
                "traffic": (traffic or {}).get("avg_dram_bytes_per_launch"),
                "traffic_source": (traffic or {}).get("source"),
                "duration_source": ("sum of per-launch CUDA events (L2 scrubbed between launches)" if scrub else
                                    "timed region / launches (CUDA events on the launching stream, max over ranks)"),
                "sum_of_launch_events_GBps": round(bytes_per_launch * len(per) / (sum(per) * 1e-3) / 1e9, 1),
                "same_run_d2d_copy_GBps": round(copy_gbps, 1),
                "frac_of_same_run_copy": round(achieved / copy_gbps, 4),
                "note": "back-to-back PDL launches overlap one grid's tail with the next grid's ramp; the peak is a "
                        "single timed 2 GiB copy, which includes its own ramp and tail, so frac can exceed 1"}

    # end to end through the public host-buffer C entry (hadacore_fwht_host)
    e2e = None
    if not args.no_e2e and wl in ("fwht", "c2", "c4"):
        hin = {dt: xin[dt].cpu().pin_memory() for dt in xin}
        hout = torch.empty(args.elems, dtype=torch.float16).pin_memory()
        ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        for dt, n in pairs[:2]:
            hc.hadacore_fwht_host(hin[dt].view(-1, n), out=hout.view(torch.int16).view(dt).view(-1, n), workspace=ws)
        barrier(dist, torch)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            for dt, n in pairs:
                hc.hadacore_fwht_host(hin[dt].view(-1, n), out=hout.view(torch.int16).view(dt).view(-1, n),
                                      workspace=ws)
        torch.cuda.synchronize()
        dt_s = time.perf_counter() - t0
        dt_s = max_over_ranks(dt_s, dist, torch)
        e2e = {"value": round(bytes_per_launch * len(pairs) * args.e2e_steps * world / dt_s / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": int(2 * args.elems * len(pairs)),
               "d2h_bytes_per_step": int(2 * args.elems * len(pairs)),
               "api": "hadacore_fwht_host (C ABI, pinned host buffers, copies + kernel pipelined in the library)",
               "ceiling": "PCIe-bound: pinned H2D + D2H running concurrently measured 93.9 GB/s on this pool "
                          "(tools/pcie_probe.py, profiles/r01_quant_bound_diag.txt)",
               "steps": args.e2e_steps}
        del hin, hout, ws

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and wl in ("fwht", "c2", "c4", "c5"):
        import oracle
        oracle.build()
        threads = oracle.default_threads()
        import numpy as np
        sample = 1 << 24
        # widened once (fp64), then whole passes over the samples until >= 10 s of oracle
        # time (bounded CPU work, the contract's 10-30 s)
        inputs = {(str(dt), n): np.ascontiguousarray(xin[dt][: (sample // n) * n].view(-1, n).cpu().double().numpy())
                  for dt, n in pairs}
        t, e, passes = 0.0, 0, 0
        while t < 10.0 and passes < 200:
            dt_, de = run_oracle_sample(inputs, sample, threads)
            t, e, passes = t + dt_, e + de, passes + 1
        del inputs
        cpu_baseline = {"value": round(4.0 * e / t / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
                        "cpu_model": cpu_model(), "gel_per_s": round(e / t / 1e9, 4),
                        "sample": f"first {sample >> 20}Mi elements of each of the {len(pairs)} (dtype, n) inputs, "
                                  f"{passes} passes ({e} elements), fp64 listing, {t:.1f} s; widening excluded"}

    if rank == 0:
        metric = METRIC if not quant else (f"Fused FWHT + per-row {qtype.upper()} quantization HBM GB/s vs "
                                           "n=2^7..2^15 (bf16/fp16 in, " + ("4" if qtype == "int4" else "8") +
                                           "-bit codes + fp32 row scales out)")
        if f32:
            metric = "FWHT HBM GB/s vs n=2^1..2^15, fp32 path (NEXT-2; north_star's fp32 path, tolerance 1e-5)"
        if c5:
            metric = ("C5: FWHT HBM GB/s, bf16 n=2^15, 2^33 elements row-sharded across the GPUs "
                      "(whole-job bytes / max-over-ranks time; strong scaling)")
        if wl == "c2":
            metric = "C2: FWHT HBM GB/s, bf16 n=128, m=2^20 rows per GPU (Llama-3 8B Q/K head_dim rotation)"
        if wl == "c4":
            metric = ("C4: FWHT HBM GB/s, fp16 n=4096, m=16384 rows per GPU (QuaRot Llama-2 7B online rotation), "
                      "L2 scrubbed before every launch")
        if wl == "small":
            metric = "FWHT HBM GB/s vs n=2^1..2^6 (bf16/fp16), rows shorter than the paper's 2^7 (NEXT-2)"
        if qkq:
            metric = ("FWHT + FP8-E4M3 quantization of the Q and K heads of fused QKV activations [T, 3, H, n] "
                      "(strided rows, codes + fp32 scales out) HBM GB/s vs n=2^7..2^15")
        elif rotate:
            metric = ("In-place FWHT of the Q and K heads of fused QKV activations [T, 3, H, n] (strided rows) "
                      "HBM GB/s vs n=2^7..2^15")
        if args.ns:
            metric = metric.replace("n=2^7..2^15", f"n in {{{args.ns}}}")
        if args.inplace and not rotate:
            metric += " [in place]"
        line = {
            "metric": metric, "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t_max / args.steps, 4), "higher_is_better": True,
            "scaling": "strong" if c5 else "weak", "vs_baseline": None,
            "dtype": "fp32" if f32 else ("bf16 (fp32 last-stage accumulate)" if wl in ("c5", "c2") else
                                         "fp16 (fp32 last-stage accumulate)" if wl == "c4" else
                                         "fp16+bf16 (fp32 last-stage accumulate)"),
            "data": "synthetic (counter-based N(0,1), synthetic/)", "config": config_block(args, world),
            "pct_of_8TBps": round(100.0 * value / world / NOMINAL_HBM_GBS, 2),
            # north_star: "reported ... both as GB/s and elements/s" (whole job, all ranks)
            "elements_per_s": float(f"{(C5_ELEMS * args.steps if c5 else sum(elems_of[p] for p in pairs) * args.steps * world) / (t_max * 1e-3):.4g}"),
            "per_n_GBps": per_n,
            "per_n_source": ("sum of per-launch events (L2 scrubbed between launches)" if scrub else
                             "back-to-back launches of each (dtype, n), CUDA events around the group, after the "
                             "timed region (its clocks: per_n_clocks; long fused-quantization runs reach the power "
                             "cap there -- profiles/r02_quant_single_n.txt has single-n timed regions)"),
            "per_n_clocks": per_pair_clocks,
            "launch_us_p10_p50_p90": launch_pct, "inplace": bool(args.inplace),
            "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e,
            "gpu_launches": int(args.steps * sum(hc.launches_per_call(elems_of[(dt, n)] // n, n, dt) for dt, n in pairs)),
            "clocks": clocks, "remeasured_for_clocks": remeasured, "check": check,
        }
        if args.misshard:
            line["negative_control"] = "--misshard: rank %d generated its rows one base row off" % (world - 1)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    if check is not None and not check["pass"]:
        sys.exit(3)


if __name__ == "__main__":
    main()
