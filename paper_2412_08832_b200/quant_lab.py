"""Quantization-error lab on the GPU (SPEC quant_lab S:397-464).

The paper's motivating claim (P:24 [Sec. 1]; P:180 [Sec. 4.2]): a Hadamard rotation
spreads activation outliers over the row, so low-precision quantization of the
rotated row loses less.  This module reproduces it on controlled synthetic
activations (SPEC OutlierSpec) with the library's own kernels:

    x        = outlier matrix (fp32, on the GPU)
    plain    = fake_quant(x)                               (hadacore_fake_quant)
    rotated  = H fake_quant(H x)                           (hadacore_fwht, fp32 path,
                                                            normalized H is an involution)
    mse_*    = sum(row_sq_error(*, x)) / (m n)             (hadacore_row_sq_error, fp64)

per trial, with per-trial seeds derived from the spec's seed; the report holds the
per-trial values and the aggregate (means and the win rate of rotated over plain).

    python -m paper_2412_08832_b200.quant_lab --target int4 --trials 100 [--csv out.csv]
"""
from __future__ import annotations

import argparse
import csv
import dataclasses
import json
import sys
import time

import torch

from . import fake_quant, hadacore_fwht, row_sq_error


@dataclasses.dataclass(frozen=True)
class OutlierSpec:
    """Gaussian(0, base_std) bulk, an outlier_rate fraction at +-outlier_scale*base_std."""
    rows: int = 64
    cols: int = 1024
    base_std: float = 1.0
    outlier_rate: float = 1e-3
    outlier_scale: float = 100.0
    seed: int = 1


def trial_seed(spec: OutlierSpec, trial: int) -> int:
    """Per-trial RNG stream derived deterministically from (seed, trial) (SPEC concurrency model)."""
    return spec.seed * 1_000_003 + trial


def trial_input(spec: OutlierSpec, trial: int, device) -> torch.Tensor:
    import synthetic  # the shared seeded generator (no method arithmetic)
    return synthetic.outlier_matrix(spec.rows, spec.cols, trial_seed(spec, trial), spec.base_std,
                                    spec.outlier_rate, spec.outlier_scale, device=device).contiguous()


def run_trial(x: torch.Tensor, target: str, per_tensor: bool) -> dict:
    """One trial on a resident fp32 CUDA matrix; every arithmetic step is a library kernel."""
    m, n = x.shape
    y = hadacore_fwht(x)                                   # rotate (normalized H, fp32 path)
    yq, amax_rot = fake_quant(y, target, per_tensor)       # quantize -> dequantize the rotated rows
    back = hadacore_fwht(yq)                               # inverse rotation (H H = I)
    xq, amax_plain = fake_quant(x, target, per_tensor)     # quantize -> dequantize the original rows
    e_rot = row_sq_error(back, x).sum()
    e_plain = row_sq_error(xq, x).sum()
    stats = torch.stack([e_plain / (m * n), e_rot / (m * n), amax_plain.max().double(), amax_rot.max().double()])
    mse_plain, mse_rot, max_plain, max_rot = stats.tolist()
    return {"mse_plain": mse_plain, "mse_rotated": mse_rot, "max_abs_plain": max_plain, "max_abs_rotated": max_rot}


def run_experiment(spec: OutlierSpec, target: str = "int4", granularity: str = "row", trials: int = 100,
                   device=None) -> dict:
    """SPEC run_experiment: per-trial and aggregate ExperimentReport."""
    if granularity not in ("row", "tensor"):
        raise ValueError("granularity must be 'row' or 'tensor'")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    per = []
    t0 = time.perf_counter()
    for t in range(trials):
        x = trial_input(spec, t, dev)
        r = run_trial(x, target, granularity == "tensor")
        r["trial"] = t
        per.append(r)
    torch.cuda.synchronize(dev)
    secs = time.perf_counter() - t0
    agg = {
        "mse_plain": sum(r["mse_plain"] for r in per) / max(1, trials),
        "mse_rotated": sum(r["mse_rotated"] for r in per) / max(1, trials),
        "win_rate": sum(r["mse_rotated"] < r["mse_plain"] for r in per) / max(1, trials),
        "max_abs_plain": max((r["max_abs_plain"] for r in per), default=0.0),
        "max_abs_rotated": max((r["max_abs_rotated"] for r in per), default=0.0),
    }
    return {"spec": dataclasses.asdict(spec), "target": target, "granularity": granularity, "trials": trials,
            "aggregate": agg, "per_trial": per, "seconds": secs}


def write_csv(report: dict, path_or_file) -> None:
    """One row per trial plus an aggregate row (SPEC External Interfaces)."""
    cols = ["trial", "mse_plain", "mse_rotated", "max_abs_plain", "max_abs_rotated"]
    own = isinstance(path_or_file, str)
    f = open(path_or_file, "w", newline="") if own else path_or_file
    try:
        w = csv.writer(f)
        w.writerow(cols + ["win_rate"])
        for r in report["per_trial"]:
            w.writerow([r[c] for c in cols] + [""])
        a = report["aggregate"]
        w.writerow(["aggregate", a["mse_plain"], a["mse_rotated"], a["max_abs_plain"], a["max_abs_rotated"],
                    a["win_rate"]])
    finally:
        if own:
            f.close()


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--target", choices=["e4m3", "int8", "int4"], default="int4")
    ap.add_argument("--granularity", choices=["row", "tensor"], default="row")
    ap.add_argument("--rows", type=int, default=64)
    ap.add_argument("--cols", type=int, default=1024)
    ap.add_argument("--base-std", type=float, default=1.0)
    ap.add_argument("--outlier-rate", type=float, default=1e-3)
    ap.add_argument("--outlier-scale", type=float, default=100.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--trials", type=int, default=100)
    ap.add_argument("--csv", default=None)
    a = ap.parse_args(argv)
    spec = OutlierSpec(a.rows, a.cols, a.base_std, a.outlier_rate, a.outlier_scale, a.seed)
    rep = run_experiment(spec, a.target, a.granularity, a.trials)
    if a.csv:
        write_csv(rep, a.csv)
    summary = {k: rep[k] for k in ("spec", "target", "granularity", "trials", "aggregate", "seconds")}
    print(json.dumps(summary))
    return 0


if __name__ == "__main__":
    sys.exit(main())
