"""Run the NEXT-4 quantization lab over targets x granularity x outlier settings on the
GPU and print a markdown table (profiles/r01_quant_lab_matrix.md)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_08832_b200 import quant_lab  # noqa: E402

rows = []
for rate, scale in ((1e-3, 100.0), (0.0, 1.0)):
    for target in ("int4", "int8", "e4m3"):
        for gran in ("row", "tensor"):
            spec = quant_lab.OutlierSpec(rows=64, cols=1024, outlier_rate=rate, outlier_scale=scale, seed=1)
            r = quant_lab.run_experiment(spec, target, gran, trials=100)
            a = r["aggregate"]
            rows.append((rate, scale, target, gran, a["mse_plain"], a["mse_rotated"], a["mse_rotated"] / a["mse_plain"],
                         a["win_rate"], a["max_abs_plain"], a["max_abs_rotated"], r["seconds"]))
print("| outlier rate x scale | target | granularity | mse_plain | mse_rotated | rotated/plain | win rate | "
      "max_abs plain | max_abs rotated | s (100 trials) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for (rate, scale, t, g, mp, mr, q, w, xp, xr, sec) in rows:
    print(f"| {rate:g} x {scale:g} | {t} | {g} | {mp:.4e} | {mr:.4e} | {q:.3f} | {w:.2f} | {xp:.2f} | {xr:.2f} | {sec:.2f} |")
print(json.dumps({"rows": rows}))
