"""Digest an ncu source page (SASS) of one kernel launch: instruction counts, warp-stall
samples and shared-memory wavefronts grouped by opcode, plus the hottest lines.

    ncu -i rep.ncu-rep --page source --csv --print-source sass --launch-skip K --launch-count 1 > src.csv
    python tools/sass_profile.py src.csv [--top 30] [--per-unit UNITS]

--per-unit divides instruction counts by UNITS (e.g. warp-level 256-element chunks of the
launch) so the table reads as "warp instructions per unit".
"""
import csv
import io
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    per = float(sys.argv[sys.argv.index("--per-unit") + 1]) if "--per-unit" in sys.argv else None
    text = open(path).read()
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows, seen = [], set()
    for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))):
        # the page repeats its table (and header rows); count every SASS address once
        if not r["Address"].startswith("0x") or r["Address"] in seen:
            continue
        seen.add(r["Address"])
        rows.append(r)

    def f(r, k):
        try:
            return float(r.get(k, "0") or 0)
        except ValueError:
            return 0.0
    by_op = defaultdict(lambda: [0.0, 0.0, 0.0, 0.0, 0])
    tot_i = tot_s = 0.0
    for r in rows:
        src = r["Source"].strip()
        tok = src.split()
        if not tok:
            continue
        op = tok[0]
        if op.startswith("@"):
            op = tok[1] if len(tok) > 1 else op
        op = op.rstrip(";")
        ins, smp = f(r, "Instructions Executed"), f(r, "Warp Stall Sampling (All Samples)")
        wf, wfi = f(r, "L1 Wavefronts Shared"), f(r, "L1 Wavefronts Shared Ideal")
        b = by_op[op]
        b[0] += ins
        b[1] += smp
        b[2] += wf
        b[3] += wfi
        b[4] += 1
        tot_i += ins
        tot_s += smp
    print(f"total warp instructions {tot_i:.0f}" + (f" ({tot_i / per:.1f} per unit)" if per else "") +
          f", stall samples {tot_s:.0f}")
    print(f"{'opcode':28s} {'instr':>12s} {'%':>6s} {'per unit':>9s} {'samples %':>9s} {'smem wf':>10s} {'ideal':>10s}")
    for op, (ins, smp, wf, wfi, cnt) in sorted(by_op.items(), key=lambda t: -t[1][0]):
        if ins == 0 and smp == 0:
            continue
        print(f"{op:28s} {ins:12.0f} {100 * ins / tot_i:6.2f} {ins / per if per else 0:9.2f} "
              f"{100 * smp / max(tot_s, 1):9.2f} {wf:10.0f} {wfi:10.0f}")
    print(f"\nhottest lines (by stall samples):")
    hot = sorted(rows, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]
    for r in hot:
        print(f"{r['Address'][-5:]} {f(r, 'Warp Stall Sampling (All Samples)'):7.0f} "
              f"{f(r, 'Instructions Executed'):10.0f}  {r['Source'].strip()[:90]}")
    exc = sorted(rows, key=lambda r: -(f(r, "L1 Wavefronts Shared") - f(r, "L1 Wavefronts Shared Ideal")))[:10]
    print("\nexcess shared wavefronts by line:")
    for r in exc:
        d = f(r, "L1 Wavefronts Shared") - f(r, "L1 Wavefronts Shared Ideal")
        if d <= 0:
            break
        print(f"{r['Address'][-5:]} excess {d:10.0f} of {f(r, 'L1 Wavefronts Shared'):10.0f}  {r['Source'].strip()[:90]}")


if __name__ == "__main__":
    main()
