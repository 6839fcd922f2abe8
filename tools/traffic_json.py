"""Per-launch DRAM traffic JSON for bench.py's roofline.traffic, from an `ncu --metrics
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv` launch list (one
launch per (dtype, n), in the order tools/ncu_quant.py / ncu_one.py issue them).

    python tools/traffic_json.py launches.csv out.json "<source note>" [alg_bytes_per_el] [ns] [dtypes: fp16,bf16]
"""
import csv
import io
import json
import re
import sys


def main():
    src, out, note = sys.argv[1], sys.argv[2], sys.argv[3]
    bpe = float(sys.argv[4]) if len(sys.argv) > 4 else 4.0
    ns = [int(v) for v in sys.argv[5].split(",")] if len(sys.argv) > 5 else [1 << k for k in range(7, 16)]
    text = open(src).read()
    body = text[text.index('"ID"'):]
    per = {}
    for r in csv.DictReader(io.StringIO(body)):
        per.setdefault(int(r["ID"]), {"kernel": r["Kernel Name"]})[r["Metric Name"]] = float(r["Metric Value"])
    launches = [per[k] for k in sorted(per)]
    dts = sys.argv[6].split(",") if len(sys.argv) > 6 else ["fp16", "bf16"]
    order = [(dt, n) for dt in dts for n in ns]
    rows = []
    for (dt, n), l in zip(order, launches):
        rd, wr = l.get("dram__bytes_read.sum", 0.0), l.get("dram__bytes_write.sum", 0.0)
        dur = l.get("gpu__time_duration.sum", 0.0)
        alg = bpe * (1 << 28) + (4.0 * ((1 << 28) // n) if bpe < 4.0 else 0.0)  # + row scales when quantizing
        m = re.match(r"void (?:hadacore::)?(\w+)", l["kernel"])
        rows.append({"n": n, "dtype": dt, "kernel": m.group(1) if m else l["kernel"][:40], "dram_bytes": rd + wr,
                     "read_bytes": rd, "write_bytes": wr, "duration_us": dur / 1e3 if dur > 1e4 else dur,
                     "algorithmic_bytes": alg, "traffic_over_algorithmic": round((rd + wr) / alg, 4)})
    avg = sum(r["dram_bytes"] for r in rows) / max(1, len(rows))
    json.dump({"source": note, "algorithmic_bytes_per_element": bpe, "avg_dram_bytes_per_launch": round(avg),
               "per_launch": rows}, open(out, "w"), indent=1)
    for r in rows:
        print(r["dtype"], r["n"], r["kernel"], f"{r['dram_bytes'] / 1e6:.1f} MB", r["traffic_over_algorithmic"])


if __name__ == "__main__":
    main()
