"""Summarize an ncu --set full capture of the fwht kernels (run here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_full.md [--traffic profiles/ncu_traffic.json]
        [--alg-bytes B]   (algorithmic bytes per element: 4 for the 16-bit transform (default), 3 for
                           E4M3/INT8 fused quantization, 2.5 for INT4; the 4-byte row scales are added)

Writes a markdown table per launch: n, dtype, duration, DRAM read/write bytes,
DRAM throughput %, issue %, warps active %, HMMA pipe %, shared bank conflicts,
top stall reasons; optionally the per-launch traffic JSON that bench.py reports.
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = {
    "dur_us": "gpu__time_duration.sum",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "hmma_pct": "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "inst": "smsp__inst_executed.sum",
    "bank_conf": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "regs": "launch__registers_per_thread",
    "tensor_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
}


def unit_scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(
        unit, 1)


def main():
    rep, out_md = sys.argv[1], sys.argv[2]
    traffic_path = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    alg_b = float(sys.argv[sys.argv.index("--alg-bytes") + 1]) if "--alg-bytes" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = ["| kernel | n | dtype | time µs | DRAM rd MB | DRAM wr MB | (rd+wr)/algorithmic | DRAM % | issue % | "
             "warps % | HMMA % | tensor pipe % | smem bank confl. | regs | top stalls |", "|" + "---|" * 15]
    traffic = []
    for d in data:
        name = d[hdr.index("Kernel Name")]
        mm = re.search(r"(fwht_\w+)<(?:\(int\))?(\d+), (?:\(int\))?(\d+)", name)
        kern, n, dt = (mm.group(1), int(mm.group(2)), "fp16" if mm.group(3) == "0" else "bf16") if mm else (name[:30], 0, "?")
        if "f32" in kern or "f32_pair" in name:  # fp32 kernels: <N, TILE_BYTES, ...>, the pair kernel is n = 2^15
            kern = "fwht_f32_pair_kernel" if "pair" in name else kern
            n, dt = (32768 if "pair" in name else n), "fp32"
        v = {}
        for k, col in KEYS.items():
            if col in hdr:
                i = hdr.index(col)
                try:
                    v[k] = float(d[i]) * (unit_scale(units[i]) if k in ("rd", "wr", "dur_us") else 1)
                except ValueError:
                    v[k] = float("nan")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                nm = h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
                if nm != "selected":
                    try:
                        stalls.append((float(d[i]), nm))
                    except ValueError:
                        pass
        stalls.sort(reverse=True)
        alg = (alg_b * (1 << 28) + 4.0 * (1 << 28) / max(n, 1)) if alg_b else (8.0 if dt == "fp32" else 4.0) * (1 << 28)
        ratio = (v.get("rd", 0) + v.get("wr", 0)) / alg
        lines.append(f"| {kern} | {n} | {dt} | {v.get('dur_us', 0):.1f} | {v.get('rd', 0)/1e6:.1f} | {v.get('wr', 0)/1e6:.1f} | "
                     f"{ratio:.3f} | {v.get('dram_pct', 0):.1f} | {v.get('issue_pct', 0):.1f} | {v.get('warps_pct', 0):.1f} | "
                     f"{v.get('hmma_pct', 0):.1f} | {v.get('tensor_pct', float('nan')):.1f} | {v.get('bank_conf', 0):.0f} | {v.get('regs', 0):.0f} | "
                     + ", ".join(f"{nm} {x:.2f}" for x, nm in stalls[:3]) + " |")
        traffic.append({"n": n, "dtype": dt, "dram_bytes": v.get("rd", 0) + v.get("wr", 0), "duration_us": v.get("dur_us")})
    alg_note = (f"{alg_b} B x 2^28 + 4 B per row (fused quantization: 2 B read + codes + row scales)" if alg_b else
                f"4 B x 2^28 = {4 * (1 << 28)} (16-bit; 8 B x 2^28 for fp32; read + write once)")
    open(out_md, "w").write(f"# ncu --set full summary of `{rep}`\n\nAlgorithmic bytes per launch = {alg_note}.\n\n"
                            + "\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_path:
        avg = sum(t["dram_bytes"] for t in traffic) / max(1, len(traffic))
        json.dump({"source": f"ncu --set full --clock-control none ({rep}), dram__bytes_read.sum + dram__bytes_write.sum",
                   "avg_dram_bytes_per_launch": round(avg), "per_launch": traffic}, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    main()
