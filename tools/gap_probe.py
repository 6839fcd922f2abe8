"""Inter-launch gap probe (dev tool): the C3 sweep timed as one region with and
without per-launch CUDA events between the kernels (an event record between two
PDL launches may break the programmatic overlap), plus back-to-back repeats of
one (dtype, n)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_08832_b200 as hc  # noqa: E402

NS = [1 << k for k in range(7, 16)]
E = 1 << 28


def main():
    xin = {dt: torch.randn(E, device="cuda").to(dt) for dt in (torch.float16, torch.bfloat16)}
    out = torch.empty(E, dtype=torch.float16, device="cuda")
    pairs = [(dt, n) for dt in xin for n in NS]
    st = torch.cuda.current_stream()

    def launch(dt, n):
        hc.hadacore_fwht(xin[dt].view(-1, n), out=out.view(dt).view(-1, n), stream=st)

    def region(steps, per_launch_events):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps * len(pairs))]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        i = 0
        for _ in range(steps):
            for dt, n in pairs:
                if per_launch_events:
                    evs[i][0].record(st)
                launch(dt, n)
                if per_launch_events:
                    evs[i][1].record(st)
                i += 1
        b.record(st)
        torch.cuda.synchronize()
        tot = a.elapsed_time(b)
        s = sum(x.elapsed_time(y) for x, y in evs) if per_launch_events else float("nan")
        return 4.0 * E * steps * len(pairs) / (tot * 1e-3) / 1e9, 4.0 * E * steps * len(pairs) / (s * 1e-3) / 1e9

    for _ in range(2):
        region(2, False)
    for rep in range(4):
        v0, _ = region(10, False)
        v1, v1k = region(10, True)
        print(f"rep {rep}: no events {v0:.0f} GB/s | per-launch events: region {v1:.0f} GB/s, sum-of-launches {v1k:.0f} GB/s",
              flush=True)
    for dt, n in [(torch.float16, 128), (torch.bfloat16, 4096), (torch.bfloat16, 32768)]:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launch(dt, n)
        a.record(st)
        for _ in range(20):
            launch(dt, n)
        b.record(st)
        torch.cuda.synchronize()
        print(f"{dt} n={n}: 20 back-to-back launches {4.0 * E * 20 / (a.elapsed_time(b) * 1e-3) / 1e9:.0f} GB/s")


if __name__ == "__main__":
    main()
