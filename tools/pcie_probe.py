"""PCIe ceiling vs the host-buffer entry (hadacore_fwht_host): pinned H2D alone, D2H alone,
both directions concurrently, and the library's pipelined H2D -> kernel -> D2H, in GB/s."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_08832_b200 as hc  # noqa: E402

N = 1 << 28  # fp16 elements: 512 MiB each way
h_in = torch.empty(N, dtype=torch.float16).pin_memory()
h_out = torch.empty(N, dtype=torch.float16).pin_memory()
d_a = torch.empty(N, dtype=torch.float16, device="cuda")
d_b = torch.empty(N, dtype=torch.float16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
B = 2 * N


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


t = timeit(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D alone      {B / t / 1e9:7.1f} GB/s")
t = timeit(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H alone      {B / t / 1e9:7.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


t = timeit(both)
print(f"H2D + D2H      {2 * B / t / 1e9:7.1f} GB/s total ({B / t / 1e9:.1f} per direction)")
for ws_mb in (64, 256):
    ws = torch.empty(ws_mb << 20, dtype=torch.uint8, device="cuda")
    for n in (256, 4096):
        x, y = h_in.view(-1, n), h_out.view(-1, n)
        t = timeit(lambda: hc.hadacore_fwht_host(x, out=y, workspace=ws))
        print(f"fwht_host n={n:5d} ws={ws_mb:3d} MiB: {2 * B / t / 1e9:7.1f} GB/s algorithmic (4 B/el) "
              f"= {B / t / 1e9:.1f} GB/s per direction")
