"""World-size-2 (and 3) gloo tests of the multi-GPU host logic on CPU: the row
partition covers every row exactly once, per-rank seeded shards equal the
single-process matrix (the generator is keyed on global indices), and gathering the
per-rank transforms reproduces the single-process result bit for bit.  The per-rank
transform here is the oracle (no GPU on this host); on a GPU box bench.py runs the
same partition with hadacore_fwht."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_08832_b200.shard import gather_rows, row_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_row_range_partition():
    for m in [0, 1, 5, 7, 1024, 1 << 18]:
        for g in [1, 2, 3, 4, 8]:
            ranges = [row_range(m, r, g) for r in range(g)]
            assert ranges[0][0] == 0 and ranges[-1][1] == m
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        row_range(10, 2, 2)


def _worker(rank, world, port, m, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synthetic
        lo, hi = row_range(m, rank, world)
        x = synthetic.generate(hi - lo, n, torch.bfloat16, 1234, dist="D1", row0=lo)
        y = torch.from_numpy(oracle.fwht(x.double().numpy(), threads=1)).to(torch.bfloat16)
        full_x = gather_rows(x, m, dist)
        full_y = gather_rows(y, m, dist)
        # max-over-ranks timing reduction as bench.py does it
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            q.put((full_x.view(torch.int16).numpy(), full_y.view(torch.int16).numpy(), t.item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_equals_single_process(world):
    m, n = 37, 512
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    fx, fy, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    import oracle
    import synthetic
    x = synthetic.generate(m, n, torch.bfloat16, 1234, dist="D1")
    y = torch.from_numpy(oracle.fwht(x.double().numpy(), threads=1)).to(torch.bfloat16)
    assert np.array_equal(fx, x.view(torch.int16).numpy())
    assert np.array_equal(fy, y.view(torch.int16).numpy())
    assert tmax == float(world)
