"""Host logic of bench.py's multi-rank result check ("gather of outputs (or
sampled rows) to rank 0 for the oracle check and for a bitwise comparison against the G = 1
output"), on CPU with gloo at world size 2: rows regenerated from their global index equal
the resident slices, the gather + check passes when every rank transforms its own rows, and
the --misshard negative control (one rank's slice generated one base row off) fails it.
The per-rank transform here is the oracle rounded to the dtype (no GPU on this host); on a
GPU box bench.py runs the same functions with hadacore_fwht."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import synthetic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_transform(x):
    import oracle
    return torch.from_numpy(oracle.fwht(x.double().numpy(), threads=1)).to(x.dtype)


@pytest.mark.parametrize("n", [128, 256, 1024])
def test_gen_rows_matches_resident_slices(n):
    elems, world = 1 << 13, 3
    for rank in range(world):
        flat0, el, total = bench.rank_layout("fwht", rank, world, elems)
        assert (flat0, el, total) == (rank * elems, elems, world * elems)
        buf = torch.empty(el, dtype=torch.bfloat16)
        bench.fill_resident(buf, "fwht", torch.bfloat16, flat0)
        rows = buf.view(-1, n)
        for i in bench.sample_local_rows(n, torch.bfloat16, rank, rows.shape[0], 5):
            g = flat0 // n + i
            assert torch.equal(bench.gen_rows("fwht", torch.bfloat16, n, g, 1, "cpu")[0].view(torch.int16),
                               rows[i].view(torch.int16))
    # a workload whose base width is its n (C4) regenerates exactly synthetic.generate's rows
    a = bench.gen_rows("c4", torch.float16, 4096, 77, 3, "cpu")
    b = synthetic.generate(3, 4096, torch.float16, bench.seed_of("c4", torch.float16), row0=77)
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))


def test_sample_rows_deterministic_and_bounded():
    for m in (1, 2, 5, 1000):
        a = bench.sample_local_rows(512, torch.float16, 1, m, 4)
        assert a == bench.sample_local_rows(512, torch.float16, 1, m, 4)
        assert len(a) == 4 and a[0] == 0 and a[1] == m - 1 and all(0 <= i < m for i in a)
    assert bench.sample_local_rows(512, torch.float16, 0, 1000, 4) != bench.sample_local_rows(512, torch.float16, 1,
                                                                                                1000, 4)


def _worker(rank, world, port, misshard, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        elems, k = 1 << 12, 4
        flat0, el, _ = bench.rank_layout("fwht", rank, world, elems)
        shift = 256 if (misshard and rank == world - 1) else 0
        gathered = {}
        for dt in (torch.float16, torch.bfloat16):
            buf = torch.empty(el, dtype=dt)
            bench.fill_resident(buf, "fwht", dt, flat0, shift)
            for n in (128, 512):
                y = _oracle_transform(buf.view(-1, n))
                gathered[(dt, n)] = bench.gather_sample(y, n, dt, rank, world, k, dist)
        if rank == 0:
            res = bench.sampled_rows_check(gathered, "fwht", world, elems, k, dist, _oracle_transform, "cpu")
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("misshard", [False, True])
def test_two_rank_gather_and_check(misshard):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, misshard, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res["ranks"] == 2 and res["rows_checked"] == 2 * 2 * 2 * 4
    assert res["gather"].startswith("gloo")
    if not misshard:
        assert res["pass"] and res["oracle_pass"] and res["bitwise_mismatches_vs_rank0_recompute"] == 0
        assert max(res["oracle_max_rel_err"].values()) <= 1.6e-2
    else:
        # rank 1's rows are other global rows: both the oracle and the bitwise check catch it,
        # and only rank 1's rows fail
        assert not res["pass"] and not res["oracle_pass"]
        assert res["bitwise_mismatches_vs_rank0_recompute"] == 2 * 2 * 4
        assert all(r["row"] >= (1 << 12) // r["n"] for r in res["failing_rows"])
