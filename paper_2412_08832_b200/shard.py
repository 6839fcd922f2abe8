"""Row sharding across ranks (host logic only).

Rows are independent (P:77 [Sec. 2.3]), so a multi-GPU run gives every rank a
contiguous block of rows and calls hadacore_fwht on it -- no collective on the hot
path.  Collectives (torch.distributed) are only used to gather results or timings
for checking.
"""
from __future__ import annotations


def row_range(m: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [lo, hi) owned by `rank` of `world`: floor(r*m/G) .. floor((r+1)*m/G)."""
    if world < 1 or not (0 <= rank < world) or m < 0:
        raise ValueError(f"bad partition m={m} rank={rank} world={world}")
    return (rank * m) // world, ((rank + 1) * m) // world


def gather_rows(local, m: int, dist, dst: int = 0):
    """Gather every rank's row block (same dtype/width) into the full m x n matrix on
    `dst` (None elsewhere).  Blocks may differ in length by one row."""
    import torch
    world, rank = dist.get_world_size(), dist.get_rank()
    n = local.shape[-1]
    sizes = [row_range(m, r, world)[1] - row_range(m, r, world)[0] for r in range(world)]
    cap = max(sizes)
    buf = torch.zeros((cap, n), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    # gather the raw payload as int32 words (n is even), which gloo and NCCL both accept
    payload = buf.view(torch.int32)
    out = [torch.empty_like(payload) for _ in range(world)] if rank == dst else None
    dist.gather(payload, out, dst=dst)
    if rank != dst:
        return None
    full = torch.cat([o[:s] for o, s in zip(out, sizes)])
    return full.view(local.dtype)
