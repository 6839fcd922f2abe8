"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no Hadamard, no butterfly, no
normalization).  It only draws numbers: a counter-based generator keyed on the
GLOBAL element index (row * n + col), so a row-sharded run on G GPUs produces
bit-identical data to the 1-GPU run.

Recipe:
  z  = splitmix64(seed * 0x9E3779B97F4A7C15 + (row * n + col))
  u1 = ((z >> 40) + 1) / 2^24          in (0, 1]
  u2 = ((z >> 16) & 0xFFFFFF) / 2^24   in [0, 1)
  D0: Box-Muller in fp32, r = sqrt(-2 ln u1), v = r cos(2 pi u2) ~ N(0, 1)
  D1: D0, with a 1e-3 fraction of entries replaced by +-100 (the activation-outlier
      shape of the paper's motivation, P:24 [Sec. 1]; SPEC OutlierSpec defaults),
      chosen by a second splitmix64 draw.
  then round-to-nearest-even to the requested dtype (torch's .to()).
Both distributions stay in the normal range of fp16/bf16.

Seeds: BASE_SEED = 241208832 (the arXiv id) + config index, + 100 for bf16.
"""
from __future__ import annotations

import torch

BASE_SEED = 241208832
_GOLDEN = -7046029254386353131  # 0x9E3779B97F4A7C15 as two's-complement int64
_M1 = -4658895280553007687      # 0xBF58476D1CE4E5B9
_M2 = -7723592293110705685      # 0x94D049BB133111EB
_SALT = 0x5DEECE66D
OUTLIER_RATE = 1e-3
OUTLIER_VALUE = 100.0


def seed_for(config_index: int, dtype: torch.dtype) -> int:
    return BASE_SEED + int(config_index) + (100 if dtype == torch.bfloat16 else 0)


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns (torch's >> is arithmetic)."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64 finalizer on int64 tensors holding uint64 bit patterns (wrapping)."""
    z = x + _GOLDEN
    z = (z ^ _lsr(z, 30)) * _M1
    z = (z ^ _lsr(z, 27)) * _M2
    return z ^ _lsr(z, 31)


def _wrap64(v: int) -> int:
    """Python int -> the int64 with the same low 64 bits (two's complement)."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def _uniform_pair(idx: torch.Tensor, seed: int):
    z = splitmix64(idx + _wrap64(seed * _GOLDEN))
    u1 = (_lsr(z, 40) + 1).to(torch.float32) * (1.0 / 16777216.0)
    u2 = ((z >> 16) & 0xFFFFFF).to(torch.float32) * (1.0 / 16777216.0)
    return u1, u2


def normal_block(row0: int, m: int, n: int, seed: int, dist: str = "D0",
                 device="cpu", outlier_rate: float = OUTLIER_RATE, outlier_value: float = OUTLIER_VALUE
                 ) -> torch.Tensor:
    """fp32 (m, n) block of rows [row0, row0+m) of the global seeded matrix."""
    rows = torch.arange(row0, row0 + m, device=device, dtype=torch.int64)
    cols = torch.arange(n, device=device, dtype=torch.int64)
    idx = rows[:, None] * n + cols[None, :]
    u1, u2 = _uniform_pair(idx, seed)
    v = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos((2.0 * torch.pi) * u2)
    if dist == "D1":
        h = splitmix64(idx ^ _wrap64(_SALT + seed))
        pick = (_lsr(h, 11).to(torch.float64) * (1.0 / 9007199254740992.0)) < outlier_rate
        sign = torch.where((h & 1) == 1, -1.0, 1.0).to(torch.float32)
        v = torch.where(pick, sign * float(outlier_value), v)
    elif dist != "D0":
        raise ValueError(f"unknown distribution {dist!r}")
    return v


def generate(m: int, n: int, dtype: torch.dtype, seed: int, dist: str = "D0", row0: int = 0,
             device="cpu", out: torch.Tensor | None = None, chunk_elems: int = 1 << 24) -> torch.Tensor:
    """Seeded (m, n) matrix of `dtype` (RNE from fp32), generated in row chunks."""
    if out is None:
        out = torch.empty((m, n), dtype=dtype, device=device)
    rows_per_chunk = max(1, chunk_elems // max(n, 1))
    for r in range(0, m, rows_per_chunk):
        k = min(rows_per_chunk, m - r)
        out[r:r + k].copy_(normal_block(row0 + r, k, n, seed, dist, device=out.device).to(dtype))
    return out


def special_rows(n: int, dtype: torch.dtype) -> tuple[torch.Tensor, list[str]]:
    """Edge-case rows; returned with their names.

    zeros, one-hot at 0, one-hot at n-1, constant 4.0 (fp16 range trap for
    unnormalized intermediates), all-ones, a lone +Inf among finite values, a lone
    NaN, and a row in the subnormal range of the dtype.
    """
    names, rows = [], []

    def add(name, vals):
        names.append(name)
        rows.append(vals)

    add("zeros", torch.zeros(n))
    e0 = torch.zeros(n); e0[0] = 1.0; add("onehot0", e0)
    el = torch.zeros(n); el[n - 1] = -2.0; add("onehot_last", el)
    add("const4", torch.full((n,), 4.0))
    add("ones", torch.ones(n))
    g = normal_block(0, 1, n, BASE_SEED + 7)[0]
    inf_row = g.clone(); inf_row[n // 3] = float("inf"); add("inf", inf_row)
    nan_row = g.clone(); nan_row[n // 5] = float("nan"); add("nan", nan_row)
    tiny = torch.finfo(dtype).tiny  # smallest normal
    add("subnormal", g * (tiny / 8.0))
    return torch.stack(rows).to(dtype), names


def outlier_matrix(m: int, n: int, seed: int, base_std: float = 1.0, outlier_rate: float = OUTLIER_RATE,
                   outlier_scale: float = OUTLIER_VALUE, device="cpu") -> torch.Tensor:
    """SPEC quant_lab OutlierSpec: fp32 (m, n) Gaussian(0, base_std) entries
    with an outlier_rate fraction resampled at +-outlier_scale * base_std (the D1 draw
    with parameters); deterministic per seed."""
    if not (0.0 <= outlier_rate <= 1.0) or outlier_scale < 1.0 or base_std <= 0.0:
        raise ValueError("BadSpec: need 0 <= outlier_rate <= 1, outlier_scale >= 1, base_std > 0")
    v = normal_block(0, m, n, seed, "D1", device=device, outlier_rate=outlier_rate, outlier_value=outlier_scale)
    return v * float(base_std)
