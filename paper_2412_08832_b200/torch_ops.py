"""torch.library custom ops over the C ABI (NEXT-3 in SURVEY.md 8(f): the paper's
deployment context -- online Q/K rotation before FP8 attention).

    import paper_2412_08832_b200.torch_ops            # registers the ops
    y = torch.ops.hadacore.fwht(x, None)               # scale None -> 1/sqrt(n)
    torch.ops.hadacore.fwht_(qkv[:, 0:2], None)        # in place, also on strided views
    q, s = torch.ops.hadacore.fwht_quant(qkv[:, 0:2], "e4m3", None)

The ops launch the same kernels as ``hadacore_fwht`` (no PyTorch compute).  A view
whose last dimension is contiguous and whose leading dimensions collapse to at most
two strided row dimensions (the Q and K heads of a fused ``[T, 3, H, d]`` projection,
a padded-pitch matrix) goes through the strided entry points (``hadacore_fwht_strided``,
``hadacore_fwht_quant_strided``; n >= 8), read and written where it lies -- no
``.contiguous()`` copy.  Fake (meta) implementations make the ops traceable by
``torch.compile`` / ``torch.export``.  The transform is linear and H_n is symmetric,
so the backward of ``fwht`` is ``fwht`` of the incoming gradient with the same scale.
"""
from __future__ import annotations

import math

import torch

from . import (QTYPES, HadacoreError, _row_grid, hadacore_fwht, hadacore_fwht_quant, hadacore_fwht_quant_strided,
               hadacore_fwht_strided)

STRIDED_MIN_N = 8  # the strided entry points need rows of >= 16 bytes (TMA boxes)


def _strided_ok(x: torch.Tensor) -> bool:
    """True if the strided C entry takes this view as it lies: contiguous last dim, n >= 8,
    <= 2 collapsible row dims with strides that are multiples of 8 elements, 16-byte aligned."""
    n = x.shape[-1]
    if x.dim() < 2 or x.stride(-1) != 1 or n < STRIDED_MIN_N or x.numel() == 0:
        return False
    if x.data_ptr() % 16:
        return False
    try:
        _, _, so, si = _row_grid(x, n)
    except HadacoreError:
        return False
    return so % 8 == 0 and si % 8 == 0


@torch.library.custom_op("hadacore::fwht", mutates_args=())
def fwht(x: torch.Tensor, scale: float | None = None) -> torch.Tensor:
    if x.is_contiguous():
        return hadacore_fwht(x, scale=scale)
    if _strided_ok(x):  # strided rows read in place, result written contiguously
        return hadacore_fwht_strided(x, scale=scale)
    return hadacore_fwht(x.contiguous(), scale=scale)


@fwht.register_fake
def _(x: torch.Tensor, scale: float | None = None) -> torch.Tensor:
    # the real op always returns a new contiguous tensor
    return torch.empty(x.shape, dtype=x.dtype, device=x.device)


def _fwht_backward(ctx, grad):
    # d/dx (s H x) = s H^T = s H (H symmetric)
    return torch.ops.hadacore.fwht(grad, ctx.scale), None


def _fwht_setup(ctx, inputs, output):
    x, scale = inputs
    ctx.scale = scale if scale is not None else 1.0 / math.sqrt(x.shape[-1])


fwht.register_autograd(_fwht_backward, setup_context=_fwht_setup)


@torch.library.custom_op("hadacore::fwht_", mutates_args=("x",))
def fwht_(x: torch.Tensor, scale: float | None = None) -> None:
    if x.is_contiguous():
        hadacore_fwht(x, out=x, scale=scale)
    elif _strided_ok(x):  # e.g. qkv[:, 0:2]: the Q and K heads rotated where they lie
        hadacore_fwht_strided(x, out=x, scale=scale)
    else:
        raise ValueError("hadacore::fwht_ needs a contiguous tensor or a view with a contiguous last dim "
                         f"(n >= {STRIDED_MIN_N}) and at most two row dims with strides that are multiples of 8")


@fwht_.register_fake
def _(x: torch.Tensor, scale: float | None = None) -> None:
    return None


@torch.library.custom_op("hadacore::fwht_quant", mutates_args=())
def fwht_quant(x: torch.Tensor, qtype: str = "e4m3", scale: float | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    if not x.is_contiguous() and _strided_ok(x):
        # strided rows (e.g. Q/K heads of a QKV view): read in place, no copy
        return hadacore_fwht_quant_strided(x, qtype=qtype, scale=scale)
    return hadacore_fwht_quant(x.contiguous(), qtype=qtype, scale=scale)


@fwht_quant.register_fake
def _(x: torch.Tensor, qtype: str = "e4m3", scale: float | None = None):
    shape = x.shape if qtype != "int4" else (*x.shape[:-1], x.shape[-1] // 2)  # int4: two codes per byte
    return (torch.empty(shape, dtype=QTYPES[qtype][1], device=x.device),
            torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device))
