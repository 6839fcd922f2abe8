"""torch.library custom ops over the C ABI (NEXT-3 in SURVEY.md 8(f): the paper's
deployment context -- online Q/K rotation before FP8 attention).

    import paper_2412_08832_b200.torch_ops            # registers the ops
    y = torch.ops.hadacore.fwht(x, None)               # scale None -> 1/sqrt(n)
    torch.ops.hadacore.fwht_(x, None)                  # in place
    q, s = torch.ops.hadacore.fwht_quant(x, "e4m3", None)

The ops launch the same kernels as ``hadacore_fwht`` (no PyTorch compute); fake
(meta) implementations make them traceable by ``torch.compile`` / ``torch.export``.
The transform is linear and H_n is symmetric, so the backward of ``fwht`` is
``fwht`` of the incoming gradient with the same scale (registered below).
"""
from __future__ import annotations

import math

import torch

from . import QTYPES, HadacoreError, hadacore_fwht, hadacore_fwht_quant, hadacore_fwht_quant_strided


@torch.library.custom_op("hadacore::fwht", mutates_args=())
def fwht(x: torch.Tensor, scale: float | None = None) -> torch.Tensor:
    return hadacore_fwht(x.contiguous(), scale=scale)


@fwht.register_fake
def _(x: torch.Tensor, scale: float | None = None) -> torch.Tensor:
    return torch.empty_like(x)


def _fwht_backward(ctx, grad):
    # d/dx (s H x) = s H^T = s H (H symmetric)
    return torch.ops.hadacore.fwht(grad.contiguous(), ctx.scale), None


def _fwht_setup(ctx, inputs, output):
    x, scale = inputs
    ctx.scale = scale if scale is not None else 1.0 / math.sqrt(x.shape[-1])


fwht.register_autograd(_fwht_backward, setup_context=_fwht_setup)


@torch.library.custom_op("hadacore::fwht_", mutates_args=("x",))
def fwht_(x: torch.Tensor, scale: float | None = None) -> None:
    if not x.is_contiguous():
        raise ValueError("hadacore::fwht_ needs a contiguous tensor")
    hadacore_fwht(x, out=x, scale=scale)


@fwht_.register_fake
def _(x: torch.Tensor, scale: float | None = None) -> None:
    return None


@torch.library.custom_op("hadacore::fwht_quant", mutates_args=())
def fwht_quant(x: torch.Tensor, qtype: str = "e4m3", scale: float | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    if not x.is_contiguous() and x.stride(-1) == 1 and x.shape[-1] >= 128:
        try:  # strided rows (e.g. Q/K heads of a QKV view): read in place, no copy
            return hadacore_fwht_quant_strided(x, qtype=qtype, scale=scale)
        except HadacoreError:
            pass  # more than two row dims or unsupported strides: fall through to a contiguous copy
    return hadacore_fwht_quant(x.contiguous(), qtype=qtype, scale=scale)


@fwht_quant.register_fake
def _(x: torch.Tensor, qtype: str = "e4m3", scale: float | None = None):
    shape = x.shape if qtype != "int4" else (*x.shape[:-1], x.shape[-1] // 2)  # int4: two codes per byte
    return (torch.empty(shape, dtype=QTYPES[qtype][1], device=x.device),
            torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device))
