"""B200-native batched normalized Walsh-Hadamard transform (HadaCore, arXiv 2412.08832).

Thin Python binding over the C ABI in ``include/hadacore.h`` (``libhadacore.so``,
built in-tree for sm_100a).  Argument marshalling only: every step of the
transform runs in the CUDA kernel.  There is no CPU or PyTorch fallback -- if the
library is missing or no GPU is present, calls raise.

    out = hadacore_fwht(x)                 # scale = 1/sqrt(n), out-of-place
    hadacore_fwht(x, out=x)                # in place (App. B)
    y = hadacore_fwht_host(x_cpu)          # host buffers, copies pipelined in C

``x`` is a CUDA tensor of dtype float16 or bfloat16 whose last dimension n is a
power of two in [2, 32768] (the paper's 2^7..2^15, plus n = 2..64: SURVEY.md 8(f)
NEXT-2); all leading dimensions are rows (m = numel / n).  The strided entry
points take n = 2^3..2^15 (rows of >= 16 bytes: TMA boxes).  ``scale`` must be
finite and > 0.
"""
from __future__ import annotations

import ctypes
import math
import os

import torch

__all__ = ["ARG_ERROR", "hadacore_fwht", "hadacore_fwht_host", "hadacore_fwht_quant", "hadacore_fwht_strided", "fwht", "HadacoreError",
           "library_path", "version", "launches_per_call", "STATUS", "QTYPES", "fake_quant", "row_sq_error",
           "hadacore_fwht_quant_strided"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libhadacore.so")
_lib = None

ARG_ERROR = -1  # Python-side argument check (tensor shape / dtype / device / layout mismatch), not a C status
STATUS = {
    ARG_ERROR: "PYTHON_ARGUMENT",
    0: "HADACORE_OK", 1: "HADACORE_ERR_INVALID_N", 2: "HADACORE_ERR_INVALID_M", 3: "HADACORE_ERR_NULL",
    4: "HADACORE_ERR_MISALIGNED", 5: "HADACORE_ERR_OVERLAP", 6: "HADACORE_ERR_DTYPE",
    7: "HADACORE_ERR_SCALE", 8: "HADACORE_ERR_CUDA", 9: "HADACORE_ERR_WORKSPACE",
}
_DTYPES = {torch.float16: 0, torch.bfloat16: 1, torch.float32: 2}
QTYPES = {"e4m3": (0, torch.float8_e4m3fn), "int8": (1, torch.int8), "int4": (2, torch.uint8)}  # int4: 2 per byte
LAB_QTYPES = {"e4m3": 0, "int8": 1, "int4": 2}  # hadacore_fake_quant (quant lab, NEXT-4)


class HadacoreError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def library_path() -> str:
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: build it with `python -m paper_2412_08832_b200.build` "
                          "(nvcc, sm_100a). There is no fallback implementation.")
    lib = ctypes.CDLL(_LIB_PATH)
    vp, i64, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_float
    lib.hadacore_fwht.argtypes = [vp, vp, i64, i64, ctypes.c_int, f32, vp]
    lib.hadacore_fwht.restype = ctypes.c_int
    lib.hadacore_fwht_host.argtypes = [vp, vp, i64, i64, ctypes.c_int, f32, vp, ctypes.c_size_t, vp]
    lib.hadacore_fwht_host.restype = ctypes.c_int
    lib.hadacore_fwht_quant.argtypes = [vp, vp, vp, i64, i64, ctypes.c_int, ctypes.c_int, f32, vp]
    lib.hadacore_fwht_quant.restype = ctypes.c_int
    lib.hadacore_fwht_strided.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, ctypes.c_int, f32, vp]
    lib.hadacore_fwht_strided.restype = ctypes.c_int
    lib.hadacore_fwht_quant_strided.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, ctypes.c_int, ctypes.c_int, f32, vp]
    lib.hadacore_fwht_quant_strided.restype = ctypes.c_int
    lib.hadacore_fake_quant.argtypes = [vp, vp, vp, i64, i64, ctypes.c_int, ctypes.c_int, vp]
    lib.hadacore_fake_quant.restype = ctypes.c_int
    lib.hadacore_row_sq_error.argtypes = [vp, vp, vp, i64, i64, vp]
    lib.hadacore_row_sq_error.restype = ctypes.c_int
    lib.hadacore_status_string.argtypes = [ctypes.c_int]
    lib.hadacore_status_string.restype = ctypes.c_char_p
    lib.hadacore_version.argtypes = []
    lib.hadacore_version.restype = ctypes.c_int
    lib.hadacore_launches_per_call.argtypes = [i64, i64]
    lib.hadacore_launches_per_call.restype = ctypes.c_int
    lib.hadacore_launches_per_call_dtype.argtypes = [i64, i64, ctypes.c_int]
    lib.hadacore_launches_per_call_dtype.restype = ctypes.c_int
    _lib = lib
    return lib


def _check(rc: int):
    if rc != 0:
        raise HadacoreError(rc, _load().hadacore_status_string(rc).decode())


def version() -> int:
    return _load().hadacore_version()


def launches_per_call(m: int, n: int, dtype: torch.dtype | None = None) -> int:
    if dtype is None:
        return _load().hadacore_launches_per_call(int(m), int(n))
    return _load().hadacore_launches_per_call_dtype(int(m), int(n), _DTYPES[dtype])


def _shape(x: torch.Tensor):
    if x.dtype not in _DTYPES:
        raise HadacoreError(6, f"dtype {x.dtype} (expected float16, bfloat16 or float32)")
    if x.dim() < 1:
        raise HadacoreError(ARG_ERROR, "need at least one dimension")
    n = x.shape[-1]
    m = x.numel() // n if n else 0
    return m, n


def hadacore_fwht(x: torch.Tensor, out: torch.Tensor | None = None, scale: float | None = None,
                  stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """out[..., :] = scale * H_n x[..., :] on the GPU (scale defaults to 1/sqrt(n)).

    ``out=x`` transforms in place.  Launches on ``stream`` (default: the current
    torch stream of x's device); asynchronous like any CUDA op.
    """
    m, n = _shape(x)
    if not x.is_cuda:
        raise HadacoreError(ARG_ERROR, "x must be a CUDA tensor (use hadacore_fwht_host for host buffers)")
    if not x.is_contiguous():
        raise HadacoreError(ARG_ERROR, "x must be contiguous (row pitch = n; strided views: hadacore_fwht_strided)")
    if out is None:
        out = torch.empty_like(x)
    elif out.shape != x.shape or out.dtype != x.dtype or out.device != x.device or not out.is_contiguous():
        raise HadacoreError(ARG_ERROR, "out must be a contiguous tensor with x's shape, dtype and device")
    if scale is None:
        scale = 1.0 / math.sqrt(n) if n > 0 else 1.0
    with torch.cuda.device(x.device):
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        _check(_load().hadacore_fwht(x.data_ptr(), out.data_ptr(), m, n, _DTYPES[x.dtype], float(scale),
                                     st.cuda_stream))
    return out


fwht = hadacore_fwht


def hadacore_fwht_host(x: torch.Tensor, out: torch.Tensor | None = None, scale: float | None = None,
                       workspace: torch.Tensor | None = None, device=None,
                       stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Host-buffer entry (C: hadacore_fwht_host): H2D, kernel, D2H pipelined in the library.

    ``x``/``out`` are CPU tensors (pin them for full PCIe bandwidth).  ``workspace``
    is a CUDA uint8 tensor (default: 256 MiB, allocated here once per call).
    Returns after the results are in ``out``.
    """
    m, n = _shape(x)
    if x.is_cuda or not x.is_contiguous():
        raise HadacoreError(ARG_ERROR, "x must be a contiguous CPU tensor")
    if out is None:
        out = torch.empty_like(x, pin_memory=x.is_pinned())
    elif out.is_cuda or out.shape != x.shape or out.dtype != x.dtype or not out.is_contiguous():
        raise HadacoreError(ARG_ERROR, "out must be a contiguous CPU tensor with x's shape and dtype")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if workspace is None:
        es = x.element_size()
        workspace = torch.empty(min(256 << 20, max(2 * es * n, 2 * m * n * es)), dtype=torch.uint8, device=dev)
    if scale is None:
        scale = 1.0 / math.sqrt(n) if n > 0 else 1.0
    with torch.cuda.device(workspace.device):
        st = stream if stream is not None else torch.cuda.current_stream(workspace.device)
        _check(_load().hadacore_fwht_host(x.data_ptr(), out.data_ptr(), m, n, _DTYPES[x.dtype], float(scale),
                                          workspace.data_ptr(), workspace.numel(), st.cuda_stream))
    return out


def hadacore_fwht_quant(x: torch.Tensor, qtype: str = "e4m3", scale: float | None = None,
                        out: torch.Tensor | None = None, row_scale: torch.Tensor | None = None,
                        stream: torch.cuda.Stream | None = None):
    """Fused transform + per-row symmetric quantization (C: hadacore_fwht_quant).

    Returns ``(q, row_scale)``: ``q`` has x's shape and dtype float8_e4m3fn ("e4m3")
    or int8 ("int8"), or x's shape with the last dim halved and dtype uint8 ("int4":
    element 2j in the low nibble of byte j, two's complement, codes in [-7, 7]);
    ``row_scale`` is float32 with x's shape minus the last dim, so
    ``codes * row_scale[..., None]`` ~= ``hadacore_fwht(x, scale=scale)``.
    """
    m, n = _shape(x)
    if qtype not in QTYPES:
        raise HadacoreError(6, f"qtype {qtype!r} (expected one of {sorted(QTYPES)})")
    code, qdt = QTYPES[qtype]
    if x.dtype == torch.float32:
        raise HadacoreError(6, "the fused quantization takes float16/bfloat16 inputs")
    if not x.is_cuda or not x.is_contiguous():
        raise HadacoreError(ARG_ERROR, "x must be a contiguous CUDA tensor")
    qshape = x.shape if qtype != "int4" else (*x.shape[:-1], n // 2)
    if out is None:
        out = torch.empty(qshape, dtype=qdt, device=x.device)
    if row_scale is None:
        row_scale = torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device)
    if out.dtype != qdt or tuple(out.shape) != tuple(qshape) or not out.is_contiguous() or out.device != x.device:
        raise HadacoreError(ARG_ERROR, f"out must be a contiguous {qdt} tensor of shape {tuple(qshape)} on x's device")
    if row_scale.dtype != torch.float32 or row_scale.numel() != m or not row_scale.is_contiguous() \
            or row_scale.device != x.device:
        raise HadacoreError(ARG_ERROR, "row_scale must be a contiguous float32 tensor with one entry per row on "
                                       "x's device")
    if scale is None:
        scale = 1.0 / math.sqrt(n) if n > 0 else 1.0
    with torch.cuda.device(x.device):
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        _check(_load().hadacore_fwht_quant(x.data_ptr(), out.data_ptr(), row_scale.data_ptr(), m, n,
                                           _DTYPES[x.dtype], code, float(scale), st.cuda_stream))
    return out, row_scale


def _row_grid(t: torch.Tensor, n: int):
    """Collapse a view's leading dims (dropping size-1 dims) into <= 2 strided row dims:
    (m_outer, m_inner, stride_outer, stride_inner) in elements."""
    dims = [(s, st) for s, st in zip(t.shape[:-1], t.stride()[:-1]) if s != 1]
    merged = []
    for size, st in dims:
        if merged and merged[-1][1] == st * size:
            merged[-1] = (merged[-1][0] * size, st)
        else:
            merged.append((size, st))
    if len(merged) > 2:
        raise HadacoreError(ARG_ERROR, "more than two non-collapsible row dimensions")
    while len(merged) < 2:
        merged.insert(0, (1, n * (merged[0][0] if merged else 1)))
    (mo, so), (mi, si) = merged
    return mo, mi, so, si


def hadacore_fwht_strided(x: torch.Tensor, out: torch.Tensor | None = None, scale: float | None = None,
                          stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Transform the last dimension of a strided view (C: hadacore_fwht_strided).

    ``x`` may be any CUDA view whose last dimension n is contiguous and whose
    leading dimensions collapse to at most two strided row dimensions, e.g.
    ``qkv[:, 0]`` of a ``[tokens, 3, H, d]`` projection (rows = tokens x H).
    ``out=x`` transforms the view in place (the rest of the buffer is untouched);
    by default the result is a new contiguous tensor.
    """
    m, n = _shape(x)
    if not x.is_cuda or x.stride(-1) != 1:
        raise HadacoreError(ARG_ERROR, "x must be a CUDA view with a contiguous last dimension")
    if out is None:
        out = torch.empty(x.shape, dtype=x.dtype, device=x.device)
    if out.shape != x.shape or out.dtype != x.dtype or out.stride(-1) != 1 or out.device != x.device:
        raise HadacoreError(ARG_ERROR, "out must have x's shape, dtype and device and a contiguous last dimension")

    mo, mi, so, si = _row_grid(x, n)
    if out.is_contiguous():  # rows in (i, j) order: any grid maps onto it
        mo2, mi2, oso, osi = mo, mi, mi * n, n
    else:
        mo2, mi2, oso, osi = _row_grid(out, n)
    if (mo2, mi2) != (mo, mi):
        raise HadacoreError(ARG_ERROR, "out's row grid differs from x's")
    if scale is None:
        scale = 1.0 / math.sqrt(n) if n > 0 else 1.0
    with torch.cuda.device(x.device):
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        _check(_load().hadacore_fwht_strided(x.data_ptr(), out.data_ptr(), mo, mi, so, si, oso, osi, n,
                                             _DTYPES[x.dtype], float(scale), st.cuda_stream))
    return out


def fake_quant(x: torch.Tensor, qtype: str = "int4", per_tensor: bool = False, out: torch.Tensor | None = None,
               stream: torch.cuda.Stream | None = None):
    """Symmetric quantize -> dequantize of fp32 rows (C: hadacore_fake_quant; quant lab).

    Returns ``(out, row_amax)``: ``out`` fp32 like ``x``; ``row_amax`` the per-row max
    |x| (per_tensor: the matrix max in every entry); the scale used is row_amax / Q.
    """
    m, n = _shape(x)
    if qtype not in LAB_QTYPES:
        raise HadacoreError(6, f"qtype {qtype!r} (expected one of {sorted(LAB_QTYPES)})")
    if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous():
        raise HadacoreError(ARG_ERROR, "x must be a contiguous float32 CUDA tensor")
    if out is None:
        out = torch.empty_like(x)
    amax = torch.empty(max(m, 1), dtype=torch.float32, device=x.device)
    with torch.cuda.device(x.device):
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        _check(_load().hadacore_fake_quant(x.data_ptr(), out.data_ptr(), amax.data_ptr(), m, n, LAB_QTYPES[qtype],
                                           int(bool(per_tensor)), st.cuda_stream))
    return out, amax[:m]


def row_sq_error(a: torch.Tensor, b: torch.Tensor, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Per-row sum of squared differences of two fp32 CUDA matrices, fp64 (C: hadacore_row_sq_error)."""
    m, n = _shape(a)
    if a.shape != b.shape or a.dtype != torch.float32 or b.dtype != torch.float32 or not (a.is_cuda and b.is_cuda) \
            or not (a.is_contiguous() and b.is_contiguous()):
        raise HadacoreError(ARG_ERROR, "a, b must be contiguous float32 CUDA tensors of one shape")
    out = torch.empty(max(m, 1), dtype=torch.float64, device=a.device)
    with torch.cuda.device(a.device):
        st = stream if stream is not None else torch.cuda.current_stream(a.device)
        _check(_load().hadacore_row_sq_error(a.data_ptr(), b.data_ptr(), out.data_ptr(), m, n, st.cuda_stream))
    return out[:m]


def hadacore_fwht_quant_strided(x: torch.Tensor, qtype: str = "e4m3", scale: float | None = None,
                                out: torch.Tensor | None = None, row_scale: torch.Tensor | None = None,
                                stream: torch.cuda.Stream | None = None):
    """Transform + per-row quantization of a strided view (C: hadacore_fwht_quant_strided), e.g.
    ``qkv[:, 0:2]`` of a ``[tokens, 3, H, d]`` projection: the Q and K heads rotated and quantized
    in one pass (FP8 attention).  Returns contiguous ``(q, row_scale)`` with the view's row shape:
    ``q`` [..., n] (``[..., n/2]`` uint8 for "int4"), ``row_scale`` [...] float32; x is not modified."""
    m, n = _shape(x)
    if qtype not in QTYPES:
        raise HadacoreError(6, f"qtype {qtype!r} (expected one of {sorted(QTYPES)})")
    if not x.is_cuda or x.stride(-1) != 1:
        raise HadacoreError(ARG_ERROR, "x must be a CUDA view with a contiguous last dimension")
    code, qdt = QTYPES[qtype]
    qshape = (*x.shape[:-1], n // 2 if qtype == "int4" else n)
    q = out if out is not None else torch.empty(qshape, dtype=qdt, device=x.device)
    rs = row_scale if row_scale is not None else torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device)
    if q.dtype != qdt or q.numel() != m * qshape[-1] or not q.is_contiguous() or q.device != x.device:
        raise HadacoreError(ARG_ERROR, f"out must be a contiguous {qdt} tensor of {m * qshape[-1]} elements on x's device")
    if rs.dtype != torch.float32 or rs.numel() != m or not rs.is_contiguous() or rs.device != x.device:
        raise HadacoreError(ARG_ERROR, "row_scale must be a contiguous float32 tensor with one entry per row on "
                                       "x's device")
    mo, mi, so, si = _row_grid(x, n)
    if scale is None:
        scale = 1.0 / math.sqrt(n) if n > 0 else 1.0
    with torch.cuda.device(x.device):
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        _check(_load().hadacore_fwht_quant_strided(x.data_ptr(), q.data_ptr(), rs.data_ptr(), mo, mi, so, si, n,
                                                   _DTYPES[x.dtype], code, float(scale), st.cuda_stream))
    return q, rs
