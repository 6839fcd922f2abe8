"""fp64 CPU oracle for HadaCore's batched normalized Walsh-Hadamard transform.

TEST INFRASTRUCTURE ONLY -- only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
package.  The product path (``paper_2412_08832_b200``) never imports it, and this
package never imports the product path: the two share no code, header, table or
constant generator.  Only the seeded input generators (``synthetic/``, which
holds none of the method's arithmetic) serve both.

The arithmetic lives in plain C (``fwht_oracle.c``, fp64, compiled here with gcc)
and follows /root/reference/PAPER.md:

* ``fwht``        -- the FWHT listing, P:50-64 [Sec. 2.2], scale applied once at
                     the end (reading R3).
* ``dense_entry`` -- the definition y_l = scale * sum_j (-1)^popcount(j&l) x_j,
                     P:41 [Sec. 2.1] + Sylvester's construction P:45 [Sec. 2.2].
* ``dense``       -- the definition for a whole (small) matrix.
* ``quantize`` / ``fake_quant`` / ``lab_trial`` -- symmetric quantization and the
                     rotated-vs-plain quantization-error trial of SPEC's quant_lab
                     (the paper's motivation P:24 [Sec. 1], P:180
                     [Sec. 4.2]), in fp64.

Parity status: pinned (see tests/test_oracle.py and DESIGN.md "Oracle pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fwht_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle in-tree (gcc -O2, no fast-math: IEEE fp64)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-std=c11",
                               "-fno-fast-math", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_fwht_f64.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_int]
        lib.oracle_fwht_f64.restype = ctypes.c_int
        lib.oracle_dense_f64.argtypes = [dp, dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double]
        lib.oracle_dense_f64.restype = ctypes.c_int
        lib.oracle_dense_entry_f64.argtypes = [dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double]
        lib.oracle_dense_entry_f64.restype = ctypes.c_double
        lib.oracle_e4m3_value.argtypes = [ctypes.c_int]
        lib.oracle_e4m3_value.restype = ctypes.c_double
        lib.oracle_e4m3_encode.argtypes = [ctypes.c_double]
        lib.oracle_e4m3_encode.restype = ctypes.c_int
        lib.oracle_quantize_rows_f64.argtypes = [dp, ctypes.POINTER(ctypes.c_uint8), dp, ctypes.c_int64,
                                                 ctypes.c_int64, ctypes.c_int]
        lib.oracle_quantize_rows_f64.restype = ctypes.c_int
        lib.oracle_quantize_f64.argtypes = [dp, ctypes.POINTER(ctypes.c_uint8), dp, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        lib.oracle_quantize_f64.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _as_f64_2d(x) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if a.ndim == 1:
        a = a[None, :]
    if a.ndim != 2:
        raise ValueError("oracle expects a 2-D (m, n) matrix")
    return a


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def fwht(x, scale: float | None = None, threads: int | None = None) -> np.ndarray:
    """y[i,:] = scale * H_n x[i,:] in fp64 via the P:50-64 listing (scale once at end).

    ``scale`` defaults to 1/sqrt(n) (the normalized transform).
    """
    a = _as_f64_2d(x)
    m, n = a.shape
    if scale is None:
        scale = 1.0 / np.sqrt(n)
    out = np.empty_like(a)
    rc = _load().oracle_fwht_f64(_ptr(a), _ptr(out), m, n, float(scale),
                                 int(threads or default_threads()))
    if rc != 0:
        raise ValueError(f"oracle_fwht_f64 rejected m={m} n={n}")
    return out


def dense(x, scale: float | None = None) -> np.ndarray:
    """The definition (O(m n^2)): y_l = scale * sum_j (-1)^popcount(j&l) x_j."""
    a = _as_f64_2d(x)
    m, n = a.shape
    if scale is None:
        scale = 1.0 / np.sqrt(n)
    out = np.empty_like(a)
    if _load().oracle_dense_f64(_ptr(a), _ptr(out), m, n, float(scale)) != 0:
        raise ValueError(f"oracle_dense_f64 rejected m={m} n={n}")
    return out


def dense_entry(row, l: int, scale: float | None = None) -> float:
    """One output of the definition for one row: scale * sum_j (-1)^popcount(j&l) row_j."""
    a = np.ascontiguousarray(np.asarray(row, dtype=np.float64).reshape(-1))
    n = a.shape[0]
    if scale is None:
        scale = 1.0 / np.sqrt(n)
    return float(_load().oracle_dense_entry_f64(_ptr(a), n, int(l), float(scale)))


QTYPES = {"e4m3": 0, "int8": 1, "int4": 2}
QMAX = {"e4m3": 448.0, "int8": 127.0, "int4": 7.0}


def e4m3_value(code: int) -> float:
    """Value of an FP8 E4M3 (OCP e4m3fn) code, fp64."""
    return _load().oracle_e4m3_value(int(code))


def e4m3_encode(x: float) -> int:
    """Nearest-even E4M3 code of x, saturating at +-448."""
    return _load().oracle_e4m3_encode(float(x))


def quantize_rows(y, qtype: str):
    """Per-row symmetric quantization of transformed rows.

    Returns (codes uint8 (m, n), scales float64 (m,)): scale = max|y|/Q (Q = 448 for
    e4m3, 127 for int8; 1 for an all-zero row), codes = round(y / scale).
    """
    a = _as_f64_2d(y)
    m, n = a.shape
    codes = np.empty((m, n), dtype=np.uint8)
    scales = np.empty(m, dtype=np.float64)
    rc = _load().oracle_quantize_rows_f64(_ptr(a), codes.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                                          _ptr(scales), m, n, QTYPES[qtype])
    if rc != 0:
        raise ValueError("oracle_quantize_rows_f64 rejected its arguments")
    return codes, scales


def quantize(y, qtype: str, per_tensor: bool = False):
    """Symmetric quantization, SPEC quant_lab S:419-427: scale = max_abs / Q (Q = 448,
    127, 7 for e4m3, int8, int4), codes = round(y / scale) (ties to even; e4m3 by
    enumeration, saturating; integers clamped to +-Q); max_abs per row or over the
    whole matrix (per_tensor, the scale then repeated per row); all-zero -> scale 1.
    Returns (codes uint8 (m, n), scales float64 (m,))."""
    a = _as_f64_2d(y)
    m, n = a.shape
    codes = np.empty((m, n), dtype=np.uint8)
    scales = np.empty(m, dtype=np.float64)
    rc = _load().oracle_quantize_f64(_ptr(a), codes.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                                     _ptr(scales), m, n, QTYPES[qtype], int(bool(per_tensor)))
    if rc != 0:
        raise ValueError("oracle_quantize_f64 rejected its arguments")
    return codes, scales


def fake_quant(x, qtype: str, per_tensor: bool = False) -> np.ndarray:
    """quantize -> dequantize (SPEC S:419 'dequantize multiplies back'), fp64."""
    codes, scales = quantize(x, qtype, per_tensor)
    return dequantize_rows(codes, scales, qtype)


def lab_trial(x, qtype: str, per_tensor: bool = False) -> dict:
    """One trial of SPEC's run_experiment, in fp64 on the original x:
    (a) plain: fake-quantize x -> mse_plain; (b) rotated: y = H x (normalized,
    P:41), fake-quantize y, inverse-rotate with H again (involution) -> mse_rotated;
    max_abs of x and of y."""
    a = _as_f64_2d(x)
    y = fwht(a)
    back = fwht(fake_quant(y, qtype, per_tensor))
    plain = fake_quant(a, qtype, per_tensor)
    return {"mse_plain": float(np.mean((plain - a) ** 2)), "mse_rotated": float(np.mean((back - a) ** 2)),
            "max_abs_plain": float(np.abs(a).max()), "max_abs_rotated": float(np.abs(y).max())}


def dequantize_rows(codes, scales, qtype: str) -> np.ndarray:
    """codes (m, n) uint8 and per-row scales -> fp64 values."""
    codes = np.asarray(codes, dtype=np.uint8)
    if qtype in ("int8", "int4"):
        v = codes.view(np.int8).astype(np.float64)
    else:
        table = np.array([e4m3_value(c) for c in range(256)])
        v = table[codes]
    return v * np.asarray(scales, dtype=np.float64)[:, None]
