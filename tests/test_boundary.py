"""C-ABI boundary checks that need no GPU: the library builds and loads, exports
every function declared in include/hadacore.h, and validates arguments before
any CUDA call (include/hadacore.h "Errors")."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2412_08832_b200 as hc
from paper_2412_08832_b200 import build as hc_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hadacore.h")

OK, INVALID_N, INVALID_M, NULL, MISALIGNED, OVERLAP, DTYPE, SCALE, CUDA, WORKSPACE = range(10)


@pytest.fixture(scope="module")
def lib():
    hc_build.build()
    return hc._load()


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[A-Za-z_][A-Za-z0-9_]*\s*\*?\s+)+\**(hadacore_[a-z_]+)\s*\(", text, re.M)))


def test_header_declares_expected_entry_points():
    assert declared_functions() == sorted(["hadacore_fwht", "hadacore_fwht_host", "hadacore_fwht_quant",
                                           "hadacore_fwht_strided", "hadacore_fake_quant", "hadacore_row_sq_error",
                                           "hadacore_fwht_quant_strided",
                                           "hadacore_status_string", "hadacore_version",
                                           "hadacore_launches_per_call", "hadacore_launches_per_call_dtype"])


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", hc.library_path()], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\s[TW]\s+(hadacore_\w+)", out))
    for name in declared_functions():
        assert name in exported, name
        assert getattr(lib, name) is not None


def test_library_targets_sm100a_only(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", hc.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", hc.library_path()], capture_output=True, text=True).stdout
    assert "HMMA.16816" in sass          # tensor-core contractions
    assert "UTMALDG.3D" in sass          # 3-D TMA tensor loads of (n, rows, outer) boxes (n <= 256)
    assert "UTMALDG.5D" in sass and "UTMASTG.5D" in sass  # 5-D TMA tensor load/store, SWIZZLE_128B (n >= 512)
    assert "UGETNEXTWORKID" in sass      # cluster launch control work stealing
    assert "LDSM.16.MT88.4" in sass and "STSM.16.MT88.4" in sass  # cross-chunk exchange


def call(lib, in_ptr, out_ptr, m, n, dtype=0, scale=1.0):
    return lib.hadacore_fwht(in_ptr, out_ptr, m, n, dtype, scale, None)


def test_validation_codes(lib):
    a, b = 0x10000, 0x8000000
    assert call(lib, a, b, 4, 100) == INVALID_N
    assert call(lib, a, b, 4, 1) == INVALID_N       # n = 2..2^15 (NEXT-2 widened the paper's 2^7 floor)
    assert call(lib, a, b, 4, 3) == INVALID_N
    assert call(lib, a, b, 4, 96) == INVALID_N
    assert call(lib, a, b, 4, 65536) == INVALID_N
    assert call(lib, a, b, 4, 0) == INVALID_N
    assert call(lib, a, b, 4, -128) == INVALID_N
    for n in (2, 4, 8, 16, 32, 64):                 # accepted: m == 0 is a no-op without a GPU
        assert call(lib, None, None, 0, n) == OK
        assert call(lib, a + 8, b, 4, n) == MISALIGNED
        assert call(lib, a, a + 16, 64, n) == OVERLAP
    assert call(lib, a, b, -1, 256) == INVALID_M
    assert call(lib, a, b, 1 << 62, 256) == INVALID_M
    assert call(lib, a, b, 4, 256, dtype=3) == DTYPE
    assert call(lib, a, b, 4, 256, dtype=-1) == DTYPE
    assert call(lib, a, b, 4, 256, scale=float("nan")) == SCALE
    assert call(lib, a, b, 4, 256, scale=float("inf")) == SCALE
    assert call(lib, a, b, 4, 256, scale=0.0) == SCALE              # scale > 0
    assert call(lib, a, b, 4, 256, scale=-0.0) == SCALE
    assert call(lib, a, b, 4, 256, scale=-0.5) == SCALE
    assert call(lib, a, b, 4, 64, scale=-1.0) == SCALE
    assert call(lib, None, b, 4, 256) == NULL
    assert call(lib, a, None, 4, 256) == NULL
    assert call(lib, a + 8, b, 4, 256) == MISALIGNED
    assert call(lib, a, b + 2, 4, 256) == MISALIGNED
    assert call(lib, a, a + 512, 4, 256) == OVERLAP      # partial overlap
    assert call(lib, a + 512, a, 4, 256) == OVERLAP
    # m == 0 is a successful no-op (no CUDA call, works without a GPU)
    assert call(lib, None, None, 0, 256) == OK
    assert call(lib, a, b, 0, 32768, dtype=1) == OK


def test_host_entry_validation(lib):
    a, b, ws = 0x10000, 0x8000000, 0x20000000
    f = lib.hadacore_fwht_host
    assert f(a, b, 4, 100, 0, 1.0, ws, 1 << 20, None) == INVALID_N
    assert f(a, b, 4, 256, 0, 1.0, None, 1 << 20, None) == WORKSPACE
    assert f(a, b, 4, 256, 0, 1.0, ws, 1000, None) == WORKSPACE     # < two rows
    assert f(a, b, 4, 256, 0, 1.0, ws + 4, 1 << 20, None) == WORKSPACE
    assert f(a, a + 2, 4, 256, 0, 1.0, ws, 1 << 20, None) == OVERLAP
    assert f(a, b, 4, 256, 0, 0.0, ws, 1 << 20, None) == SCALE
    assert f(None, None, 0, 256, 0, 1.0, None, 0, None) == OK


def test_quant_entry_validation(lib):
    a, q, rs = 0x10000, 0x8000000, 0x20000000
    f = lib.hadacore_fwht_quant
    assert f(a, q, rs, 4, 256, 0, 3, 1.0, None) == DTYPE          # unknown qtype
    assert f(a, a + 512, rs, 4, 256, 0, 2, 1.0, None) == OVERLAP   # int4 codes inside the input
    assert f(a, q, rs, 4, 256, 3, 0, 1.0, None) == DTYPE          # unknown dtype
    assert f(a, q, rs, 4, 100, 0, 0, 1.0, None) == INVALID_N
    assert f(a, q, rs, 4, 1, 0, 0, 1.0, None) == INVALID_N       # fused quantization: n = 2..2^15
    assert f(a, q, rs, 4, 65536, 0, 0, 1.0, None) == INVALID_N
    assert f(a, q, rs, 4, 256, 0, 1, float("nan"), None) == SCALE
    assert f(a, q, rs, 4, 256, 0, 0, 0.0, None) == SCALE            # scale > 0
    assert f(a, q, rs, 4, 256, 0, 2, -1.0, None) == SCALE
    assert f(a, q, rs, 4, 16, 1, 0, -0.25, None) == SCALE
    assert f(a, None, rs, 4, 256, 0, 0, 1.0, None) == NULL
    assert f(a, q, None, 4, 256, 0, 0, 1.0, None) == NULL
    assert f(a, q + 8, rs, 4, 256, 0, 0, 1.0, None) == MISALIGNED
    assert f(a, q, rs + 2, 4, 256, 0, 0, 1.0, None) == MISALIGNED
    assert f(a, a + 1024, rs, 4, 256, 0, 0, 1.0, None) == OVERLAP  # codes inside the input
    assert f(a, q, a + 64, 4, 256, 0, 0, 1.0, None) == OVERLAP     # scales inside the input
    assert f(a, q, q + 256, 4, 256, 0, 0, 1.0, None) == OVERLAP    # scales inside the codes
    assert f(None, None, None, 0, 256, 1, 1, 1.0, None) == OK


def test_status_strings_and_version(lib):
    for code in range(10):
        s = lib.hadacore_status_string(code)
        assert s and len(s) > 1
    assert lib.hadacore_status_string(1234) == b"unknown status"
    assert lib.hadacore_version() >= 100
    assert lib.hadacore_launches_per_call(0, 256) == 0
    assert lib.hadacore_launches_per_call(10, 256) == 1
    assert lib.hadacore_launches_per_call(10, 100) == 0
    assert lib.hadacore_launches_per_call(10, 2) == 1
    assert lib.hadacore_launches_per_call_dtype(10, 32768, 2) == 1     # fp32 n = 2^15: one cluster launch
    assert lib.hadacore_launches_per_call_dtype(10, 32768, 1) == 1
    assert lib.hadacore_launches_per_call_dtype(0, 32768, 2) == 0


def test_python_binding_rejects_without_fallback():
    import torch
    x = torch.zeros(4, 256, dtype=torch.float16)
    with pytest.raises(hc.HadacoreError):
        hc.hadacore_fwht(x)                    # CPU tensor: no CPU fallback
    with pytest.raises(hc.HadacoreError):
        hc.hadacore_fwht(torch.zeros(4, 256, dtype=torch.float64))


def test_product_path_does_not_import_oracle():
    """The CUDA path and the oracle share no code: nothing under the product package
    imports, links or opens oracle/ (task rule 3)."""
    pkg = os.path.join(ROOT, "paper_2412_08832_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "liboracle", "fwht_oracle", "oracle_fwht"):
                    assert bad not in text, (f, bad)


def test_strided_entry_validation(lib):
    a, b = 0x10000, 0x80000000
    f = lib.hadacore_fwht_strided
    # (in, out, m_outer, m_inner, in_so, in_si, out_so, out_si, n, dtype, scale, stream)
    assert f(a, b, 4, 3, 1004, 128, 384, 128, 128, 0, 1.0, None) == INVALID_M       # stride not multiple of 8
    assert f(a, b, 4, 3, 384, 64, 384, 128, 128, 0, 1.0, None) == INVALID_M         # inner rows overlap
    assert f(a, b, 4, 3, 256, 128, 384, 128, 128, 0, 1.0, None) == INVALID_M        # outer rows overlap
    assert f(a, b, 4, 3, 384, 128, 384, 128, 100, 0, 1.0, None) == INVALID_N
    assert f(a, b, 4, 3, 384, 128, 384, 128, 4, 0, 1.0, None) == INVALID_N    # row grids: n >= 8 (16-byte TMA rows)
    assert f(a, b, 0, 3, 384, 128, 384, 128, 64, 0, 1.0, None) == OK          # n = 8..64 accepted (m_outer = 0)
    assert f(a, b, 4, 3, 384, 128, 384, 128, 128, 2, 1.0, None) == DTYPE            # fp32: contiguous API only
    assert f(a, a, 4, 3, 384, 128, 768, 128, 128, 0, 1.0, None) == OVERLAP          # in place needs equal strides
    assert f(a, a + 256, 4, 3, 384, 128, 384, 128, 128, 0, 1.0, None) == OVERLAP    # extents overlap
    assert f(a + 2, b, 4, 3, 384, 128, 384, 128, 128, 0, 1.0, None) == MISALIGNED
    assert f(None, None, 0, 3, 384, 128, 384, 128, 128, 0, 1.0, None) == OK
    assert f(a, b, 4, 3, 384, 128, 384, 128, 128, 0, 0.0, None) == SCALE
    assert f(a, b, 4, 3, 384, 128, 384, 128, 128, 0, -2.0, None) == SCALE


def test_lab_entry_validation(lib):
    a, b, s = 0x10000, 0x8000000, 0x20000000
    f = lib.hadacore_fake_quant
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                  ctypes.c_int, ctypes.c_void_p]
    assert f(a, b, s, 4, 256, 3, 0, None) == DTYPE            # qtype outside {E4M3, INT8, INT4}
    assert f(a, b, s, 4, 100, 2, 0, None) == INVALID_N
    assert f(a, b, s, -1, 256, 2, 0, None) == INVALID_M
    assert f(None, b, s, 4, 256, 2, 0, None) == NULL
    assert f(a, b, None, 4, 256, 2, 0, None) == NULL
    assert f(a + 4, b, s, 4, 256, 2, 0, None) == MISALIGNED
    assert f(a, a + 16, s, 4, 256, 2, 0, None) == OVERLAP
    assert f(a, b, a + 16, 4, 256, 2, 1, None) == OVERLAP
    assert f(None, None, None, 0, 256, 2, 0, None) == OK
    g = lib.hadacore_row_sq_error
    g.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
    assert g(a, b, s, 4, 0, None) == INVALID_N
    assert g(a, b, s + 4, 4, 16, None) == MISALIGNED
    assert g(None, b, s, 4, 16, None) == NULL
    assert g(None, None, None, 0, 16, None) == OK


def test_quant_strided_entry_validation(lib):
    a, q, rs = 0x10000, 0x8000000, 0x20000000
    f = lib.hadacore_fwht_quant_strided
    assert f(a, q, rs, 4, 3, 384, 128, 128, 0, 3, 1.0, None) == DTYPE        # qtype
    assert f(a, q, rs, 4, 3, 384, 128, 128, 2, 0, 1.0, None) == DTYPE        # fp32 input
    assert f(a, q, rs, 4, 3, 384, 128, 4, 0, 0, 1.0, None) == INVALID_N      # n >= 8 (16-byte TMA rows)
    assert f(a, q, rs, 4, 3, 384, 64, 128, 0, 0, 1.0, None) == INVALID_M     # inner rows overlap
    assert f(a, q, rs, 4, 3, 384, 128, 128, 0, 0, float("inf"), None) == SCALE
    assert f(a, q, rs, 4, 3, 384, 128, 128, 0, 0, 0.0, None) == SCALE
    assert f(a, q, rs, 4, 3, 384, 128, 128, 0, 0, -1.0, None) == SCALE
    assert f(a, None, rs, 4, 3, 384, 128, 128, 0, 0, 1.0, None) == NULL
    assert f(a + 8, q, rs, 4, 3, 384, 128, 128, 0, 0, 1.0, None) == MISALIGNED
    assert f(a, a + 256, rs, 4, 3, 384, 128, 128, 0, 0, 1.0, None) == OVERLAP
    assert f(a, q, rs, 0, 3, 384, 128, 128, 0, 0, 1.0, None) == OK
