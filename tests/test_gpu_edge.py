"""Edge readings and test hygiene (VERDICT r1 "Test hygiene"; R13, R14):

* R13 non-finite rows, element by element against the fp64 oracle: where the oracle is NaN
  the GPU is NaN; where the oracle is +-Inf the GPU is the same-signed Inf or NaN (the
  structural zeros of the I (x) H tiles, turn 0 * Inf into NaN); rows without
  non-finite inputs are unaffected.  Fused quantization: the row scale is non-finite, NaN
  wherever the oracle's max |y| is NaN.
* R14 subnormal rows: the per-row 2-norm error bound derived in DESIGN.md from the
  16-bit roundings of the pipeline, ||y_gpu - y||_2 <= (R/2) (u sqrt(n) + eps ||x||_2),
  u = the dtype's subnormal spacing, eps its machine epsilon, R the roundings of a row.
* Canary borders: guard bytes around every contiguous output (n = 2..2^15 transform,
  fp32, and fused-quantization codes + row scales) stay untouched.
* Negative control: libhadacore_negctl.so (the same source built with -DHC_NEGCTL: one
  sign of the H_16 constant flipped) must FAIL the parity check, so
  the parity tests are shown to be able to fail.
"""
import ctypes
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

NS_ALL = [1 << k for k in range(1, 16)]
NS = [1 << k for k in range(7, 16)]
DTYPES = [torch.float16, torch.bfloat16]
TOL = {torch.float16: 2e-3, torch.bfloat16: 1.6e-2, torch.float32: 1e-5}


@pytest.fixture(scope="module")
def hc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_08832_b200 as hc
    hc._load()
    return hc


def widen(t):
    return t.detach().cpu().to(torch.float64).numpy()


def rel_l2_rows(got, ref):
    den = np.linalg.norm(ref, axis=1)
    return np.linalg.norm(got - ref, axis=1) / np.where(den == 0, 1.0, den)


# ---------------------------------------------------------------- R13: non-finite rows
def nonfinite_rows(n, dtype):
    g = synthetic.normal_block(0, 6, n, 4242)
    rows = []
    a = g[0].clone(); a[n // 3] = float("inf"); rows.append(a)                       # lone +Inf
    b = g[1].clone(); b[n // 5] = float("-inf"); rows.append(b)                      # lone -Inf
    c = g[2].clone(); c[0] = float("nan"); rows.append(c)                            # lone NaN
    d = g[3].clone(); d[n // 2] = float("inf"); d[n - 1] = float("-inf"); rows.append(d)  # +Inf and -Inf
    e = g[4].clone(); e[1] = float("inf"); e[n - 2] = float("inf"); rows.append(e)   # two +Inf
    f = g[5].clone(); f[:] = float("inf"); rows.append(f)                            # all +Inf
    return torch.stack(rows).to(dtype)


def check_classification(y, ref):
    """Element-wise R13 rule; returns the fraction of oracle-Inf positions that came out NaN."""
    nan_ref, inf_ref = np.isnan(ref), np.isinf(ref)
    assert np.all(np.isnan(y[nan_ref])), "oracle NaN must be GPU NaN"
    yi, ri = y[inf_ref], ref[inf_ref]
    assert np.all(np.isnan(yi) | (yi == ri)), "oracle +-Inf must be GPU NaN or the same-signed Inf"
    assert not np.any(np.isfinite(y[~np.isfinite(ref)]))
    return float(np.mean(np.isnan(yi))) if yi.size else 0.0


@pytest.mark.parametrize("dtype", DTYPES + [torch.float32], ids=["fp16", "bf16", "fp32"])
@pytest.mark.parametrize("n", NS_ALL)
def test_r13_nonfinite_classification(hc, n, dtype):
    fin = synthetic.generate(8, n, dtype, 4343)
    nf = nonfinite_rows(n, dtype) if n > 2 else nonfinite_rows(4, dtype)[:, :2].contiguous()
    x = torch.cat([fin[:4], nf, fin[4:]]).contiguous()
    y = widen(hc.hadacore_fwht(x.cuda()))
    ref = oracle.fwht(widen(x))
    k = nf.shape[0]
    check_classification(y[4:4 + k], ref[4:4 + k])
    # finite rows around them are unaffected (rows never share a contraction)
    fr = np.r_[0:4, 4 + k:8 + k]
    assert np.all(np.isfinite(y[fr]))
    assert rel_l2_rows(y[fr], ref[fr]).max() <= TOL[dtype]


@pytest.mark.parametrize("qtype", ["e4m3", "int8", "int4"])
@pytest.mark.parametrize("n", [4, 16, 64, 128, 256, 1024, 8192, 32768])
def test_r13_quant_row_scale(hc, n, qtype):
    """R23: a row with a non-finite input gets a non-finite row scale -- NaN wherever the
    oracle's max |y| is NaN; finite rows' scales are unaffected."""
    fin = synthetic.generate(4, n, torch.bfloat16, 4444)
    nf = nonfinite_rows(max(n, 4), torch.bfloat16)[:, :n].contiguous()
    x = torch.cat([fin[:2], nf, fin[2:]]).contiguous()
    q, s = hc.hadacore_fwht_quant(x.cuda(), qtype)
    s = s.cpu().double().numpy()
    ref = oracle.fwht(widen(x))
    k = nf.shape[0]
    amax = np.array([np.max(np.abs(r)) if not np.any(np.isnan(r)) else np.nan for r in ref])
    for i in range(2, 2 + k):
        assert not np.isfinite(s[i]), i
        if np.isnan(amax[i]):
            assert np.isnan(s[i]), i
    for i in (0, 1, 2 + k, 3 + k):
        assert np.isfinite(s[i]) and abs(s[i] - amax[i] / {"e4m3": 448, "int8": 127, "int4": 7}[qtype]) <= \
            TOL[torch.bfloat16] * s[i]


# ---------------------------------------------------------------- R14: subnormal rows
def roundings(n):
    """16-bit roundings a row goes through on the transform path (R14): n < 128 --
    fp32 register butterflies, one final rounding; n = 128, 256 -- one 16-bit intermediate
    after the first H_16 stage + the final; n >= 512 -- two (after each H_16 of H_256) + the final."""
    return 1 if n < 128 else (2 if n <= 256 else 3)


@pytest.mark.parametrize("dtype", DTYPES, ids=["fp16", "bf16"])
@pytest.mark.parametrize("n", NS_ALL)
def test_r14_subnormal_rows_derived_bound(hc, n, dtype):
    fi = torch.finfo(dtype)
    u = fi.tiny * fi.eps  # subnormal spacing (2^-24 fp16, 2^-133 bf16)
    rows = []
    for seed in range(4):
        g = synthetic.normal_block(0, 1, n, 777 + seed)[0]
        rows.append(g * (fi.tiny / 8.0))                     # mostly subnormal
        rows.append(g * (fi.tiny / 512.0))                   # a few spacings
    x = torch.stack(rows).to(dtype)
    xs = widen(x)
    assert np.any(np.abs(xs[np.nonzero(xs)]) < fi.tiny)    # the rows really are subnormal
    y = widen(hc.hadacore_fwht(x.cuda()))
    ref = oracle.fwht(xs)
    err = np.linalg.norm(y - ref, axis=1)
    bound = roundings(n) / 2.0 * (u * math.sqrt(n) + fi.eps * np.linalg.norm(xs, axis=1))
    assert np.all(err <= bound), (err / bound).max()
    # and the result is not flushed to zero: rows whose exact result is well above the
    # bound keep their magnitude (rows at the spacing level may legitimately round to 0)
    big = np.linalg.norm(ref, axis=1) > 4 * bound
    assert big.sum() >= 4
    assert np.all(np.linalg.norm(y[big], axis=1) >= 0.5 * np.linalg.norm(ref[big], axis=1))


# ---------------------------------------------------------------- canary borders
GUARD = 4096  # bytes of canary on each side


@pytest.mark.parametrize("dtype", DTYPES + [torch.float32], ids=["fp16", "bf16", "fp32"])
@pytest.mark.parametrize("n", NS_ALL)
def test_canary_transform_outputs(hc, n, dtype):
    es = torch.tensor([], dtype=dtype).element_size()
    rows = {2: 8193, 4: 4099, 8: 2051, 16: 1031}.get(n, max(3, (1 << 18) // n) + 1)
    x = synthetic.generate(rows, n, dtype, 4545).cuda()
    nbytes = rows * n * es
    buf = torch.full((GUARD + nbytes + GUARD,), 0xA5, dtype=torch.uint8, device="cuda")
    out = buf[GUARD: GUARD + nbytes].view(dtype).view(rows, n)
    hc.hadacore_fwht(x, out=out)
    torch.cuda.synchronize()
    assert torch.all(buf[:GUARD] == 0xA5) and torch.all(buf[GUARD + nbytes:] == 0xA5)
    assert rel_l2_rows(widen(out), oracle.fwht(widen(x))).max() <= TOL[dtype]


@pytest.mark.parametrize("qtype", ["e4m3", "int8", "int4"])
@pytest.mark.parametrize("n", NS_ALL)
def test_canary_quant_codes_and_scales(hc, n, qtype):
    rows = {2: 8193, 4: 4099, 8: 2051, 16: 1031}.get(n, max(3, (1 << 18) // n) + 1)
    x = synthetic.generate(rows, n, torch.float16, 4646, dist="D1").cuda()
    cb = n // 2 if qtype == "int4" else n
    qbytes, sbytes = rows * cb, rows * 4
    qbuf = torch.full((GUARD + qbytes + GUARD,), 0x5A, dtype=torch.uint8, device="cuda")
    sbuf = torch.full((GUARD + sbytes + GUARD,), 0x3C, dtype=torch.uint8, device="cuda")
    qv = qbuf[GUARD: GUARD + qbytes].view(rows, cb)
    qv = qv.view(torch.float8_e4m3fn) if qtype == "e4m3" else (qv.view(torch.int8) if qtype == "int8" else qv)
    sv = sbuf[GUARD: GUARD + sbytes].view(torch.float32)
    hc.hadacore_fwht_quant(x, qtype=qtype, out=qv, row_scale=sv)
    torch.cuda.synchronize()
    assert torch.all(qbuf[:GUARD] == 0x5A) and torch.all(qbuf[GUARD + qbytes:] == 0x5A)
    assert torch.all(sbuf[:GUARD] == 0x3C) and torch.all(sbuf[GUARD + sbytes:] == 0x3C)
    q2, s2 = hc.hadacore_fwht_quant(x, qtype=qtype)
    assert torch.equal(qv.view(torch.uint8), q2.view(torch.uint8)) and torch.equal(sv, s2)


# ---------------------------------------------------------------- negative control
@pytest.fixture(scope="module")
def negctl_lib(hc):
    from paper_2412_08832_b200 import build as hc_build
    path = hc_build.LIB_NEGCTL
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: __graft_entry__.build() / paper_2412_08832_b200.build builds it")
    lib = ctypes.CDLL(path)
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    lib.hadacore_fwht.argtypes = [vp, vp, i64, i64, ctypes.c_int, ctypes.c_float, vp]
    lib.hadacore_fwht.restype = ctypes.c_int
    lib.hadacore_fwht_quant.argtypes = [vp, vp, vp, i64, i64, ctypes.c_int, ctypes.c_int, ctypes.c_float, vp]
    lib.hadacore_fwht_quant.restype = ctypes.c_int
    return lib


@pytest.mark.parametrize("dtype", DTYPES, ids=["fp16", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_negative_control_fails_parity(hc, negctl_lib, n, dtype):
    """The same parity check as tests/test_gpu_parity.py passes on the product library and
    fails on the sign-flipped build -- for every n the tensor-core path serves."""
    m = max(4, (1 << 17) // n)
    x = synthetic.generate(m, n, dtype, 4747).cuda()
    ref = oracle.fwht(widen(x))
    good = hc.hadacore_fwht(x)
    bad = torch.empty_like(x)
    rc = negctl_lib.hadacore_fwht(x.data_ptr(), bad.data_ptr(), m, n, {torch.float16: 0, torch.bfloat16: 1}[dtype],
                                  1.0 / math.sqrt(n), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert rc == 0
    assert rel_l2_rows(widen(good), ref).max() <= TOL[dtype]
    assert rel_l2_rows(widen(bad), ref).max() > 10 * TOL[dtype]


@pytest.mark.parametrize("n", [2048, 16384, 32768])
def test_negative_control_fails_quant_parity(hc, negctl_lib, n):
    """The fused quantization's parity check (dequantized outputs vs the oracle's transform) passes
    on the product library and fails on the sign-flipped build, for the register-epilogue kernel
    (n = 2048) and the tcgen05 kernel, whose H_128 B operand carries the flipped sign (n >= 16384)."""
    m = 8
    x = synthetic.generate(m, n, torch.bfloat16, 4848).cuda()
    ref = oracle.fwht(widen(x))
    q, s = hc.hadacore_fwht_quant(x, "int8")
    qb = torch.empty_like(q)
    sb = torch.empty_like(s)
    rc = negctl_lib.hadacore_fwht_quant(x.data_ptr(), qb.data_ptr(), sb.data_ptr(), m, n, 1, 1, 1.0 / math.sqrt(n),
                                        torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert rc == 0
    # error in units of the row's code step: the product build is within half a step plus the
    # bf16 transform error; one flipped sign of H_16 / H_128 moves whole outputs by several steps
    good = np.abs(widen(q.float()) * widen(s)[:, None] - ref) / widen(s)[:, None]
    bad = np.abs(widen(qb.float()) * widen(sb)[:, None] - ref) / widen(sb)[:, None]
    assert good.max() <= 1.0
    assert bad.max() > 3.0
