"""GPU parity of the fused transform + per-row quantization (hadacore_fwht_quant,
SURVEY.md 8(f) NEXT-1) against the fp64 oracle (oracle.fwht + oracle.quantize_rows).

The quantized code is an integer decided by floating point, so it is compared as
follows (task rule: several results may be correct near rounding boundaries):
* row scales: |s_gpu - s_ref| <= tol(dtype) * s_ref, where tol is the transform's
  own tolerance (the scale is max|y| / Q and inherits y's error);
* codes: most are identical, and where the code grid is coarse compared with the
  transform's own error (spacing >= 8x the per-row RMS error allowed by tol, i.e.
  eps = tol ||y|| / sqrt(n) in code units), every GPU code is the oracle's code or
  an adjacent representable value (the GPU decides the rounding on its own y);
* dequantized values q*s against the exact y, with the error bound that follows
  from the arithmetic:
    int8: ||q s - y|| <= (s/2) sqrt(n) + tol ||y||
    e4m3: ||q s - y|| <= (2^-4 + tol) ||y|| + 2^-10 s sqrt(n)
* exact case: identity input -> every |y| = 1/sqrt(n) = max, so codes are +-Q
  bitwise (E4M3 0x7E/0xFE, INT8 +-127) and s = (1/sqrt(n)) / Q.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

NS = [1 << k for k in range(1, 16)]  # n < 128: fwht_small_kernel's fused epilogue
DTYPES = [torch.float16, torch.bfloat16]
TOL = {torch.float16: 2e-3, torch.bfloat16: 1.6e-2}
QMAX = {"e4m3": 448.0, "int8": 127.0, "int4": 7.0}
QTYPES = ["e4m3", "int8", "int4"]


def unpack_int4(q_u8: np.ndarray) -> np.ndarray:
    """(m, n/2) bytes -> (m, n) int8 codes: element 2j = low nibble of byte j (two's complement)."""
    lo = (q_u8 & 0x0F).astype(np.int16)
    hi = (q_u8 >> 4).astype(np.int16)
    out = np.empty((q_u8.shape[0], 2 * q_u8.shape[1]), dtype=np.int16)
    out[:, 0::2], out[:, 1::2] = lo, hi
    out = np.where(out >= 8, out - 16, out)
    return out.astype(np.int8).view(np.uint8)


def gpu_codes(q: torch.Tensor, qtype: str) -> np.ndarray:
    c = q.view(torch.uint8).cpu().numpy()
    return unpack_int4(c) if qtype == "int4" else c


@pytest.fixture(scope="module")
def hc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_08832_b200 as hc
    hc._load()
    return hc


def e4m3_sorted_values():
    vals = sorted({oracle.e4m3_value(c) for c in range(256) if c not in (0x7F, 0xFF)})
    return np.array(vals)


E4M3_VALUES = None


def code_values(codes_u8: np.ndarray, qtype: str) -> np.ndarray:
    if qtype in ("int8", "int4"):
        return codes_u8.view(np.int8).astype(np.float64)
    table = np.array([oracle.e4m3_value(c) for c in range(256)])
    return table[codes_u8]


def adjacent(v_gpu: np.ndarray, v_ref: np.ndarray, qtype: str) -> np.ndarray:
    """True where the two code values are equal or neighbours on the code grid."""
    if qtype in ("int8", "int4"):
        return np.abs(v_gpu - v_ref) <= 1
    global E4M3_VALUES
    if E4M3_VALUES is None:
        E4M3_VALUES = e4m3_sorted_values()
    ig = np.searchsorted(E4M3_VALUES, v_gpu)
    ir = np.searchsorted(E4M3_VALUES, v_ref)
    return np.abs(ig - ir) <= 1


def ragged_m(n):
    return max(3, (1 << 19) // n) + 1  # odd: n <= 4 ends in a partial 16-byte granule


@pytest.mark.parametrize("qtype", QTYPES)
@pytest.mark.parametrize("dist", ["D0", "D1"])
@pytest.mark.parametrize("dtype", DTYPES, ids=["fp16", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_quant_parity(hc, n, dtype, dist, qtype):
    m = ragged_m(n)
    x = synthetic.generate(m, n, dtype, synthetic.seed_for(3, dtype), dist=dist).cuda()
    q, s = hc.hadacore_fwht_quant(x, qtype=qtype)
    torch.cuda.synchronize()
    codes = gpu_codes(q, qtype)
    s_gpu = s.cpu().double().numpy()
    y = oracle.fwht(x.cpu().double().numpy())
    codes_ref, s_ref = oracle.quantize_rows(y, qtype)
    tol = TOL[dtype]
    assert np.all(np.abs(s_gpu - s_ref) <= tol * s_ref), "row scales"
    vg, vr = code_values(codes, qtype), code_values(codes_ref, qtype)
    eps = (tol * np.linalg.norm(y, axis=1) / math.sqrt(n) / s_ref)[:, None]   # RMS error, code units
    spacing = np.ones_like(vr) if qtype != "e4m3" else np.maximum(np.abs(vr) * 2.0 ** -3, 2.0 ** -9)
    coarse = spacing >= 8 * eps
    assert np.all(adjacent(vg, vr, qtype) | ~coarse), "codes not adjacent to the oracle's"
    same = np.mean(codes == codes_ref)
    assert same >= (0.9 if dtype == torch.float16 else 0.6), f"only {same:.3f} of codes identical"
    deq = vg * s_gpu[:, None]
    err = np.linalg.norm(deq - y, axis=1)
    ny = np.linalg.norm(y, axis=1)
    if qtype != "e4m3":
        bound = s_gpu / 2 * math.sqrt(n) + tol * ny
    else:
        bound = (2.0 ** -4 + tol) * ny + 2.0 ** -10 * s_gpu * math.sqrt(n)
    assert np.all(err <= bound * 1.0001), f"dequantized error {np.max(err / bound):.3f} x bound"


@pytest.mark.parametrize("qtype", QTYPES)
@pytest.mark.parametrize("dtype", DTYPES, ids=["fp16", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_quant_identity_exact(hc, n, dtype, qtype):
    """Identity input: y = +-1/sqrt(n) everywhere, all equal to the row max, so every
    code is +-Q exactly and the scale is (1/sqrt(n))/Q (closed form, no oracle)."""
    rows = min(n, 256)
    x = torch.zeros(rows, n, dtype=dtype, device="cuda")
    x[torch.arange(rows), torch.arange(rows)] = 1.0
    q, s = hc.hadacore_fwht_quant(x, qtype=qtype)
    i = torch.arange(rows, device="cuda", dtype=torch.int64)[:, None]
    j = torch.arange(n, device="cuda", dtype=torch.int64)[None, :]
    a = i & j
    par = torch.zeros_like(a)
    for b in range(15):
        par ^= (a >> b) & 1
    if qtype == "e4m3":
        expect = torch.where(par == 1, 0xFE, 0x7E).to(torch.uint8)
    else:
        qm = int(QMAX[qtype])
        expect = torch.where(par == 1, -qm, qm).to(torch.int8).view(torch.uint8)
    got = torch.from_numpy(gpu_codes(q, qtype)).cuda()
    assert torch.equal(got, expect)
    s_exp = (1.0 / math.sqrt(n)) / QMAX[qtype]
    assert torch.allclose(s.double(), torch.full_like(s.double(), s_exp), rtol=1e-6, atol=0)


@pytest.mark.parametrize("n", NS)
def test_quant_special_rows(hc, n):
    dtype = torch.bfloat16
    sp, names = synthetic.special_rows(n, dtype)
    g = synthetic.generate(4, n, dtype, 5)
    x = torch.cat([g[:2], sp, g[2:]]).contiguous().cuda()
    for qtype in QTYPES:
        q, s = hc.hadacore_fwht_quant(x, qtype=qtype)
        sc = s.cpu().double().numpy()
        y = oracle.fwht(x.cpu().double().numpy())
        for r in range(x.shape[0]):
            name = names[r - 2] if 2 <= r < 2 + len(names) else "finite"
            if name in ("inf", "nan"):
                assert not np.isfinite(sc[r]), (name, qtype)
            elif name == "zeros":
                assert sc[r] == 1.0 and not q[r].view(torch.uint8).any()
            elif name != "subnormal":
                amax = np.abs(y[r]).max()
                assert abs(sc[r] - amax / QMAX[qtype]) <= TOL[dtype] * amax / QMAX[qtype], (name, qtype)


def test_quant_matches_fwht_then_quantize_on_gpu_values(hc):
    """The fused output equals quantizing the unfused kernel's own bf16 output for
    n <= 256 up to one code step (the fused path quantizes the fp32 value, the
    unfused one rounds to 16 bits first)."""
    for n in (128, 256, 1024):
        x = synthetic.generate(300, n, torch.bfloat16, 8).cuda()
        y16 = hc.hadacore_fwht(x).cpu().double().numpy()
        q, s = hc.hadacore_fwht_quant(x, qtype="int8")
        codes_ref, _ = oracle.quantize_rows(y16, "int8")
        vg = code_values(q.view(torch.uint8).cpu().numpy(), "int8")
        vr = code_values(codes_ref, "int8")
        assert np.all(np.abs(vg - vr) <= 1)


@pytest.mark.parametrize("n", [2, 8, 64, 128, 256, 512, 4096, 32768])
def test_int4_packing_and_views(hc, n):
    """INT4 layout: (m, n/2) bytes, element 2j in the low nibble of byte j; leading dims
    are rows; a ragged m; the codes unpack to the oracle's within one step."""
    x = synthetic.generate(2 * 3 * 5, n, torch.float16, 17, dist="D1").reshape(2, 3, 5, n).cuda()
    q, s = hc.hadacore_fwht_quant(x, qtype="int4")
    assert q.shape == (2, 3, 5, n // 2) and q.dtype == torch.uint8 and s.shape == (2, 3, 5)
    y = oracle.fwht(x.reshape(-1, n).cpu().double().numpy())
    cr, sr = oracle.quantize_rows(y, "int4")
    cg = gpu_codes(q.reshape(-1, n // 2), "int4")
    assert np.all(np.abs(code_values(cg, "int4") - code_values(cr, "int4")) <= 1)
    assert np.mean(cg == cr) >= 0.95


@pytest.mark.parametrize("qtype", QTYPES)
@pytest.mark.parametrize("n", [2, 4, 8, 16, 64])
def test_small_n_quant_tail_and_bounds(hc, n, qtype):
    """n < 128: every ragged tail (odd m for n <= 4 leaves a partial granule) writes
    exactly the valid codes and scales -- bytes past the end are untouched."""
    for m in (1, 2, 3, 5, 7, 4097):
        x = synthetic.generate(m, n, torch.bfloat16, 60 + m, dist="D1").cuda()
        cb = n // 2 if qtype == "int4" else n
        qbuf = torch.full((m * cb + 32,), 0xAB, dtype=torch.uint8, device="cuda")
        sbuf = torch.full((m + 8,), -7.0, dtype=torch.float32, device="cuda")
        qv = qbuf[: m * cb].view(m, cb)
        qv = qv.view(torch.float8_e4m3fn) if qtype == "e4m3" else (qv.view(torch.int8) if qtype == "int8" else qv)
        hc.hadacore_fwht_quant(x, qtype=qtype, out=qv, row_scale=sbuf[:m])
        assert torch.all(qbuf[m * cb:] == 0xAB) and torch.all(sbuf[m:] == -7.0), m
        y = oracle.fwht(x.cpu().double().numpy())
        cr, sr = oracle.quantize_rows(y, qtype)
        cg = gpu_codes(qv, qtype)
        assert np.all(np.abs(sbuf[:m].cpu().double().numpy() - sr) <= TOL[torch.bfloat16] * sr), m
        assert np.all(adjacent(code_values(cg, qtype), code_values(cr, qtype), qtype)), m


def test_small_n_quant_unaligned_row_scale(hc):
    """row_scale needs only 4-byte alignment (C contract): n = 2, 4 with a row_scale at an
    odd float offset (the kernel falls back from vector scale stores)."""
    for n in (2, 4):
        m = 4099
        x = synthetic.generate(m, n, torch.float16, 3).cuda()
        big = torch.zeros(m + 1, dtype=torch.float32, device="cuda")
        q, s = hc.hadacore_fwht_quant(x, qtype="int8", row_scale=big[1:])
        q2, s2 = hc.hadacore_fwht_quant(x, qtype="int8")
        assert torch.equal(s, s2) and torch.equal(q.view(torch.uint8), q2.view(torch.uint8))


@pytest.mark.parametrize("qtype", QTYPES)
@pytest.mark.parametrize("n,heads", [(8, 4), (16, 3), (32, 8), (64, 32), (64, 300), (128, 32), (128, 3), (256, 8),
                                     (1024, 5), (4096, 2), (32768, 1)])
def test_quant_strided_qk_heads(hc, n, heads, qtype):
    """FP8-attention deployment path: the Q and K heads of a fused QKV
    projection [T, 3, H, d] rotated + quantized in one pass (hadacore_fwht_quant_strided)
    give bitwise the codes and scales of the contiguous entry on a copy; the input is
    untouched."""
    tokens = max(3, (1 << 19) // (3 * heads * n)) + 1
    qkv = synthetic.generate(tokens * 3 * heads, n, torch.bfloat16, 33, dist="D1").reshape(tokens, 3, heads, n).cuda()
    before = qkv.clone()
    view = qkv[:, 0:2]
    q, s = hc.hadacore_fwht_quant_strided(view, qtype=qtype)
    assert torch.equal(qkv.view(torch.int16), before.view(torch.int16))
    q2, s2 = hc.hadacore_fwht_quant(view.contiguous(), qtype=qtype)
    assert q.shape == q2.shape and s.shape == s2.shape == (tokens, 2, heads)
    assert torch.equal(q.view(torch.uint8), q2.view(torch.uint8)) and torch.equal(s, s2)


@pytest.mark.parametrize("qtype", QTYPES)
@pytest.mark.parametrize("n", [16, 64, 256, 2048])
def test_quant_strided_padded_pitch(hc, n, qtype):
    """Rows with a padded pitch (m_inner = 1, stride_outer = n + 64): codes and scales equal the
    contiguous entry's on a copy, bitwise."""
    m, pitch = 777, n + 64
    base = synthetic.generate(m, pitch, torch.float16, 35, dist="D1").cuda()
    x = base[:, :n]
    q, s = hc.hadacore_fwht_quant_strided(x, qtype=qtype)
    q2, s2 = hc.hadacore_fwht_quant(x.contiguous(), qtype=qtype)
    assert torch.equal(q.view(torch.uint8), q2.view(torch.uint8)) and torch.equal(s, s2)
