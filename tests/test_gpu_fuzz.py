"""Seeded random sweep over the entry points' argument space (n, m, dtype, in/out of
place, scale, row grids, quantization) against the fp64 oracle -- small problems that
hit every kernel family and its edge handling (partial tiles, partial granules,
row-grid boxes at the 256-row cap, zero rows)."""
import math

import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

TOL = {torch.float16: 2e-3, torch.bfloat16: 1.6e-2, torch.float32: 1e-5}


@pytest.fixture(scope="module")
def hc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_08832_b200 as hc
    hc._load()
    return hc


def rel_err(got, ref):
    den = np.linalg.norm(ref, axis=1)
    return (np.linalg.norm(got - ref, axis=1) / np.where(den == 0, 1.0, den)).max(initial=0.0)


@pytest.mark.parametrize("case", range(48))
def test_fuzz_transform(hc, case):
    rng = np.random.default_rng(1000 + case)
    n = 1 << int(rng.integers(1, 16))
    m = int(rng.integers(0, max(2, (1 << 19) // n)))
    dt = [torch.float16, torch.bfloat16, torch.float32][int(rng.integers(0, 3))]
    scale = float(rng.choice([1.0 / math.sqrt(n), 1.0, 0.37]))
    x = synthetic.generate(m, n, dt, 500 + case, dist="D1" if case % 2 else "D0").cuda()
    if rng.integers(0, 2):
        y = x.clone()
        hc.hadacore_fwht(y, out=y, scale=scale)
    else:
        y = hc.hadacore_fwht(x, scale=scale)
    if m == 0:
        assert y.shape == (0, n)
        return
    ref = oracle.fwht(x.cpu().double().numpy(), scale=scale)
    assert rel_err(y.cpu().double().numpy(), ref) <= TOL[dt], (n, m, dt, scale)


@pytest.mark.parametrize("case", range(24))
def test_fuzz_strided_and_quant(hc, case):
    rng = np.random.default_rng(2000 + case)
    n = 1 << int(rng.integers(3, 16))
    heads = int(rng.integers(1, max(2, min(300, (1 << 16) // n))))
    tokens = int(rng.integers(1, max(2, (1 << 18) // (3 * heads * n))))
    dt = [torch.float16, torch.bfloat16][int(rng.integers(0, 2))]
    qkv = synthetic.generate(tokens * 3 * heads, n, dt, 600 + case, dist="D1").reshape(tokens, 3, heads, n).cuda()
    view = qkv[:, 0:2]
    y_ref = hc.hadacore_fwht(view.contiguous())
    y = hc.hadacore_fwht_strided(view)
    assert torch.equal(y.view(torch.int16), y_ref.view(torch.int16)), (n, heads, tokens)
    qt = ["e4m3", "int8", "int4"][int(rng.integers(0, 3))]
    q, s = hc.hadacore_fwht_quant_strided(view, qtype=qt)
    q2, s2 = hc.hadacore_fwht_quant(view.contiguous(), qtype=qt)
    assert torch.equal(q.view(torch.uint8), q2.view(torch.uint8)) and torch.equal(s, s2), (n, heads, tokens, qt)
    ref = oracle.fwht(view.contiguous().reshape(-1, n).cpu().double().numpy())
    assert rel_err(y.reshape(-1, n).cpu().double().numpy(), ref) <= TOL[dt]


@pytest.mark.parametrize("case", range(24))
def test_fuzz_quant_sampled_rows(hc, case):
    """Fused quantization over random (n, m, dtype, qtype, scale) with up to 2^22 elements -- several
    tiles per CTA and a ragged last tile for every kernel family and launch-table entry -- checked on
    sampled rows (first, last, random) against the fp64 oracle: row scales within the transform
    tolerance and the dequantized rows within the quantization bound of test_gpu_quant.py."""
    from test_gpu_quant import gpu_codes, code_values
    rng = np.random.default_rng(3000 + case)
    n = 1 << int(rng.integers(1, 16))
    m = int(rng.integers(1, max(2, (1 << 22) // n)))
    dt = [torch.float16, torch.bfloat16][int(rng.integers(0, 2))]
    qt = ["e4m3", "int8", "int4"][int(rng.integers(0, 3))]
    scale = float(rng.choice([1.0 / math.sqrt(n), 1.0, 0.37]))
    x = synthetic.generate(m, n, dt, 700 + case, dist="D1" if case % 2 else "D0").cuda()
    q, s = hc.hadacore_fwht_quant(x, qtype=qt, scale=scale)
    rows = sorted(set([0, m - 1] + rng.integers(0, m, 62).tolist()))
    codes = gpu_codes(q[rows], qt)
    s_gpu = s[rows].cpu().double().numpy()
    y = oracle.fwht(x[rows].cpu().double().numpy(), scale=scale)
    _, s_ref = oracle.quantize_rows(y, qt)
    tol = TOL[dt]
    assert np.all(np.abs(s_gpu - s_ref) <= tol * s_ref), (n, m, dt, qt, scale)
    deq = code_values(codes, qt) * s_gpu[:, None]
    err = np.linalg.norm(deq - y, axis=1)
    ny = np.linalg.norm(y, axis=1)
    if qt != "e4m3":
        bound = s_gpu / 2 * math.sqrt(n) + tol * ny
    else:
        bound = (2.0 ** -4 + tol) * ny + 2.0 ** -10 * s_gpu * math.sqrt(n)
    assert np.all(err <= bound * 1.0001), (n, m, dt, qt, scale, float(np.max(err / bound)))
