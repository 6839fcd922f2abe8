"""GPU parity for rows shorter than 128 (n = 2..64).

The same bar as tests/test_gpu_parity.py: max per-row relative L2 vs the fp64
oracle <= 2e-3 (fp16) / 1.6e-2 (bf16), identity input bitwise against the closed
form (-1)^popcount(i&j) * RNE(1/sqrt(n)), in place == out of place bitwise,
determinism, non-finite rows isolated.  Shapes exercise the kernel's edges:
several 32 KiB tiles with a ragged tail, and (n = 2, 4) totals that are not a
multiple of 16 bytes (the last partial granule bypasses the bulk copy).
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

NS = [2, 4, 8, 16, 32, 64]
DTYPES = [torch.float16, torch.bfloat16]
TOL = {torch.float16: 2e-3, torch.bfloat16: 1.6e-2}
TILE_BYTES = 32 * 1024  # hadacore.cu TunedS: 32 KiB ring stages


@pytest.fixture(scope="module")
def hc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_08832_b200 as hc
    hc._load()
    return hc


def widen(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().to(torch.float64).numpy()


def rel_l2_rows(got: np.ndarray, ref: np.ndarray) -> np.ndarray:
    num = np.linalg.norm(got - ref, axis=1)
    den = np.linalg.norm(ref, axis=1)
    return num / np.where(den == 0, 1.0, den)


def tile_rows(n: int) -> int:
    return TILE_BYTES // (2 * n)


@pytest.mark.parametrize("dist", ["D0", "D1"])
@pytest.mark.parametrize("dtype", DTYPES, ids=["fp16", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_parity_vs_oracle(hc, n, dtype, dist):
    # 5 full tiles + a ragged tail with an odd row count (not a multiple of 16 bytes for n <= 4)
    m = 5 * tile_rows(n) + tile_rows(n) // 2 + 1
    x = synthetic.generate(m, n, dtype, synthetic.seed_for(2, dtype), dist=dist).cuda()
    y = hc.hadacore_fwht(x)
    torch.cuda.synchronize()
    ref = oracle.fwht(widen(x))
    err = rel_l2_rows(widen(y), ref)
    assert np.all(np.isfinite(widen(y)))
    assert err.max() <= TOL[dtype], f"max rel-L2 {err.max():.3e} (row {err.argmax()})"


@pytest.mark.parametrize("dtype", DTYPES, ids=["fp16", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_small_m_every_tail(hc, n, dtype):
    # every m up to 3 granules + 1 (each tail length of the last partial granule), and m = 0
    for m in list(range(1, 3 * max(1, 8 // n) + 2)) + [tile_rows(n) - 1, tile_rows(n), tile_rows(n) + 1]:
        x = synthetic.generate(m, n, dtype, 100 + m).cuda()
        y = hc.hadacore_fwht(x)
        err = rel_l2_rows(widen(y), oracle.fwht(widen(x)))
        assert err.max() <= TOL[dtype], (m, err.max())
    e = torch.empty(0, n, dtype=dtype, device="cuda")
    assert hc.hadacore_fwht(e).shape == (0, n)


@pytest.mark.parametrize("n", NS)
def test_tail_does_not_write_past_the_end(hc, n):
    # the output lives inside a larger buffer: the bytes after the last row stay untouched
    for m in (1, 3, 5, 7, tile_rows(n) + 3):
        x = synthetic.generate(m, n, torch.float16, 7 + m).cuda()
        buf = torch.full((m * n + 64,), 1234.0, dtype=torch.float16, device="cuda")
        out = buf[: m * n].view(m, n)
        hc.hadacore_fwht(x, out=out)
        assert torch.all(buf[m * n:] == 1234.0), m
        assert rel_l2_rows(widen(out), oracle.fwht(widen(x))).max() <= 2e-3


@pytest.mark.parametrize("dtype", DTYPES, ids=["fp16", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_identity_exact_closed_form(hc, n, dtype):
    """I_n repeated: output row i must be bitwise (-1)^popcount(i&j) * RNE(1/sqrt(n))."""
    reps = max(1, 4096 // n)
    x = torch.eye(n, dtype=dtype).repeat(reps, 1).cuda()  # reps * n rows: several tiles for small n
    y = hc.hadacore_fwht(x).cpu()
    mag = torch.tensor(1.0 / math.sqrt(n), dtype=torch.float64).to(dtype)
    i = torch.arange(n)[:, None]
    j = torch.arange(n)[None, :]
    a = i & j
    par = torch.zeros_like(a)
    for b in range(7):
        par ^= (a >> b) & 1
    expect = torch.where(par == 1, -mag, mag).repeat(reps, 1)
    assert torch.equal(y.view(torch.int16), expect.view(torch.int16))


@pytest.mark.parametrize("dtype", DTYPES, ids=["fp16", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_special_rows_and_isolation(hc, n, dtype):
    sp, names = synthetic.special_rows(n, dtype)
    g = synthetic.generate(6, n, dtype, 99)
    x = torch.cat([g[:3], sp, g[3:]]).contiguous()
    y = widen(hc.hadacore_fwht(x.cuda()))
    ref = oracle.fwht(widen(x))
    for i in range(x.shape[0]):
        name = names[i - 3] if 3 <= i < 3 + len(names) else "finite"
        if name in ("inf", "nan"):
            assert not np.any(np.isfinite(y[i])), f"{name} row has finite outputs"
            continue
        assert np.all(np.isfinite(y[i])), f"row {i} ({name}) not finite"
        if name == "zeros":
            assert np.all(y[i] == 0.0)
        elif name == "subnormal":
            spacing = torch.finfo(dtype).tiny * torch.finfo(dtype).eps
            assert np.max(np.abs(y[i] - ref[i])) <= 8 * spacing, name
        else:
            e = rel_l2_rows(y[i:i + 1], ref[i:i + 1])[0]
            assert e <= TOL[dtype], f"row {i} ({name}) rel-L2 {e:.3e}"
    # NaN rows interleaved with finite rows (several rows share a granule for n <= 8)
    m = 2 * tile_rows(n) + 5
    z = synthetic.generate(m, n, dtype, 77).cuda()
    z[1::3] = float("nan")
    yz = hc.hadacore_fwht(z)
    finite_rows = [r for r in range(m) if r % 3 != 1]
    assert torch.isfinite(yz[finite_rows]).all()
    assert torch.isnan(yz[1::3]).all()


@pytest.mark.parametrize("dtype", DTYPES, ids=["fp16", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_inplace_bitwise_and_deterministic(hc, n, dtype):
    m = 2 * tile_rows(n) * 148 + 3  # more tiles than SMs (CLC work stealing) + ragged tail
    x = synthetic.generate(m, n, dtype, 5, device="cuda")
    y1 = hc.hadacore_fwht(x)
    y2 = hc.hadacore_fwht(x)
    xi = x.clone()
    hc.hadacore_fwht(xi, out=xi)
    torch.cuda.synchronize()
    assert torch.equal(y1.view(torch.int16), y2.view(torch.int16))
    assert torch.equal(y1.view(torch.int16), xi.view(torch.int16))


@pytest.mark.parametrize("n", NS)
def test_scale_and_involution(hc, n):
    x = synthetic.generate(1000, n, torch.float16, 8).cuda()
    y = widen(hc.hadacore_fwht(x, scale=0.37))
    assert rel_l2_rows(y, oracle.fwht(widen(x), scale=0.37)).max() <= 2e-3
    z = hc.hadacore_fwht(hc.hadacore_fwht(x))
    assert rel_l2_rows(widen(z), widen(x)).max() <= 2 * 2e-3


@pytest.mark.parametrize("n", [2, 4, 64])
def test_host_entry_small_n(hc, n):
    # a tiny workspace forces many blocks; slot offsets must stay 16-byte aligned for rows < 16 B
    x = synthetic.generate(3001, n, torch.bfloat16, 4).pin_memory()
    for ws_bytes in (max(64, 4 * n), 1000, 1 << 16):  # >= two rows (the C contract)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
        y_host = hc.hadacore_fwht_host(x, workspace=ws)
        y_dev = hc.hadacore_fwht(x.cuda()).cpu()
        assert torch.equal(y_host.view(torch.int16), y_dev.view(torch.int16)), ws_bytes


@pytest.mark.parametrize("n", NS)
def test_fp32_debug_path_small_n(hc, n):
    m = 4097  # odd: n = 2 exercises the element-wise copy of a partial group
    x = synthetic.generate(m, n, torch.float32, 21, dist="D1").cuda()
    y = hc.hadacore_fwht(x)
    assert rel_l2_rows(widen(y), oracle.fwht(widen(x))).max() <= 1e-5
    xi = x.clone()
    hc.hadacore_fwht(xi, out=xi)
    assert torch.equal(xi, y)


@pytest.mark.slow
@pytest.mark.parametrize("dtype", DTYPES, ids=["fp16", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_full_size_sampled(hc, n, dtype):
    """2^28 elements (bench.py --workload small): sampled rows vs the oracle, and
    norm preservation on every row."""
    m = (1 << 28) // n
    x = torch.empty(m, n, dtype=dtype, device="cuda")
    synthetic.generate(m, n, dtype, synthetic.seed_for(2, dtype), out=x)
    y = hc.hadacore_fwht(x)
    torch.cuda.synchronize()
    g = torch.Generator().manual_seed(n)
    rows = sorted(set([0, 1, m - 1, m // 2] + torch.randint(0, m, (200,), generator=g).tolist()))
    assert rel_l2_rows(widen(y[rows]), oracle.fwht(widen(x[rows]))).max() <= TOL[dtype]
    blk = 1 << 22
    worst = 0.0
    for r0 in range(0, m, blk):
        nx = x[r0:r0 + blk].float().norm(dim=1)
        ny = y[r0:r0 + blk].float().norm(dim=1)
        worst = max(worst, ((ny - nx).abs() / nx).max().item())
    assert worst <= TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES, ids=["fp16", "bf16"])
@pytest.mark.parametrize("n,heads", [(8, 4), (16, 3), (32, 8), (64, 32), (64, 1), (64, 300)])
def test_strided_qkv_heads_small_n(hc, n, heads, dtype):
    """Row grids for n = 8..64 (3-D TMA boxes, box dims capped at 256): the Q and K heads of
    [T, 3, H, d] rotated in place equal the contiguous transform bitwise; V untouched."""
    tokens = max(3, (1 << 18) // (3 * heads * n)) + 1
    qkv = synthetic.generate(tokens * 3 * heads, n, dtype, 31, dist="D1").reshape(tokens, 3, heads, n).cuda()
    before = qkv.clone()
    qk = qkv[:, 0:2]
    hc.hadacore_fwht_strided(qk, out=qk)
    y = hc.hadacore_fwht(before[:, 0:2].contiguous())
    assert torch.equal(qkv[:, 0:2].contiguous().view(torch.int16), y.view(torch.int16))
    assert torch.equal(qkv[:, 2].view(torch.int16), before[:, 2].view(torch.int16))
    err = rel_l2_rows(widen(y.reshape(-1, n)), oracle.fwht(widen(before[:, 0:2].reshape(-1, n))))
    assert err.max() <= TOL[dtype]


@pytest.mark.parametrize("n", [8, 32, 64])
def test_strided_padded_pitch_small_n(hc, n):
    m, pitch = 1001, n + 8
    base = synthetic.generate(m, pitch, torch.float16, 32).cuda()
    x = base[:, :n]
    y = hc.hadacore_fwht_strided(x)
    assert torch.equal(y.view(torch.int16), hc.hadacore_fwht(x.contiguous()).view(torch.int16))
    out_pad = torch.zeros(m, pitch, dtype=torch.float16, device="cuda")
    hc.hadacore_fwht_strided(x, out=out_pad[:, :n])
    assert torch.equal(out_pad[:, :n].view(torch.int16), y.view(torch.int16)) and not out_pad[:, n:].any()
