"""GPU parity of the full-speed fp32 path (north_star's fp32
path: max per-row relative L2 <= 1e-5 vs the fp64 oracle) for every n = 2..2^15.

Shapes: several 32/64 KiB tiles plus a ragged tail (odd m: for n = 2 the total is
not a multiple of 16 bytes), in place == out of place bitwise, determinism over
more tiles than SMs, the identity closed form bitwise, non-finite rows isolated,
and the two-pass n = 2^15 path.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

NS = [1 << k for k in range(1, 16)]
TOL = 1e-5


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


def tile_rows(n):
    tile = (64 if n >= 16384 else 32) * 1024
    return max(1, tile // (4 * n))


@pytest.mark.parametrize("dist", ["D0", "D1"])
@pytest.mark.parametrize("n", NS)
def test_f32_parity(hc, n, dist):
    m = max(3 * tile_rows(n) + tile_rows(n) // 2 + 1, 3)
    m = min(m, max(3, (1 << 21) // n) | 1)
    x = synthetic.generate(m, n, torch.float32, 51 + n, dist=dist).cuda()
    y = hc.hadacore_fwht(x)
    err = rel_l2_rows(widen(y), oracle.fwht(widen(x)))
    assert err.max() <= TOL, (err.max(), err.argmax())


@pytest.mark.parametrize("n", NS)
def test_f32_inplace_determinism_and_small_m(hc, n):
    m = min(2 * 148 * tile_rows(n) + 3, max(5, (1 << 24) // n))
    x = synthetic.generate(m, n, torch.float32, 7, device="cuda")
    y1 = hc.hadacore_fwht(x)
    y2 = hc.hadacore_fwht(x)
    xi = x.clone()
    hc.hadacore_fwht(xi, out=xi)
    assert torch.equal(y1, y2) and torch.equal(y1, xi)
    for mm in (1, 2, 3, 5):
        xs = synthetic.generate(mm, n, torch.float32, 70 + mm).cuda()
        buf = torch.full((mm * n + 16,), 7.0, device="cuda")
        hc.hadacore_fwht(xs, out=buf[: mm * n].view(mm, n))
        assert torch.all(buf[mm * n:] == 7.0)
        assert rel_l2_rows(widen(buf[: mm * n].view(mm, n)), oracle.fwht(widen(xs))).max() <= TOL


@pytest.mark.parametrize("n", NS)
def test_f32_identity_and_isolation(hc, n):
    rows = min(n, 256)
    e = torch.zeros(rows, n, device="cuda")
    e[torch.arange(rows), torch.arange(rows)] = 1.0
    ye = hc.hadacore_fwht(e).cpu()
    mag = torch.tensor(1.0 / math.sqrt(n), dtype=torch.float32)
    a = torch.arange(rows)[:, None] & torch.arange(n)[None, :]
    par = torch.zeros_like(a)
    for b in range(15):
        par ^= (a >> b) & 1
    assert torch.equal(ye, torch.where(par == 1, -mag, mag))
    z = synthetic.generate(3 * tile_rows(n) + 4, n, torch.float32, 9).cuda()
    z[1::3] = float("nan")
    yz = hc.hadacore_fwht(z)
    keep = [r for r in range(z.shape[0]) if r % 3 != 1]
    assert torch.isfinite(yz[keep]).all() and torch.isnan(yz[1::3]).all()


@pytest.mark.slow
@pytest.mark.parametrize("n", [2, 64, 128, 4096, 16384, 32768])
def test_f32_full_size_sampled(hc, n):
    """2^28 elements (bench.py --workload f32): sampled rows vs the oracle."""
    m = (1 << 28) // n
    x = torch.empty(m, n, dtype=torch.float32, device="cuda")
    synthetic.generate(m, n, torch.float32, 3, out=x)
    y = hc.hadacore_fwht(x)
    g = torch.Generator().manual_seed(n)
    rows = sorted(set([0, m - 1] + torch.randint(0, m, (40,), generator=g).tolist()))
    assert rel_l2_rows(widen(y[rows]), oracle.fwht(widen(x[rows]))).max() <= TOL


def test_f32_32k_kernel_repeatability_stress(hc):
    """The fp32 n = 2^15 kernel (fwht_f32_stream_kernel: chunk slots refilled as soon as every
    consumer warp has gathered its columns, results stored from registers; the HC_F32_PAIR build's
    2-CTA cluster kernel synchronizes through remote mbarriers): 40 back-to-back launches over
    more rows than SMs must all give the same bits, in place and out of place."""
    n, m = 32768, 300
    x = synthetic.generate(m, n, torch.float32, 13, device="cuda")
    ref = hc.hadacore_fwht(x)
    outs = [torch.empty_like(x) for _ in range(4)]
    for k in range(40):
        hc.hadacore_fwht(x, out=outs[k % 4])
        if k % 4 == 3:
            torch.cuda.synchronize()
            for o in outs:
                assert torch.equal(o, ref), k
    xi = x.clone()
    hc.hadacore_fwht(xi, out=xi)
    assert torch.equal(xi, ref)
    assert rel_l2_rows(widen(ref[:8]), oracle.fwht(widen(x[:8]))).max() <= TOL


@pytest.mark.parametrize("n", [2, 1024, 32768])
def test_f32_host_entry(hc, n):
    """hadacore_fwht_host with fp32 buffers (slots of >= 16 bytes for n = 2) equals the device entry bitwise."""
    m = max(3, (1 << 20) // n) + 1
    x = synthetic.generate(m, n, torch.float32, 17).pin_memory()
    ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    y_host = hc.hadacore_fwht_host(x, workspace=ws)
    y_dev = hc.hadacore_fwht(x.cuda()).cpu()
    assert torch.equal(y_host, y_dev)
