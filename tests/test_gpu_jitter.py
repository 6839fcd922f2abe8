"""Barrier protocols under perturbed timing (VERDICT r1 "prove the cluster barrier protocol
with a targeted stress test"): libhadacore_jitter.so is the product source built with
-DHC_JITTER, which sleeps for random 0-4 us at a quarter of the synchronization points of

* fwht_f32_ring_kernel (fp32 n = 2^15, the default: chunk slots refilled once the row's
  consumers released them, per-group chunk phases, the cross-chunk phase after an
  all-consumer barrier; fwht_f32_pair_kernel, the HC_F32_PAIR build, has its own sites:
  DSMEM exchange with remote mbarrier arrivals `ready` / `consumed`), and
* fwht_quant_tc_kernel (fused quantization n >= 16384: producer / phase-A / MMA / epilogue
  warp roles, TMEM double buffer, half-stage refills, code-store handoff).

A protocol that relied on a particular interleaving (a missing wait, a parity aliased two
phases ahead, a buffer reused before its reader is done) would show up as different bits or
a hang (the tests run under pytest-timeout).  Results must be bitwise those of the product
library, run after run, and within the north_star tolerance of the fp64 oracle.
"""
import ctypes
import os

import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_08832_b200 as hc
    hc._load()
    return hc


@pytest.fixture(scope="module")
def jitter_lib(hc):
    from paper_2412_08832_b200 import build as hc_build
    path = hc_build.LIB_JITTER
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: __graft_entry__.build() / paper_2412_08832_b200.build builds it")
    lib = ctypes.CDLL(path)
    vp, i64, ci, cf = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float
    lib.hadacore_fwht.argtypes = [vp, vp, i64, i64, ci, cf, vp]
    lib.hadacore_fwht.restype = ci
    lib.hadacore_fwht_quant.argtypes = [vp, vp, vp, i64, i64, ci, ci, cf, vp]
    lib.hadacore_fwht_quant.restype = ci
    return lib


def stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.timeout(300)
def test_f32_32k_kernel_under_jitter(hc, jitter_lib):
    n = 32768
    m = 3 * 148 + 7  # several rows per cluster, ragged over the clusters
    x = synthetic.generate(m, n, torch.float32, 9191).cuda()
    good = hc.hadacore_fwht(x)
    torch.cuda.synchronize()
    for rep in range(4):
        y = torch.full_like(x, float("nan"))
        assert jitter_lib.hadacore_fwht(x.data_ptr(), y.data_ptr(), m, n, 2, n ** -0.5, stream()) == 0
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int32), good.view(torch.int32)), f"rep {rep}: bits differ under jitter"
    # the perturbation is real: the jitter build is measurably slower on the same launch
    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        e0.record()
        for _ in range(3):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)
    t_good = timed(lambda: hc.hadacore_fwht(x, out=y))
    t_jit = timed(lambda: jitter_lib.hadacore_fwht(x.data_ptr(), y.data_ptr(), m, n, 2, n ** -0.5, stream()))
    assert t_jit > 1.02 * t_good, (t_jit, t_good)
    ref = oracle.fwht(x[:8].cpu().double().numpy())
    got = y[:8].cpu().double().numpy()
    err = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err.max() <= 1e-5


@pytest.mark.timeout(300)
@pytest.mark.parametrize("qtype,n", [("e4m3", 16384), ("e4m3", 32768), ("int4", 16384), ("int4", 32768),
                                     ("int4", 512)])
def test_quant_tc_kernel_under_jitter(hc, jitter_lib, n, qtype):
    # (INT4 n = 512: the tcgen05 kernel with rows of 2 chunks, 64 rows per tile)
    m = 2 * 148 * (128 // (n // 256)) * 3 + 1  # several tiles per CTA, a ragged last tile
    x = synthetic.generate(m, n, torch.bfloat16, 9292, dist="D1").cuda()
    q_good, s_good = hc.hadacore_fwht_quant(x, qtype)
    torch.cuda.synchronize()
    qcode = {"e4m3": 0, "int8": 1, "int4": 2}[qtype]
    for rep in range(3):
        q = torch.empty_like(q_good).view(torch.uint8).fill_(0xA5)
        s = torch.full_like(s_good, float("nan"))
        assert jitter_lib.hadacore_fwht_quant(x.data_ptr(), q.data_ptr(), s.data_ptr(), m, n, 1, qcode, n ** -0.5,
                                              stream()) == 0
        torch.cuda.synchronize()
        assert torch.equal(q, q_good.view(torch.uint8)), f"rep {rep}: codes differ under jitter"
        assert torch.equal(s.view(torch.int32), s_good.view(torch.int32)), f"rep {rep}: scales differ under jitter"
