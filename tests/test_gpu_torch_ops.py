"""torch custom ops on the deployment layout (NEXT-3; P:24 [Sec. 1], P:180 [Sec. 4.2]):
the Q and K heads of a fused QKV projection [T, 3, H, d] rotated (and quantized)
where they lie, through the strided C entry points -- compared bitwise with the
contiguous entry on a copy, and with the fp64 oracle.  Also the binding's device
checks (buffers on another device are rejected before any launch)."""
import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

TOL = {torch.float16: 2e-3, torch.bfloat16: 1.6e-2}


@pytest.fixture(scope="module")
def hc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_08832_b200 as hc
    import paper_2412_08832_b200.torch_ops  # noqa: F401  (registers torch.ops.hadacore.*)
    hc._load()
    return hc


def widen(t):
    return t.detach().cpu().to(torch.float64).numpy()


def rel_l2_rows(got, ref):
    return np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)


def qkv_buffer(t, h, d, dtype, seed):
    return synthetic.generate(t * 3 * h, d, dtype, seed).reshape(t, 3, h, d).cuda()


@pytest.mark.parametrize("d", [8, 64, 128, 256, 1024, 4096])
@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16], ids=["fp16", "bf16"])
def test_fwht_inplace_on_qk_heads(hc, d, dtype):
    """fwht_ on qkv[:, 0:2] transforms the Q and K heads in place (same storage), leaves V
    untouched, and matches the contiguous entry bitwise and the oracle within tolerance."""
    h = max(1, 1024 // d)
    qkv = qkv_buffer(37, h, d, dtype, 51)
    ref_in = qkv[:, 0:2].contiguous()
    v_before = qkv[:, 2].clone()
    view = qkv[:, 0:2]
    ptr = view.data_ptr()
    torch.ops.hadacore.fwht_(view, None)
    assert view.data_ptr() == ptr
    assert torch.equal(qkv[:, 2].view(torch.int16), v_before.view(torch.int16))
    want = hc.hadacore_fwht(ref_in)
    assert torch.equal(qkv[:, 0:2].contiguous().view(torch.int16), want.view(torch.int16))
    got = widen(qkv[:, 0:2].reshape(-1, d))
    assert rel_l2_rows(got, oracle.fwht(widen(ref_in.reshape(-1, d)))).max() <= TOL[dtype]


@pytest.mark.parametrize("d", [16, 128, 2048])
def test_fwht_functional_on_strided_view_no_copy(hc, d, monkeypatch):
    """fwht on a strided view takes the strided entry (no .contiguous() copy of the input)."""
    h = max(1, 512 // d)
    qkv = qkv_buffer(19, h, d, torch.bfloat16, 52)
    view = qkv[:, 0:2]
    want = hc.hadacore_fwht(view.contiguous())
    calls = []
    real = torch.Tensor.contiguous

    def spy(self, *a, **k):
        calls.append(tuple(self.shape))
        return real(self, *a, **k)
    monkeypatch.setattr(torch.Tensor, "contiguous", spy)
    y = torch.ops.hadacore.fwht(view, None)
    monkeypatch.setattr(torch.Tensor, "contiguous", real)
    assert not [c for c in calls if c == tuple(view.shape)], calls
    assert y.is_contiguous() and y.shape == view.shape
    assert torch.equal(y.view(torch.int16), want.view(torch.int16))


@pytest.mark.parametrize("d", [8, 32, 64, 128, 4096])
@pytest.mark.parametrize("qtype", ["e4m3", "int8", "int4"])
def test_fwht_quant_strided_every_n(hc, d, qtype):
    """fwht_quant on qkv[:, 0:2] uses the strided entry for n >= 8 and equals the
    contiguous entry on a copy, bitwise."""
    h = max(1, 512 // d)
    qkv = qkv_buffer(23, h, d, torch.float16, 53)
    q, s = torch.ops.hadacore.fwht_quant(qkv[:, 0:2], qtype, None)
    q2, s2 = hc.hadacore_fwht_quant(qkv[:, 0:2].contiguous(), qtype)
    assert torch.equal(q.view(torch.uint8), q2.view(torch.uint8)) and torch.equal(s, s2)


def test_torch_compile_fullgraph_on_qkv_view(hc):
    """torch.compile(fullgraph=True) traces both ops on a QKV view; results equal eager bitwise."""
    d, h = 128, 8
    qkv = qkv_buffer(29, h, d, torch.bfloat16, 54)

    def rotate(t):
        return torch.ops.hadacore.fwht(t[:, 0:2], None)

    def rotate_inplace(t):
        torch.ops.hadacore.fwht_(t[:, 0:2], None)
        return t

    def rotate_quant(t):
        return torch.ops.hadacore.fwht_quant(t[:, 0:2], "e4m3", None)

    eager = rotate(qkv)
    comp = torch.compile(rotate, fullgraph=True)(qkv)
    assert torch.equal(comp.view(torch.int16), eager.view(torch.int16))
    qe, se = rotate_quant(qkv)
    qc, sc = torch.compile(rotate_quant, fullgraph=True)(qkv)
    assert torch.equal(qc.view(torch.uint8), qe.view(torch.uint8)) and torch.equal(sc, se)
    a, b = qkv.clone(), qkv.clone()
    rotate_inplace(a)
    out = torch.compile(rotate_inplace, fullgraph=True)(b)
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
    assert torch.equal(out.view(torch.int16), a.view(torch.int16))
    assert torch.equal(a[:, 2].view(torch.int16), qkv[:, 2].view(torch.int16))


def test_fake_impl_is_contiguous(hc):
    """The fake (meta) output of hadacore::fwht has the real op's contiguous strides."""
    from torch._subclasses.fake_tensor import FakeTensorMode
    x = torch.empty(64, 4, 256, dtype=torch.float16, device="cuda").transpose(0, 1)
    with FakeTensorMode() as mode:
        fx = mode.from_tensor(x)
        fy = torch.ops.hadacore.fwht(fx, None)
        assert fy.is_contiguous() and tuple(fy.shape) == tuple(x.shape)
    y = torch.ops.hadacore.fwht(x.contiguous(), None)
    assert y.is_contiguous()


def test_binding_rejects_foreign_device_buffers(hc):
    """out / row_scale on another device (here: the CPU) raise before any launch."""
    x = synthetic.generate(8, 256, torch.float16, 55).cuda()
    with pytest.raises(hc.HadacoreError) as e:
        hc.hadacore_fwht_strided(x, out=torch.empty(8, 256, dtype=torch.float16))
    assert e.value.code == hc.ARG_ERROR
    with pytest.raises(hc.HadacoreError) as e:
        hc.hadacore_fwht_quant(x, "e4m3", row_scale=torch.empty(8, dtype=torch.float32))
    assert e.value.code == hc.ARG_ERROR
    with pytest.raises(hc.HadacoreError) as e:
        hc.hadacore_fwht_quant_strided(x, "int8", row_scale=torch.empty(8, dtype=torch.float32))
    assert e.value.code == hc.ARG_ERROR
    with pytest.raises(hc.HadacoreError) as e:
        hc.hadacore_fwht(x, out=torch.empty(8, 256, dtype=torch.float16))
    assert e.value.code == hc.ARG_ERROR
    torch.cuda.synchronize()  # nothing was launched, the context is healthy
    assert torch.isfinite(hc.hadacore_fwht(x).float()).all()


@pytest.mark.parametrize("scale", [0.0, -1.0, float("nan")])
def test_nonpositive_scale_rejected(hc, scale):
    """scale > 0 (a zero scale broke the quantization contract)."""
    x = synthetic.generate(8, 256, torch.float16, 56).cuda()
    for f in (lambda: hc.hadacore_fwht(x, scale=scale), lambda: hc.hadacore_fwht_quant(x, "e4m3", scale=scale),
              lambda: hc.hadacore_fwht_strided(x, scale=scale),
              lambda: hc.hadacore_fwht_quant_strided(x, "int4", scale=scale)):
        with pytest.raises(hc.HadacoreError) as e:
            f()
        assert e.value.code == 7
