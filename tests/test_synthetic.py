"""The shared seeded input generator (synthetic/): determinism, sharding invariance,
and the splitmix64 bit patterns against an independent numpy uint64 transcription."""
import numpy as np
import torch

import synthetic


def _splitmix_np(v):
    v = (v + np.uint64(0x9E3779B97F4A7C15))
    v = (v ^ (v >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    v = (v ^ (v >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return v ^ (v >> np.uint64(31))


def test_splitmix64_bits_match_numpy_uint64():
    x = torch.arange(-500, 500, dtype=torch.int64) * 1234567891
    got = synthetic.splitmix64(x).numpy().view(np.uint64)
    with np.errstate(over="ignore"):
        ref = _splitmix_np(x.numpy().view(np.uint64))
    assert np.array_equal(got, ref)


def test_deterministic_and_shard_invariant():
    seed = synthetic.seed_for(2, torch.bfloat16)
    full = synthetic.generate(40, 512, torch.bfloat16, seed, dist="D1")
    again = synthetic.generate(40, 512, torch.bfloat16, seed, dist="D1")
    assert torch.equal(full.view(torch.int16), again.view(torch.int16))
    part = synthetic.generate(13, 512, torch.bfloat16, seed, dist="D1", row0=17, chunk_elems=1000)
    assert torch.equal(full[17:30].view(torch.int16), part.view(torch.int16))


def test_distributions_shape():
    a = synthetic.generate(256, 1024, torch.float32, 5).double()
    assert abs(a.mean().item()) < 0.01 and abs(a.std().item() - 1.0) < 0.01
    b = synthetic.generate(256, 1024, torch.float16, 5, dist="D1")
    frac = (b.abs() == 100).double().mean().item()
    assert 0.0005 < frac < 0.002
    assert torch.isfinite(b).all()
