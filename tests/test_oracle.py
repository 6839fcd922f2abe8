"""Pins for the fp64 CPU oracle (oracle/), run without a GPU.

The oracle must be pinned to something other than itself (task rule 3).  Each
test below checks it against what PAPER.md / the mathematics fix:

* brute force: an explicit Sylvester matrix built here by the recursion of P:45
  [Sec. 2.2] (H(2k) = [[H, H], [H, -H]]) and a dense fp64 matmul, n <= 1024;
* an independent library: scipy.linalg.hadamard (natural/Sylvester order);
* worked examples with exact values (tests/golden/spec_examples.json, each cited);
* closed forms: H e0 = 1/sqrt(n) 1 and H 1 = sqrt(n) e0 for every n = 2..2^15;
* invariants: involution (H H = I, normalized), norm preservation, dyadic shift,
  bit-permutation invariance, thread-count invariance;
* the listing with the paper's literal per-iteration /sqrt(2), for the
  scale-placement reading R3.

A plausible mistake (dropped butterfly, wrong sign, wrong stride, transposed
operand, wrong normalization) fails the Sylvester / scipy comparisons.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg

import oracle
import synthetic

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def sylvester(n: int) -> np.ndarray:
    """Explicit Sylvester Hadamard by recursion: H(2k) = [[H, H], [H, -H]]."""
    h = np.array([[1.0]])
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    return h


def rng_matrix(m, n, seed):
    return np.random.default_rng(seed).standard_normal((m, n))


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024])
def test_listing_matches_explicit_sylvester_matmul(n):
    x = rng_matrix(8, n, 7 + n)
    y = oracle.fwht(x)
    ref = (x @ sylvester(n)) / math.sqrt(n)      # right-Hadamard x H; H symmetric
    assert np.max(np.abs(y - ref)) <= 1e-10 * np.max(np.abs(x))


@pytest.mark.parametrize("n", [2, 16, 128, 1024])
def test_listing_matches_scipy_hadamard(n):
    x = rng_matrix(5, n, 11 + n)
    y = oracle.fwht(x, scale=1.0)
    ref = x @ scipy.linalg.hadamard(n).astype(np.float64)
    assert np.max(np.abs(y - ref)) <= 1e-10 * np.max(np.abs(ref))


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64, 128, 256])
def test_dense_definition_is_sylvester_exhaustive(n):
    # oracle.dense applied to I_n yields the whole matrix; compare every entry
    # against the recursion (exhaustive sign rule check, n <= 256).
    eye = np.eye(n)
    assert np.array_equal(oracle.dense(eye, scale=1.0), sylvester(n))
    assert np.array_equal(oracle.fwht(eye, scale=1.0), sylvester(n))


def test_golden_worked_examples():
    cases = json.load(open(GOLDEN))["cases"]
    for c in cases:
        n = c["n"]
        x = c["x"]
        if x == "onehot0":
            x = np.zeros(n); x[0] = 1.0
        elif x == "ones":
            x = np.ones(n)
        x = np.asarray(x, dtype=np.float64)
        y = c["y"]
        if isinstance(y, str) and y.startswith("const:"):
            y = np.full(n, float(y.split(":")[1]))
        elif isinstance(y, str) and y.startswith("e0:"):
            v = float(y.split(":")[1]); y = np.zeros(n); y[0] = v
        y = np.asarray(y, dtype=np.float64)
        got = oracle.fwht(x, scale=c["scale"])[0]
        assert np.allclose(got, y, rtol=0, atol=1e-12 * max(1.0, np.abs(y).max())), c["id"]
        got_d = oracle.dense(x, scale=c["scale"])[0]
        assert np.allclose(got_d, y, rtol=0, atol=1e-12 * max(1.0, np.abs(y).max())), c["id"]


@pytest.mark.parametrize("k", range(1, 16))
def test_closed_forms_e0_and_ones(k):
    n = 1 << k
    e0 = np.zeros((1, n)); e0[0, 0] = 1.0
    y = oracle.fwht(e0)[0]
    assert np.all(y == 1.0 / math.sqrt(n))                 # H e0 = (1/sqrt n) 1, exactly
    ones = np.ones((1, n))
    y1 = oracle.fwht(ones)[0]
    assert abs(y1[0] - math.sqrt(n)) <= 1e-12 * math.sqrt(n)   # H 1 = sqrt(n) e0
    assert np.all(y1[1:] == 0.0)


@pytest.mark.parametrize("n", [128, 4096, 32768])
def test_involution_and_norm(n):
    x = rng_matrix(3, n, 5)
    y = oracle.fwht(x)
    assert np.allclose(np.linalg.norm(y, axis=1), np.linalg.norm(x, axis=1), rtol=1e-12)
    xx = oracle.fwht(y)
    assert np.max(np.abs(xx - x)) <= 1e-12 * np.max(np.abs(x)) * 10


@pytest.mark.parametrize("n", [256, 8192])
def test_dyadic_shift_invariant(n):
    # x'(j) = x(j xor s)  =>  y'(l) = (-1)^popcount(s & l) y(l)
    x = rng_matrix(2, n, 3)
    s = 0b1011011 % n
    idx = np.arange(n)
    y = oracle.fwht(x)
    y2 = oracle.fwht(x[:, idx ^ s])
    sign = np.array([-1.0 if bin(s & l).count("1") % 2 else 1.0 for l in range(n)])
    assert np.max(np.abs(y2 - sign * y)) <= 1e-12 * np.max(np.abs(y)) * 10


def test_bit_permutation_invariant():
    # x'(j) = x(pi(j)) for a permutation pi of index bits  =>  y' = y o pi
    n, k = 1024, 10
    perm = [3, 7, 0, 9, 1, 5, 2, 8, 6, 4]
    idx = np.arange(n)
    pj = np.zeros(n, dtype=np.int64)
    for b in range(k):
        pj |= ((idx >> b) & 1) << perm[b]
    x = rng_matrix(2, n, 9)
    y = oracle.fwht(x)
    y2 = oracle.fwht(x[:, pj])
    assert np.max(np.abs(y2 - y[:, pj])) <= 1e-12 * np.max(np.abs(y)) * 10


def test_dense_entry_samples_match_listing_large_n():
    n = 32768
    x = rng_matrix(1, n, 13)
    y = oracle.fwht(x)[0]
    for l in [0, 1, 2, 255, 256, 4097, 16384, n - 1]:
        assert abs(oracle.dense_entry(x[0], l) - y[l]) <= 1e-11 * np.max(np.abs(y))


def test_thread_count_invariance_bitwise():
    x = rng_matrix(37, 2048, 21)
    a = oracle.fwht(x, threads=1)
    b = oracle.fwht(x, threads=7)
    assert np.array_equal(a, b)


def test_in_place_argument_order_irrelevant():
    # scale applied once at the end equals the listing's per-iteration /sqrt(2)
    # -- DESIGN.md reading R3 -- checked against a literal transcription of
    # the P:50-64 listing on tiny inputs.
    def listing_literal(a):
        a = list(a)
        h = 1
        while h < len(a):
            for i in range(0, len(a), h * 2):
                for j in range(i, i + h):
                    x, y = a[j], a[j + h]
                    a[j], a[j + h] = x + y, x - y
            a = [v / math.sqrt(2) for v in a]
            h *= 2
        return np.array(a)

    for n in [2, 8, 64]:
        x = rng_matrix(1, n, n)[0]
        assert np.allclose(oracle.fwht(x)[0], listing_literal(x), rtol=0, atol=1e-13 * n)


def test_rejects_bad_sizes():
    with pytest.raises(ValueError):
        oracle.fwht(np.zeros((2, 100)))
    with pytest.raises(ValueError):
        oracle.dense(np.zeros((2, 12)))
    assert oracle.fwht(np.zeros((0, 64))).shape == (0, 64)


# ---------------------------------------------------------------- quantization oracle
# Pins for oracle.quantize_rows / e4m3.

def test_e4m3_codes_match_torch_float8():
    # an independent implementation (torch.float8_e4m3fn, RNE) over the finite range
    import torch
    x = np.concatenate([np.random.default_rng(1).standard_normal(20000) * s for s in (1e-3, 0.1, 1, 10, 100)])
    # fp32-representable inputs: torch converts via fp32, which would double-round fp64 values
    x = x[np.abs(x) <= 448].astype(np.float32).astype(np.float64)
    ours = np.array([oracle.e4m3_encode(v) for v in x], dtype=np.uint8)
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(ours, ref)
    # every finite code round-trips ("identity on all valid codes")
    for c in list(range(0, 0x7F)) + list(range(0x80, 0xFF)):
        v = oracle.e4m3_value(c)
        assert oracle.e4m3_value(oracle.e4m3_encode(v)) == v


def test_e4m3_worked_values_and_saturation():
    assert oracle.e4m3_value(oracle.e4m3_encode(30.0)) == 30.0      # S:284 exact
    assert oracle.e4m3_encode(448.0) == 0x7E                         # max finite
    assert oracle.e4m3_encode(1e6) == 0x7E and oracle.e4m3_encode(-1e6) == 0xFE   # satfinite
    assert oracle.e4m3_encode(1.0) == 0x38
    assert oracle.e4m3_value(0x01) == 2.0 ** -9                      # smallest subnormal


def test_quantize_rows_closed_forms():
    # max_abs = 127 -> scale 1, integers round-trip exactly
    y = np.array([[127.0, -3.0, 0.0, 64.0]])
    codes, s = oracle.quantize_rows(y, "int8")
    assert s[0] == 1.0 and list(codes[0].view(np.int8)) == [127, -3, 0, 64]
    # [448, 0] in e4m3 round-trips exactly
    codes, s = oracle.quantize_rows(np.array([[448.0, 0.0]]), "e4m3")
    assert s[0] == 1.0 and list(codes[0]) == [0x7E, 0x00]
    # all-zero row: scale 1, zero codes (S:431 AllZeroInput)
    codes, s = oracle.quantize_rows(np.zeros((1, 8)), "int8")
    assert s[0] == 1.0 and not codes.any()
    # ties to even: 2.5 -> 2, 3.5 -> 4 (scale 1 via a 127 anchor)
    codes, _ = oracle.quantize_rows(np.array([[127.0, 2.5, 3.5, -2.5]]), "int8")
    assert list(codes[0].view(np.int8)) == [127, 2, 4, -2]


def test_quantization_error_bounds_on_random_rows():
    rng = np.random.default_rng(3)
    y = rng.standard_normal((20, 1024))
    for qtype in ("int8", "e4m3"):
        codes, s = oracle.quantize_rows(y, qtype)
        deq = oracle.dequantize_rows(codes, s, qtype)
        err = np.abs(deq - y)
        if qtype == "int8":
            assert np.all(err <= s[:, None] / 2 + 1e-12)
        else:  # relative 2^-4 in the normal range, half the subnormal spacing below it
            assert np.all(err <= np.abs(y) * 2.0 ** -4 + s[:, None] * 2.0 ** -10 + 1e-12)
        assert np.allclose(np.abs(deq).max(axis=1), np.abs(y).max(axis=1))   # the max is exact


# ---------------------------------------------------------------- quant_lab oracle (NEXT-4)
# Pins for oracle.quantize (INT4, per-tensor) and oracle.lab_trial: SPEC quant_lab
# S:397-440 worked examples, closed forms and invariants.

def test_quantize_int4_closed_forms_and_ties():
    # scale 1 via a 7 anchor: ties to even, clamp never needed below max_abs
    codes, s = oracle.quantize(np.array([[7.0, 2.5, 3.5, -2.5, 0.5, 1.5, -7.0]]), "int4")
    assert s[0] == 1.0 and list(codes[0].view(np.int8)) == [7, 2, 4, -2, 0, 2, -7]
    # S:427 single outlier 100 among unit-scale values, INT4: scale 100/7 ~ 14.3, the
    # bulk collapses to 0 after the round trip, the outlier survives
    row = np.concatenate([[100.0], np.linspace(-1.0, 1.0, 63)])[None, :]
    codes, s = oracle.quantize(row, "int4")
    assert s[0] == 100.0 / 7.0
    deq = oracle.fake_quant(row, "int4")
    assert np.all(deq[0, 1:] == 0.0) and abs(deq[0, 0] - 100.0) <= 1e-12


def test_quantize_per_tensor():
    # max_abs = 127 somewhere in the matrix, INT8 PerTensor -> scale 1.0 for every
    # row and integers round-trip exactly (per row they would not: row 1's max is 5)
    x = np.array([[127.0, -3.0, 0.0, 64.0], [5.0, -5.0, 1.0, 2.0]])
    codes, s = oracle.quantize(x, "int8", per_tensor=True)
    assert np.all(s == 1.0)
    assert np.array_equal(oracle.fake_quant(x, "int8", per_tensor=True), x)
    _, s_row = oracle.quantize(x, "int8")
    assert s_row[1] == 5.0 / 127.0
    # one row: per-tensor == per-row; brute-force tensor max on a random matrix
    rng = np.random.default_rng(5)
    r = rng.standard_normal((1, 256))
    for q in ("e4m3", "int8", "int4"):
        assert np.array_equal(oracle.fake_quant(r, q, True), oracle.fake_quant(r, q, False))
    big = rng.standard_normal((7, 64)) * np.arange(1, 8)[:, None]
    _, st = oracle.quantize(big, "int4", per_tensor=True)
    assert np.all(st == max(abs(v) for v in big.ravel()) / 7.0)


def test_fake_quant_error_bounds_all_targets():
    rng = np.random.default_rng(9)
    x = rng.standard_normal((16, 512)) * np.exp(rng.standard_normal((16, 1)))
    for per_tensor in (False, True):
        for q in ("int8", "int4"):
            codes, s = oracle.quantize(x, q, per_tensor)
            deq = oracle.dequantize_rows(codes, s, q)
            assert np.all(np.abs(deq - x) <= s[:, None] / 2 * (1 + 1e-12))   # S:421 "scale/2 per entry"
            assert np.all(np.abs(codes.view(np.int8)) <= oracle.QMAX[q])
        deq = oracle.fake_quant(x, "e4m3", per_tensor)
        _, s = oracle.quantize(x, "e4m3", per_tensor)
        assert np.all(np.abs(deq - x) <= np.abs(x) * 2.0 ** -4 + s[:, None] * 2.0 ** -10 + 1e-12)


def test_lab_trial_closed_forms():
    # x = c e0 (one row): the rotated row is constant c/sqrt(d) -> max_abs exactly that,
    # and every rotated entry is exactly representable after scaling: no rotated error
    for d in (16, 256, 4096):
        c = 3.0
        x = np.zeros((1, d)); x[0, 0] = c
        t = oracle.lab_trial(x, "int4")
        assert abs(t["max_abs_rotated"] - c / np.sqrt(d)) <= 1e-15 * c
        assert t["max_abs_plain"] == c and t["mse_plain"] == 0.0
        assert t["mse_rotated"] <= 1e-28
    # rotation alone (no quantization) is reproduced to 1e-10 by the inverse rotation
    x = synthetic.outlier_matrix(8, 1024, 3).double().numpy()
    assert np.max(np.abs(oracle.fwht(oracle.fwht(x)) - x)) <= 1e-10


def test_lab_trial_parseval_and_direction():
    # the inverse-rotated error equals the rotated-domain error (H orthogonal): an
    # independent check of the inverse-rotation step
    x = synthetic.outlier_matrix(16, 1024, 11).double().numpy()
    for q in ("int4", "int8", "e4m3"):
        t = oracle.lab_trial(x, q)
        y = oracle.fwht(x)
        rot_dom = float(np.mean((oracle.fake_quant(y, q) - y) ** 2))
        assert abs(t["mse_rotated"] - rot_dom) <= 1e-9 * rot_dom
    # S:438 (DERIVED; direction fixed by P:24 Sec. 1's outlier argument): outlier_rate 1e-3,
    # outlier_scale 100, INT4 per row -> rotated error below plain in >= 95 % of 100 trials
    wins = 0
    for trial in range(100):
        xt = synthetic.outlier_matrix(64, 1024, 1000 + trial).double().numpy()
        t = oracle.lab_trial(xt, "int4")
        wins += t["mse_rotated"] < t["mse_plain"]
        assert t["max_abs_rotated"] <= t["max_abs_plain"]
    assert wins >= 95
