"""Lane-level model of the mma.sync m16n8k16 fragment algebra used by the kernels.

Design tool (not a test oracle, not on the product path).  It models the PTX ISA
register layouts of mma.m16n8k16 (.f16/.bf16 A/B, f16/f32 C/D) and checks, with
numpy, that the stage sequences chosen in paper_2412_08832_b200/csrc/fwht_kernel.cuh
compute H_n on each row, which element sits in which (lane, register, half) slot
before/after each stage, and that the shared-memory access patterns are free of
bank conflicts.

Slot = (lane, reg, half); lane = 4*g + t.  A-layout register roles:
  R0 = M[g][2t+h], R1 = M[g+8][2t+h], R2 = M[g][2t+8+h], R3 = M[g+8][2t+8+h]
B layout (k16 x n8): B0 = B[2t+h][g], B1 = B[2t+8+h][g]
D layout (m16 x n8): D0 = D[g][2t+h], D1 = D[g+8][2t+h]
"""
from __future__ import annotations

import itertools

import numpy as np

LANES = 32


def a_slot(r, c):
    """(lane, reg, half) holding M[r][c] in the A layout."""
    g, t, h = r % 8, (c % 8) // 2, c % 2
    reg = (1 if r >= 8 else 0) + (2 if c >= 8 else 0)
    return 4 * g + t, reg, h


def stage_const_a(vals, A, roles):
    """D_T = A @ B_T with B_T built from registers roles[2T], roles[2T+1].

    vals: array [32 lanes, 4 regs, 2 halves] of floats (or labels, object).
    returns Y [32, 4, 2] with Y[:,2T+0] = D_T rows 0..7, Y[:,2T+1] = rows 8..15.
    """
    out = np.zeros_like(vals)
    for T in range(2):
        B = np.zeros((16, 8), dtype=vals.dtype)
        for k in range(16):
            for n in range(8):
                lane = 4 * n + (k % 8) // 2
                reg = roles[2 * T] if k < 8 else roles[2 * T + 1]
                B[k, n] = vals[lane, reg, k % 2]
        D = A @ B
        for i in range(16):
            for n in range(8):
                lane = 4 * (i % 8) + n // 2
                out[lane, 2 * T + (1 if i >= 8 else 0), n % 2] = D[i, n]
    return out


def stage_data_a(vals, Bc):
    """D = M @ Bc with M (16x16) the data in A layout, Bc a 16x16 constant."""
    M = np.zeros((16, 16), dtype=vals.dtype)
    for r in range(16):
        for c in range(16):
            lane, reg, h = a_slot(r, c)
            M[r, c] = vals[lane, reg, h]
    D = M @ Bc
    out = np.zeros_like(vals)
    for r in range(16):
        for c in range(16):
            lane, reg, h = a_slot(r, c)
            out[lane, reg, h] = D[r, c]
    return out


def label_stage_const_a(labels, roles):
    """Where labels go through stage_const_a (label of B_T[i][n] lands at D_T[i][n])."""
    out = np.empty_like(labels)
    contracted = {}  # (T, n) -> list of labels by k
    for T in range(2):
        for n in range(8):
            for i in range(16):
                lane_in = 4 * n + (i % 8) // 2
                reg_in = roles[2 * T] if i < 8 else roles[2 * T + 1]
                lane_out = 4 * (i % 8) + n // 2
                out[lane_out, 2 * T + (1 if i >= 8 else 0), n % 2] = labels[lane_in, reg_in, i % 2]
    return out


def kron_const(bits_kind, scale):
    """16x16 matrix = scale * kron over 4 K-bits (bit3..bit0) of H2 ('H') or I2 ('I').

    bits_kind[q] describes K-bit q (q = 0 is the LSB of the 16-index)."""
    H2 = np.array([[1.0, 1.0], [1.0, -1.0]])
    I2 = np.eye(2)
    M = np.array([[1.0]])
    for q in reversed(range(4)):
        M = np.kron(M, H2 if bits_kind[q] == "H" else I2)
    return scale * M


# K-bit q of the A-const stage (k = 2t + h + 8*[second reg]):
#   q0 = h, q1 = t0, q2 = t1, q3 = second-register bit.
# K-bit q of the data-as-A stage (k = M column = 2t + h + 8*[R2/R3]): same roles.


def sylvester(n):
    h = np.array([[1.0]])
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    return h


def check_n256():
    """One 256-chunk per warp, LDS.128: lane l holds elements 8l..8l+7, X_j = (8l+2j, +1)."""
    x = np.random.default_rng(0).standard_normal(256)
    vals = np.zeros((32, 4, 2))
    lab = np.zeros((32, 4, 2), dtype=np.int64)
    for l in range(32):
        for j in range(4):
            for h in range(2):
                e = 8 * l + 2 * j + h
                vals[l, j, h] = x[e]
                lab[l, j, h] = e
    A = kron_const("HHHH", 0.25)
    roles = (0, 2, 1, 3)
    v1 = stage_const_a(vals, A, roles)
    l1 = label_stage_const_a(lab, roles)
    v2 = stage_const_a(v1, A, roles)
    l2 = label_stage_const_a(l1, roles)
    assert np.array_equal(l2, lab), "n=256 orientation does not return to natural"
    y = sylvester(256) @ x / 16.0
    got = np.zeros(256)
    for l in range(32):
        for j in range(4):
            for h in range(2):
                got[l2[l, j, h]] = v2[l, j, h]
    assert np.allclose(got, y), "n=256 values wrong"
    return "n=256 ok (roles (0,2,1,3) both stages, output slots == input slots)"


def check_n128():
    """Two rows per fragment: X0, X2 = row A elements 4l..4l+3; X1, X3 = row B."""
    rng = np.random.default_rng(1)
    xa, xb = rng.standard_normal(128), rng.standard_normal(128)
    vals = np.zeros((32, 4, 2))
    lab = np.zeros((32, 4, 2), dtype=np.int64)  # label = row*128 + e
    for l in range(32):
        for h in range(2):
            vals[l, 0, h] = xa[4 * l + h]; lab[l, 0, h] = 4 * l + h
            vals[l, 2, h] = xa[4 * l + 2 + h]; lab[l, 2, h] = 4 * l + 2 + h
            vals[l, 1, h] = xb[4 * l + h]; lab[l, 1, h] = 128 + 4 * l + h
            vals[l, 3, h] = xb[4 * l + 2 + h]; lab[l, 3, h] = 128 + 4 * l + 2 + h
    # stage a: roles (0,2,1,3): K bits = h(e0), t0(e2), t1(e3), X2/X0(e1) -> H16
    A1 = kron_const("HHHH", 0.25)
    v1 = stage_const_a(vals, A1, (0, 2, 1, 3))
    l1 = label_stage_const_a(lab, (0, 2, 1, 3))
    # stage b: roles (0,1,2,3): K = h'(g0), t0'(g1), t1'(g2), Y1/Y0 (= stage-a i>=8 = e1) -> H8 (x) I2
    A2 = kron_const("HHHI", 0.5)
    v2 = stage_const_a(v1, A2, (0, 1, 2, 3))
    l2 = label_stage_const_a(l1, (0, 1, 2, 3))
    # check rows separated and values
    ya = sylvester(128) @ xa / 8.0
    yb = sylvester(128) @ xb / 8.0
    got = np.zeros(256)
    for l in range(32):
        for j in range(4):
            for h in range(2):
                got[l2[l, j, h]] = v2[l, j, h]
    assert np.allclose(got[:128], ya * np.sqrt(2) / np.sqrt(2)) or True
    # scale: stage a 1/4, stage b 1/2 -> 1/8 = 1/sqrt(128) * (sqrt(128)/8) ; exact H/8 expected
    assert np.allclose(got[:128], sylvester(128) @ xa / 8.0 * 1.0), "row A wrong"
    assert np.allclose(got[128:], sylvester(128) @ xb / 8.0), "row B wrong"
    # isolation: row B labels never mixed -> check structurally by NaN propagation
    vals_nan = vals.copy()
    vals_nan[5, 0, 1] = np.inf  # row A element
    w1 = stage_const_a(vals_nan, A1, (0, 2, 1, 3))
    w2 = stage_const_a(w1, A2, (0, 1, 2, 3))
    out_rows = {}
    for l in range(32):
        for j in range(4):
            for h in range(2):
                out_rows[l2[l, j, h]] = w2[l, j, h]
    rowb = np.array([out_rows[128 + e] for e in range(128)])
    assert np.all(np.isfinite(rowb)), "NaN/Inf leaked into the partner row"
    # output slot map
    omap = {(l, j, h): int(l2[l, j, h]) for l in range(32) for j in range(4) for h in range(2)}
    return omap


def show_n128_map():
    omap = check_n128()
    lines = []
    for l in [0, 1, 2, 3, 4, 5, 8, 31]:
        lines.append(f"lane {l:2d}: " + " ".join(f"Y{j}=({omap[(l, j, 0)]},{omap[(l, j, 1)]})" for j in range(4)))
    return "\n".join(lines)


if __name__ == "__main__":
    print(check_n256())
    print("n=128 output slots:")
    print(show_n128_map())


# ---------------------------------------------------------------------------
# Whole-row model for n >= 512: phase 1 (per 256-chunk), swizzled smem exchange,
# phase 2 over the chunk bits, phase 3 copy-out.  Mirrors fwht_kernel.cuh.
# ---------------------------------------------------------------------------
LANE_SLOTS = ["t0", "t1", "g0", "g1", "g2"]   # lane bit i <-> slot LANE_SLOTS[i]


def phase2_plan(q):
    """Slot assignment for q = log2(n/256) chunk bits."""
    if q <= 3:
        chunk_slots = ["r2", "t0", "t1"][:q]
        single = True
    else:
        chunk_slots = ["r1", "r2", "g0", "g1", "g2", "t0", "t1"][:q]
        single = False
    pos_lane = [s for s in LANE_SLOTS if s not in chunk_slots]
    pos_reg = [s for s in ["r1"] if s not in chunk_slots] if single else \
        [s for s in ["r1", "r2"] if s not in chunk_slots]
    word_slots = pos_lane + pos_reg            # word bits 0.. in this order
    nfrag_bits = 7 - len(word_slots)
    lane_chunk = [s for s in LANE_SLOTS if s in chunk_slots]
    return dict(single=single, chunk_slots=chunk_slots, word_slots=word_slots,
                nfrag_bits=nfrag_bits, lane_chunk=lane_chunk, a=len(pos_lane))


def slot_bits(lane, j):
    t, g = lane & 3, lane >> 2
    return {"t0": t & 1, "t1": (t >> 1) & 1, "g0": g & 1, "g1": (g >> 1) & 1, "g2": (g >> 2) & 1,
            "r1": j & 1, "r2": (j >> 1) & 1}


def swz(plan, c):
    f = 0
    for rank, s in enumerate(plan["lane_chunk"]):
        i = plan["chunk_slots"].index(s)
        f |= ((c >> i) & 1) << (plan["a"] + rank)
    return f


def p2_addr(plan, lane, j, frag):
    """(chunk, word) read by (lane, reg j) in phase-2 fragment `frag`."""
    b = slot_bits(lane, j)
    c = 0
    for i, s in enumerate(plan["chunk_slots"]):
        c |= b[s] << i
    w = 0
    for i, s in enumerate(plan["word_slots"]):
        w |= b[s] << i
    w |= frag << len(plan["word_slots"])
    return c, w


def fwht_np(x):
    x = x.copy()
    n = x.shape[-1]
    h = 1
    while h < n:
        x = x.reshape(-1, n // (2 * h), 2, h)
        a, b = x[:, :, 0, :].copy(), x[:, :, 1, :].copy()
        x[:, :, 0, :], x[:, :, 1, :] = a + b, a - b
        x = x.reshape(-1, n)
        h *= 2
    return x


def stage_kinds(plan):
    """A/B constants: list of (form, kinds q0..q3)."""
    cs = plan["chunk_slots"]
    if plan["single"]:
        # data-as-A: contracted column bits q0=h, q1=t0, q2=t1, q3=r2
        return [("dataA", "".join("H" if s in cs else "I" for s in ["h", "t0", "t1", "r2"]))]
    a = "".join("H" if s in cs else "I" for s in ["h", "t0", "t1", "r2"])
    b = "".join("H" if s in cs else "I" for s in ["g0", "g1", "g2", "r1"])
    return [("constA", a), ("constA", b)]


def pow2_scale(kinds):
    hb = kinds.count("H")
    return 2.0 ** (-(hb // 2)), hb


def check_row(n, seed=0):
    k = n.bit_length() - 1
    q = k - 8
    C = 1 << q
    plan = phase2_plan(q)
    x = np.random.default_rng(seed).standard_normal(n)
    smem = np.zeros(n)  # element-indexed words: word w of chunk c holds elements 2w,2w+1 at [c*256 + 2*(w^f)]
    E = 0  # accumulated exponent of the per-stage power-of-two normalization
    A256 = kron_const("HHHH", 0.25)
    # phase 1
    for c in range(C):
        f = swz(plan, c)
        vals = np.zeros((32, 4, 2))
        for l in range(32):
            for j in range(4):
                w = l + 32 * j
                vals[l, j] = x[c * 256 + 2 * w: c * 256 + 2 * w + 2]
        v = stage_const_a(stage_const_a(vals, A256, (0, 2, 1, 3)), A256, (0, 2, 1, 3))
        for l in range(32):
            for j in range(4):
                w = (l + 32 * j) ^ f
                smem[c * 256 + 2 * w: c * 256 + 2 * w + 2] = v[l, j]
    E += 4
    # phase 2
    kinds = stage_kinds(plan)
    conflicts = 0
    for frag in range(1 << plan["nfrag_bits"]):
        vals = np.zeros((32, 4, 2))
        for j in range(4):
            banks = set()
            for l in range(32):
                c, w = p2_addr(plan, l, j, frag)
                ww = w ^ swz(plan, c)
                banks.add(ww % 32)
                vals[l, j] = smem[c * 256 + 2 * ww: c * 256 + 2 * ww + 2]
            conflicts += 32 - len(banks)
        for form, kd in kinds:
            s, _ = pow2_scale(kd)
            M = kron_const(kd, s)
            vals = stage_data_a(vals, M) if form == "dataA" else stage_const_a(vals, M, (0, 2, 1, 3))
        for l in range(32):
            for j in range(4):
                c, w = p2_addr(plan, l, j, frag)
                ww = w ^ swz(plan, c)
                smem[c * 256 + 2 * ww: c * 256 + 2 * ww + 2] = vals[l, j]
    for form, kd in kinds:
        E += kd.count("H") // 2
    # phase 3 (un-swizzle)
    y = np.zeros(n)
    for c in range(C):
        f = swz(plan, c)
        for l in range(32):
            for j in range(4):
                w = l + 32 * j
                ww = w ^ f
                y[c * 256 + 2 * w: c * 256 + 2 * w + 2] = smem[c * 256 + 2 * ww: c * 256 + 2 * ww + 2]
    ref = fwht_np(x[None, :])[0] * 2.0 ** (-E)
    ok = np.allclose(y, ref)
    return ok, conflicts, plan, kinds, E


def main_rows():
    for k in range(9, 16):
        ok, conf, plan, kinds, E = check_row(1 << k)
        print(f"n={1<<k:6d} ok={ok} bank_conflicts={conf} stages={kinds} E={E} "
              f"a={plan['a']} frags={1<<plan['nfrag_bits']} chunk_slots={plan['chunk_slots']} word_slots={plan['word_slots']}")


# ---------------------------------------------------------------------------
# Design "L" (ldmatrix/stmatrix .trans, 16-byte granules): phase 1 LDS.128/STS.128,
# phase 2 LDSM.T.x4 -> mma -> STSM.T.x4, phase 3 LDS.128/STG.128.
# Granule = 8 consecutive elements (16 B); a chunk (256 el) has 32 granules.
# Swizzle: granule' = granule ^ (chunk & ((1 << min(q,3)) - 1)).
# Phase-2 row slots: lane L = 8*j + r provides the row address of (matrix j, row r);
# slot bits r0, r1, r2, j0, j1, then fragment-index bits f0, f1, ...
# ---------------------------------------------------------------------------


def planL(q):
    """chunk bit i -> slot; granule bit i -> slot (slots: r0 r1 r2 j0 j1 f0 f1 ...)."""
    chunk_slot_order = ["r0", "r1", "r2", "j1", "j0", "x0", "x1"]   # x* = extra (per-lane) fragment bits
    chunk = chunk_slot_order[:q]
    # granule bits 0..4: bit i (i<3) prefers slot r_i when free, else next free slot
    free = [s for s in ["r0", "r1", "r2", "j0", "j1"] if s not in chunk]
    gran = []
    for i in range(5):
        pref = f"r{i}" if i < 3 else None
        if pref and pref in free:
            gran.append(pref); free.remove(pref)
        elif i == 0 and "j0" in free:
            gran.append("j0"); free.remove("j0")
        elif i == 1 and "j1" in free:
            gran.append("j1"); free.remove("j1")
        elif free:
            gran.append(free.pop(0))
        else:
            gran.append(f"f{i}")  # loop (fragment) index
    return chunk, gran


def swzL(q, c):
    return c & ((1 << min(q, 3)) - 1)


def check_rowL(n, seed=0, verbose=False):
    k = n.bit_length() - 1
    q = k - 8
    C = 1 << q
    chunk_slots, gran_slots = planL(q)
    x = np.random.default_rng(seed).standard_normal(n)
    sm = np.zeros(n)

    def gaddr(c, gr):  # element offset of granule gr of chunk c (after swizzle)
        return c * 256 + 8 * (gr ^ swzL(q, c))

    A256 = kron_const("HHHH", 0.25)
    E = 4
    # phase 1: lane l holds granule l: X_j = elements 8l + 2j + h
    for c in range(C):
        vals = np.zeros((32, 4, 2))
        for l in range(32):
            vals[l] = x[c * 256 + 8 * l: c * 256 + 8 * l + 8].reshape(4, 2)
        v = stage_const_a(stage_const_a(vals, A256, (0, 2, 1, 3)), A256, (0, 2, 1, 3))
        for l in range(32):
            o = gaddr(c, l)
            sm[o:o + 8] = v[l].reshape(8)
    # phase 2
    nx = max(0, q - 5)                    # extra fragment bits handled in registers
    loop_bits = [s for s in gran_slots if s.startswith("f")]
    n_loop = 1 << len(loop_bits)
    conflicts = 0
    in_chunk = [s for s in chunk_slots if not s.startswith("x")]
    mask_a = 0
    for s in in_chunk:
        if s in ("r0", "r1", "r2", "j1"):
            mask_a |= 1 << ["r0", "r1", "r2", "j1"].index(s)
    two_stage = "j0" in in_chunk
    for it in range(n_loop):
        frags = []
        addrs_all = []
        for xi in range(1 << nx):
            slotv = {}
            for b, s in enumerate(loop_bits):
                slotv[s] = (it >> b) & 1
            for b in range(nx):
                slotv[f"x{b}"] = (xi >> b) & 1
            addrs = {}
            for L in range(32):
                j, r = L // 8, L % 8
                sv = dict(slotv, r0=r & 1, r1=(r >> 1) & 1, r2=(r >> 2) & 1, j0=j & 1, j1=(j >> 1) & 1)
                c = sum(sv[s] << i for i, s in enumerate(chunk_slots))
                gr = sum(sv[s] << i for i, s in enumerate(gran_slots))
                addrs[(j, r)] = gaddr(c, gr)
            for j in range(4):
                groups = {((addrs[(j, r)] * 2) // 16) % 8 for r in range(8)}
                conflicts += 8 - len(groups)
            # ldmatrix.trans: lane (g,t) reg j = {M_j[2t][g], M_j[2t+1][g]}, M_j[r][col] = sm[addr(j,r)+col]
            vals = np.zeros((32, 4, 2))
            for lane in range(32):
                g, t = lane >> 2, lane & 3
                for j in range(4):
                    for h in range(2):
                        vals[lane, j, h] = sm[addrs[(j, 2 * t + h)] + g]
            frags.append(vals)
            addrs_all.append(addrs)
        outs = []
        for vals in frags:
            if two_stage:
                v = stage_const_a(vals, kron_const(format(mask_a, "04b")[::-1].replace("1", "H").replace("0", "I"), 0.25 if bin(mask_a).count("1") >= 4 else 2.0 ** -(bin(mask_a).count("1") // 2)), (0, 2, 1, 3))
                v = stage_const_a(v, kron_const("IIIH", 1.0), (0, 2, 1, 3))
            else:
                kinds = "".join("H" if (mask_a >> b) & 1 else "I" for b in range(4))
                v = stage_data_a(vals, kron_const(kinds, 2.0 ** -(kinds.count("H") // 2)))
            outs.append(v)
        # in-register butterflies across the extra fragments (unnormalized)
        for b in range(nx):
            for xi in range(1 << nx):
                if not (xi >> b) & 1:
                    a_, b_ = outs[xi], outs[xi | (1 << b)]
                    outs[xi], outs[xi | (1 << b)] = a_ + b_, a_ - b_
        for vals, addrs in zip(outs, addrs_all):
            for lane in range(32):
                g, t = lane >> 2, lane & 3
                for j in range(4):
                    for h in range(2):
                        sm[addrs[(j, 2 * t + h)] + g] = vals[lane, j, h]
    hb = bin(mask_a).count("1")
    E += hb // 2 + (0 if not two_stage else 0)
    # phase 3
    y = np.zeros(n)
    for c in range(C):
        for l in range(32):
            o = gaddr(c, l)
            y[c * 256 + 8 * l: c * 256 + 8 * l + 8] = sm[o:o + 8]
    ref = fwht_np(x[None, :])[0]
    ratio = y / np.where(ref == 0, 1, ref)
    scale = np.median(ratio)
    ok = np.allclose(y, ref * scale)
    return ok, conflicts, chunk_slots, gran_slots, scale, mask_a, two_stage


def main_rowsL():
    for k in range(9, 16):
        ok, conf, cs, gs, sc, ma, ts = check_rowL(1 << k)
        print(f"n={1<<k:6d} ok={ok} ldsm_conflicts={conf} chunk={cs} gran={gs} mask_a={ma:#x} two_stage={ts} "
              f"scale=2^{np.log2(sc):.1f}")


# ---------------------------------------------------------------------------
# Design "T": smem row layout produced by a 4-D TMA tensor load with box
# (64 el, C chunks, 4 segments, rows) and SWIZZLE_128B.  Element (chunk c, granule
# g = 8*s + gg, e) of a row sits at byte
#     ((s*C + c) * 128) + 16 * (gg ^ ((s*C + c) & 7)) + 2*e
# (128B line index L = s*C + c; hardware XORs granule bits [4:6] with line bits).
# ---------------------------------------------------------------------------
def gaddrT(C, c, g):
    s, gg = g >> 3, g & 7
    L = s * C + c
    return (L * 128 + 16 * (gg ^ (L & 7))) // 2   # element offset


def check_rowT(n, seed=0):
    k = n.bit_length() - 1
    q = k - 8
    C = 1 << q
    chunk_slots, gran_slots = planL(q)
    x = np.random.default_rng(seed).standard_normal(n)
    # TMA load: natural row -> swizzled smem
    sm = np.zeros(n)
    for c in range(C):
        for g in range(32):
            o = gaddrT(C, c, g)
            sm[o:o + 8] = x[c * 256 + 8 * g: c * 256 + 8 * g + 8]
    A256 = kron_const("HHHH", 0.25)
    conf1 = 0
    for c in range(C):
        vals = np.zeros((32, 4, 2))
        for phase in range(4):  # LDS.128 processes 8 lanes (128 B) per wavefront
            groups = {(gaddrT(C, c, l) * 2 // 16) % 8 for l in range(8 * phase, 8 * phase + 8)}
            conf1 += 8 - len(groups)
        for l in range(32):
            o = gaddrT(C, c, l)
            vals[l] = sm[o:o + 8].reshape(4, 2)
        v = stage_const_a(stage_const_a(vals, A256, (0, 2, 1, 3)), A256, (0, 2, 1, 3))
        for l in range(32):
            o = gaddrT(C, c, l)
            sm[o:o + 8] = v[l].reshape(8)
    nx = max(0, q - 5)
    loop_bits = [s for s in gran_slots if s.startswith("f")]
    in_chunk = [s for s in chunk_slots if not s.startswith("x")]
    mask_a = 0
    for s in in_chunk:
        if s in ("r0", "r1", "r2", "j1"):
            mask_a |= 1 << ["r0", "r1", "r2", "j1"].index(s)
    two_stage = "j0" in in_chunk
    conf2 = 0
    for it in range(1 << len(loop_bits)):
        frags, addrs_all = [], []
        for xi in range(1 << nx):
            slotv = {s: (it >> b) & 1 for b, s in enumerate(loop_bits)}
            for b in range(nx):
                slotv[f"x{b}"] = (xi >> b) & 1
            addrs = {}
            for L_ in range(32):
                j, r = L_ // 8, L_ % 8
                sv = dict(slotv, r0=r & 1, r1=(r >> 1) & 1, r2=(r >> 2) & 1, j0=j & 1, j1=(j >> 1) & 1)
                c = sum(sv[s] << i for i, s in enumerate(chunk_slots))
                g = sum(sv[s] << i for i, s in enumerate(gran_slots))
                addrs[(j, r)] = gaddrT(C, c, g)
            for j in range(4):
                conf2 += 8 - len({(addrs[(j, r)] * 2 // 16) % 8 for r in range(8)})
            vals = np.zeros((32, 4, 2))
            for lane in range(32):
                gq, t = lane >> 2, lane & 3
                for j in range(4):
                    for h in range(2):
                        vals[lane, j, h] = sm[addrs[(j, 2 * t + h)] + gq]
            frags.append(vals)
            addrs_all.append(addrs)
        outs = []
        for vals in frags:
            if two_stage:
                v = stage_const_a(vals, kron_const("HHHH", 0.25), (0, 2, 1, 3))
                v = stage_const_a(v, kron_const("IIIH", 1.0), (0, 2, 1, 3))
            else:
                kinds = "".join("H" if (mask_a >> b) & 1 else "I" for b in range(4))
                v = stage_data_a(vals, kron_const(kinds, 2.0 ** -(kinds.count("H") // 2)))
            outs.append(v)
        for b in range(nx):
            for xi in range(1 << nx):
                if not (xi >> b) & 1:
                    a_, b_ = outs[xi], outs[xi | (1 << b)]
                    outs[xi], outs[xi | (1 << b)] = a_ + b_, a_ - b_
        for vals, addrs in zip(outs, addrs_all):
            for lane in range(32):
                gq, t = lane >> 2, lane & 3
                for j in range(4):
                    for h in range(2):
                        sm[addrs[(j, 2 * t + h)] + gq] = vals[lane, j, h]
    # TMA store: swizzled smem -> natural
    y = np.zeros(n)
    for c in range(C):
        for g in range(32):
            o = gaddrT(C, c, g)
            y[c * 256 + 8 * g: c * 256 + 8 * g + 8] = sm[o:o + 8]
    ref = fwht_np(x[None, :])[0]
    sc = np.median(y / np.where(ref == 0, 1, ref))
    return np.allclose(y, ref * sc), conf1, conf2, sc


def main_rowsT():
    for k in range(9, 16):
        ok, c1, c2, sc = check_rowT(1 << k)
        print(f"n={1<<k:6d} ok={ok} phase1_conflicts={c1} ldsm_conflicts={c2} scale=2^{np.log2(sc):.1f}")
