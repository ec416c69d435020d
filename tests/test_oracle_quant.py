"""Pins for oracle/quant.py, oracle/layout.py and oracle/gemm.py.

Each test checks the oracle against something it does not compute itself:
exact-rational brute force (Fractions), golden fixtures hand-derived from the
paper (tests/golden/), closed forms, invariants, library routines.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import gemm, layout, quant
from oracle import quant as oq
import synth
from oracle import numerics as nm

GOLD = os.path.join(os.path.dirname(__file__), "golden")
F = Fraction
GRID = [F(v) for v in nm.E4M3_POS_GRID]


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def fr(s):
    return F(s)


# ------------------------------------------------------------------ exact helpers
def sigma_exact(m: Fraction) -> Fraction:
    """Largest grid s with 7 s <= m (RZ of m/7), capped at 448."""
    best = F(0)
    for g in GRID:
        if 7 * g <= m:
            best = g
    return best


def rne_int(q: Fraction) -> int:
    fl = q.numerator // q.denominator
    rem = q - fl
    if rem > F(1, 2) or (rem == F(1, 2) and fl % 2 == 1):
        return fl + 1
    return fl


def codes_exact(ws, sigma):
    if sigma == 0:
        return [0] * len(ws)
    return [max(-8, min(7, rne_int(w / sigma))) for w in ws]


# ------------------------------------------------------------------------ layout
def test_layout_known_offsets():
    K = 512
    G = K // 128
    b = lambda n, k: tuple(int(x) for x in layout.packed_byte_index(n, k, K))
    assert b(0, 0) == (0, 0) and b(0, 1) == (0, 1) and b(0, 2) == (1, 0)
    assert b(0, 31) == (15, 1)
    assert b(0, 32) == (128 * 16, 0)          # next K-slice j=1
    assert b(1, 0) == (16, 0)                 # next row inside the tile
    assert b(0, 128) == (8192, 0)             # next group: next 8 KiB block
    assert b(128, 0) == (G * 8192, 0)         # next row tile
    assert int(layout.scale_index(5, 2, K)) == 2 * 128 + 5
    assert int(layout.scale_index(130, 1, K)) == (1 * G + 1) * 128 + 2


def test_layout_bijection_and_roundtrip():
    rng = np.random.default_rng(0)
    N, K = 256, 384
    n, k = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
    byte, half = layout.packed_byte_index(n, k, K)
    flat = byte * 2 + half
    assert np.array_equal(np.sort(flat.ravel()), np.arange(N * K))
    codes = rng.integers(-8, 8, size=(N, K)).astype(np.int8)
    assert np.array_equal(layout.unpack_codes(layout.pack_codes(codes), N, K), codes)
    sc = rng.integers(0, 127, size=(N, K // 128)).astype(np.uint8)
    assert np.array_equal(layout.unpack_scales(layout.pack_scales(sc), N, K), sc)
    # two consecutive groups of one row tile are one contiguous 16 KiB range
    blk = byte[:128, :256]
    assert blk.min() == 0 and blk.max() == 16383


def test_pack_nibble_encoding():
    codes = np.zeros((128, 128), dtype=np.int8)
    codes[0, 0], codes[0, 1] = -8, 7          # byte 0 = 0x78
    codes[0, 2], codes[0, 3] = -1, 1          # byte 1 = 0x1F
    p = layout.pack_codes(codes)
    assert p[0] == 0x78 and p[1] == 0x1F


# ----------------------------------------------------------------- group scale / codes
def test_group_scale_vs_exact():
    rng = np.random.default_rng(1)
    g = nm.E4M3_POS_GRID
    cands = np.concatenate([7 * g, np.nextafter(7 * g, 0), np.nextafter(7 * g, 1e9),
                            rng.uniform(0, 3200, 500), np.exp2(rng.uniform(-14, 12, 500)), [0.0, 1e9]])
    cands = nm.f32(cands)                         # W_tilde values are fp32
    got = quant.group_scale(cands)
    for m, s in zip(cands, got):
        assert F(float(s)) == sigma_exact(F(float(m))), m


def test_lemma1_suite():
    rng = np.random.default_rng(2)
    T = 7 * 2.0 ** -9
    small = rng.uniform(-1, 1, size=(1000, 128)) * T * rng.uniform(0, 0.999, size=(1000, 1))
    sig, codes = quant.quantize_groups(nm.f32(small))
    assert np.all(sig == 0) and np.all(codes == 0)                 # P:504 Lemma 1
    big = small.copy()
    big[:, 5] = T * rng.uniform(1.0, 100.0, size=1000) * rng.choice([-1, 1], size=1000)
    sig, _ = quant.quantize_groups(nm.f32(big))
    assert np.all(sig > 0)                                           # converse guard


def test_group_codes_vs_exact():
    rng = np.random.default_rng(3)
    for trial in range(300):
        w = nm.f32(rng.standard_normal(128) * 2.0 ** rng.integers(-12, 8))
        if trial % 3 == 0:    # plant exact ties v.5 * sigma
            s0 = float(quant.group_scale(np.abs(w).max()))
            if s0 > 0:
                w[:8] = nm.f32((rng.integers(-8, 8, 8) + 0.5) * s0)
        sig, codes = quant.quantize_groups(w[None, :])
        s = F(float(sig[0, 0]))
        assert s == sigma_exact(max(abs(F(float(x))) for x in w))
        assert list(codes[0]) == codes_exact([F(float(x)) for x in w], s)


def test_minus8_only_on_negative_side():
    rng = np.random.default_rng(4)
    w = nm.f32(rng.standard_normal((512, 1024)) * 0.02)
    _, codes = quant.quantize_groups(w)
    assert codes.min() >= -8 and codes.max() <= 7
    assert np.all(w[codes == -8] < 0)
    assert np.mean(codes == -8) > 0          # it is common (SURVEY finding 4)


def test_spec_group_examples():
    for ex in load("spec_examples.json")["group_quant"]:
        vals = np.array([float(fr(v)) for v in ex["values"]], dtype=np.float64)
        w = np.zeros((1, 128))
        w[0, :len(vals)] = vals
        sig, codes = quant.quantize_groups(w)
        assert F(float(sig[0, 0])) == fr(ex["sigma"]), ex["cite"]
        assert list(codes[0, :len(vals)]) == ex["codes"], ex["cite"]


# --------------------------------------------------------------------------- PTS
def S_exact(vals, n):
    T = F(7, 512)
    return sum(max(F(0), T - abs(v) * F(2) ** n) for v in vals)


def pts_literal_exact(vals, imax=4):
    """Def. 2 with exact rationals: condition 1 checked for i = 1..imax."""
    for n in range(61):
        c1 = all(S_exact(vals, n) == S_exact(vals, n + i) for i in range(1, imax + 1))
        lo, hi = 7 * F(2) ** (5 - n), 7 * F(2) ** (6 - n)
        c2 = any(lo <= abs(v) < hi for v in vals)
        if c1 or c2:
            return n
    return None


def test_pts_vs_exact_literal():
    rng = np.random.default_rng(5)
    for trial in range(150):
        size = rng.integers(1, 12)
        v = rng.standard_normal(size) * 2.0 ** rng.integers(-25, 10, size)
        if trial % 5 == 0:
            v[0] = 0.0
        if trial % 7 == 0:
            v[-1] = 224.0 * 2.0 ** -rng.integers(0, 12)
        v = nm.f32(v)
        exp = pts_literal_exact([F(float(x)) for x in v])
        n, _ = quant.pts_exponent(v)
        assert n == exp, (v, n, exp)


def test_pts_spec_examples():
    assert quant.pts_exponent(np.full(10, 2.0 ** -12))[0] == 6
    assert quant.pts_exponent(np.array([224.0, 0.001]))[0] == 0
    assert quant.pts_exponent(np.zeros(7)) == (0, "underflow-stable")
    assert quant.pts_exponent(np.array([1000.0, 0.01]))[0] == 1
    with pytest.raises(ValueError):
        quant.pts_exponent(np.array([2.0 ** -120]))


def test_pts_no_band_element_below_n():
    # Post-PTS guarantee: for n' < n no element is in the overflow band.
    rng = np.random.default_rng(6)
    W = nm.f32(rng.standard_normal((64, 64)) * 0.02)
    n, reason = quant.pts_exponent(W)
    a = np.abs(W)
    for m in range(n):
        assert not np.any((a * 2.0 ** m >= 224) & (a * 2.0 ** m < 448))
    in_band = np.any((a * 2.0 ** n >= 224) & (a * 2.0 ** n < 448))
    stable = np.all(a[a > 0] * 2.0 ** n >= 7 * 2.0 ** -9)
    assert (reason == "overflow-risk" and in_band) or (reason == "underflow-stable" and stable)


# --------------------------------------------------------------------------- CAS
def test_cas_equalization_and_off():
    rng = np.random.default_rng(7)
    W = nm.bf16_rn(rng.standard_normal((256, 384)) * np.exp(rng.normal(0, 0.5, 384))[None, :] * 0.02)
    lam, c = quant.cas_lambda(W, 1)
    Wb = quant.cas_apply(W, lam)
    absm = np.abs(Wb).mean(axis=0)
    target = np.abs(W).mean(axis=0).mean()
    assert np.max(np.abs(absm - target) / target) < 1e-5            # S:275 invariant
    lam0, c0 = quant.cas_lambda(W, 0)
    assert np.all(lam0 == 1) and np.all(c0 == 1)
    # merge equivalence (X Lambda^-1)(Lambda^T W^T) = X W^T (Eq. at), fp64
    X = rng.standard_normal((8, 384))
    lhs = (X / lam[None, :]) @ (W * lam[None, :]).T
    assert np.max(np.abs(lhs - X @ W.T)) <= 1e-9 * np.max(np.abs(X @ W.T))
    # c = bf16(1/lambda): relative error <= 2^-8
    assert np.all(np.abs(c * lam - 1) <= 2.0 ** -8)


def test_cas_spec_example_two_channels():
    ex = load("spec_examples.json")["cas"][0]
    W = np.array([[1.0, 4.0], [-1.0, -4.0]] * 64)     # absmeans {1, 4}
    W = np.concatenate([W] * 64, axis=1)[:, :128]
    lam, _ = quant.cas_lambda(W, 1)
    assert F(float(lam[0])) == fr(ex["lambda"][0]) and F(float(lam[1])) == fr(ex["lambda"][1])


def test_cas_zero_channel():
    W = np.ones((128, 128))
    W[:, 3] = 0
    lam, c = quant.cas_lambda(W, 1)
    assert lam[3] == 1.0


# --------------------------------------------------------- quantize_weight golden
def test_f_edge_golden():
    g = load("f_edge.json")
    K = 128 * g["K_groups"]
    W = np.zeros((128, K))
    for i, row in enumerate(g["rows"]):
        W[i, :len(row["values"])] = [float(fr(v)) for v in row["values"]]
    assert np.array_equal(nm.bf16_rn(W), W)                          # BF16-exact inputs
    q = quant.quantize_weight(W, g["cas_mode"])
    assert q.n == g["pts_n"]
    wdeq = gemm.dequantize_weight(q.packed, q.scales, 128, K)
    for i, row in enumerate(g["rows"]):
        L = len(row["values"])
        assert F(float(q.sigma[i, 0])) == fr(row["sigma"]), row["exercises"]
        assert list(q.codes[i, :L]) == row["codes"], row["exercises"]
        assert [F(float(x)) for x in wdeq[i, :L]] == [fr(x) for x in row["deq"]], row["exercises"]
    assert np.all(q.codes[:, 128:] == 0) and np.all(q.sigma[:, 1] == 0)


def test_boundary_ones_golden():
    ex = load("spec_examples.json")["boundary_ones"]
    W = np.ones((128, 128))
    for mode in (0, 1):
        q = quant.quantize_weight(W, mode)
        assert q.n == ex["n"] and np.all(q.sigma == float(fr(ex["sigma"])))
        assert np.all(q.codes == ex["code"])
        assert np.all(gemm.dequantize_weight(q.packed, q.scales, 128, 128) == 1.0)


def test_quantize_weight_roundtrip_error():
    # Eq. 1 round-trip: |w - deq| <= sigma/2 inside the clamp range, per group, plus LUT rounding
    rng = np.random.default_rng(8)
    W = nm.bf16_rn(rng.standard_normal((128, 256)) * 0.02)
    q = quant.quantize_weight(W, 1)
    Wt = q.W_bar * 2.0 ** q.n
    deq = gemm.dequantize_weight(q.packed, q.scales, 128, 256)
    sig = np.repeat(q.sigma, 128, axis=1)
    inside = np.abs(Wt) <= 7.5 * sig
    lut_err = np.abs(deq - q.codes * sig)              # FP8 re-rounding of v*sigma: <= 2^-4 relative
    assert np.all(lut_err <= 2.0 ** -4 * np.abs(q.codes * sig) + 2.0 ** -10)
    assert np.all(np.abs(Wt - q.codes * sig)[inside] <= sig[inside] / 2 + 1e-30)


# ---------------------------------------------------------------------- activations
def test_act_spec_examples():
    for ex in load("spec_examples.json")["act"]:
        X = np.zeros((1, 128))
        X[0, :2] = [float(fr(v)) for v in ex["row"]]
        codes, beta = quant.quantize_act(X)
        assert F(float(beta[0])) == fr(ex["beta"])
        assert [F(float(v)) for v in nm.e4m3_decode(codes[0, :2])] == [fr(v) for v in ex["x_hat"]]


def test_act_vs_exact():
    rng = np.random.default_rng(9)
    X = nm.bf16_rn(rng.standard_normal((6, 128)) * 2.0 ** rng.integers(-10, 10, (6, 1)))
    c = nm.bf16_rn(np.exp(rng.normal(0, 0.5, 128)))
    codes, beta = quant.quantize_act(X, c)
    from test_oracle_numerics import rn_exact
    for m in range(6):
        xp = [F(float(nm.bf16_rn(np.float64(X[m, k]) * c[k]))) for k in range(128)]
        amax = max(abs(v) for v in xp)
        b = amax / 448
        # exact-rational RNE of b onto bf16 (8-bit significand)
        e = 0
        while b >= 2:
            b /= 2; e += 1
        while b < 1:
            b *= 2; e -= 1
        bb = F(rne_int(b * 128), 128) * F(2) ** e
        assert F(float(beta[m])) == bb
        for k in range(0, 128, 7):
            assert F(float(nm.e4m3_decode(codes[m, k]))) == rn_exact(xp[k] / bb)
    assert np.all(np.abs(nm.e4m3_decode(codes)) <= 448)


# ---------------------------------------------------------------------------- LUT
def test_lut_exhaustive_vs_exact():
    table = gemm.lut_of_luts()
    from test_oracle_numerics import rn_exact
    for s in range(127):
        sig = GRID[s]
        for u in range(16):
            v = u if u < 8 else u - 16
            val = F(float(nm.E4M3_DECODE[table[s, u]]))
            assert val == rn_exact(v * sig)
            if v * sig == 0 and v < 0:
                assert table[s, u] == 0x80                 # IEEE -0 for (-v) * 0
    # SPEC / survey LUT examples
    for ex in load("spec_examples.json")["lut"]:
        lut = gemm.lut_for_sigma(float(fr(ex["sigma"])))
        vals = [F(float(nm.E4M3_DECODE[lut[v & 15]])) for v in range(-8, 8)]
        assert vals == [fr(x) for x in ex["entries_v_-8_to_7"]], ex["cite"]


def test_lut_not_exact_share():
    # SURVEY finding 3 counts the (sigma, v) pairs whose v*sigma is off the E4M3
    # grid; an independent set-membership brute force gives 810 inexact / 1,222
    # exact of 2,032 (the survey text has the two numbers swapped).
    table = nm.E4M3_DECODE[gemm.lut_of_luts()]
    exact = table == nm.E4M3_POS_GRID[:, None] * gemm.NIBBLE_VALUES[None, :]
    grid = set(F(float(v)) for v in nm.E4M3_POS_GRID)
    brute = sum(1 for s in grid for v in range(-8, 8) if abs(v * s) not in grid)
    assert (~exact).sum() == brute == 810


# --------------------------------------------------------------------------- GEMM
def test_gemm_reference_vs_fraction_bruteforce():
    rng = np.random.default_rng(10)
    N, K, M = 128, 256, 2
    W = nm.bf16_rn(rng.standard_normal((N, K)) * 0.02)
    q = quant.quantize_weight(W, 1)
    X = nm.bf16_rn(rng.standard_normal((M, K)))
    xc, beta = quant.quantize_act(X, q.c)
    r = gemm.gemm_reference(xc, beta, q.packed, q.scales, N, K, q.n)
    codes = layout.unpack_codes(q.packed, N, K)
    scodes = layout.unpack_scales(q.scales, N, K)
    from test_oracle_numerics import rn_exact
    for (m, n) in [(0, 0), (1, 77), (0, 127)]:
        acc = F(0)
        for k in range(K):
            sig = GRID[scodes[n, k // 128]]
            wv = rn_exact(int(codes[n, k]) * sig)
            acc += F(float(nm.E4M3_DECODE[xc[m, k]])) * wv
        exact = acc * F(float(beta[m])) / F(2) ** q.n
        assert abs(F(float(r[m, n])) - exact) <= abs(exact) * F(1, 2 ** 50)


def test_gemm_reference_residual():
    """Step 3's fused addition: the exact-rational brute force of one output plus the
    residual value; and an all-zero weight gives exactly the residual (zero groups: sigma = 0,
    every LUT entry 0)."""
    rng = np.random.default_rng(12)
    N, K, M = 128, 256, 2
    W = nm.bf16_rn(rng.standard_normal((N, K)) * 0.02)
    q = quant.quantize_weight(W, 1)
    X = nm.bf16_rn(rng.standard_normal((M, K)))
    R = nm.bf16_rn(rng.standard_normal((M, N)))
    xc, beta = quant.quantize_act(X, q.c)
    r = gemm.gemm_reference(xc, beta, q.packed, q.scales, N, K, q.n, residual=R)
    codes = layout.unpack_codes(q.packed, N, K)
    scodes = layout.unpack_scales(q.scales, N, K)
    from test_oracle_numerics import rn_exact
    for (m, n) in [(0, 3), (1, 100)]:
        acc = F(0)
        for k in range(K):
            acc += F(float(nm.E4M3_DECODE[xc[m, k]])) * rn_exact(int(codes[n, k]) * GRID[scodes[n, k // 128]])
        exact = acc * F(float(beta[m])) / F(2) ** q.n + F(float(R[m, n]))
        assert abs(F(float(r[m, n])) - exact) <= abs(exact) * F(1, 2 ** 50)
    q0 = quant.quantize_weight(np.zeros((N, K)), 0)
    r0 = gemm.gemm_reference(xc, beta, q0.packed, q0.scales, N, K, q0.n, residual=R)
    assert np.array_equal(r0, R)


def test_gemm_exactness_corridor_and_zero_groups():
    # integer operands, sigma = 1, beta = 1, n = 0: reference is an exact integer dot product
    rng = np.random.default_rng(11)
    N, K, M = 128, 256, 3
    codes = rng.integers(-8, 8, size=(N, K)).astype(np.int8)
    sc = np.full((N, K // 128), 56, dtype=np.uint8)        # code 56 = 1.0
    assert nm.E4M3_DECODE[56] == 1.0
    sc[5, 1] = 0                                            # a zero-sigma group contributes 0
    packed, scales = layout.pack_codes(codes), layout.pack_scales(sc)
    xi = rng.integers(-4, 5, size=(M, K)).astype(np.float64)
    xc = nm.e4m3_encode(xi)
    r = gemm.gemm_reference(xc, np.ones(M), packed, scales, N, K, 0)
    wv = codes.astype(np.float64)
    wv[5, 128:] = 0
    assert np.array_equal(r, xi @ wv.T)
    # PTS transparency: 2^-n folding is exact
    r3 = gemm.gemm_reference(xc, np.ones(M), packed, scales, N, K, 3)
    assert np.array_equal(r3 * 8, r)


def test_g4_separates_bugs():
    """G4 criterion calibration: correct ~0.004, injected bugs >= 0.4."""
    rng = np.random.default_rng(12)
    N, K, M = 256, 1024, 16
    W = nm.bf16_rn(rng.standard_normal((N, K)) * 0.02)
    q = quant.quantize_weight(W, 1)
    X = nm.bf16_rn(rng.standard_normal((M, K)) * np.where(np.arange(K) % 97 == 0, 20, 1))
    xc, beta = quant.quantize_act(X, q.c)
    r = gemm.gemm_reference(xc, beta, q.packed, q.scales, N, K, q.n)
    y_ok = nm.bf16_rn(nm.f32(r))                                  # correct kernel: BF16 output rounding
    assert gemm.g4_error(y_ok, r) < 5e-3
    x = nm.E4M3_DECODE[xc]
    sig = np.repeat(q.sigma, 128, axis=1)
    s = beta[:, None] * 2.0 ** -q.n
    bugs = {
        "no LUT re-rounding": q.codes * sig,
        "-8 decoded as -7": np.where(q.codes == -8, -7, q.codes) * sig,
        "nibble order swapped": q.codes.reshape(N, K // 2, 2)[:, :, ::-1].reshape(N, K) * sig,
        "group index off by one": q.codes * np.roll(sig, 128, axis=1),
    }
    wdeq = gemm.dequantize_weight(q.packed, q.scales, N, K)
    assert np.array_equal(gemm.gemm_reference(xc, beta, q.packed, q.scales, N, K, q.n, w_deq=wdeq), r)
    for name, wb in bugs.items():
        yb = nm.bf16_rn((x @ wb.T) * s)
        assert gemm.g4_error(yb, r) > 0.05, name


def test_dequant_cost():
    ex = load("spec_examples.json")["dequant_cost"]
    assert gemm.dequant_cost_ops(ex["b"], ex["d_in"], ex["d_out"]) == ex["ops"]


def test_underflow_group_fraction():
    W = np.full((4, 512), 1.0)
    W[:, :128] = 1e-4                       # 1 of 4 groups per row is tiny
    assert quant.underflow_group_fraction(W) == 0.25
    n, _ = quant.pts_exponent(W)
    assert quant.underflow_group_fraction(W * 2.0 ** n) <= 0.25


def test_quantize_weight_rows_subset_equals_full():
    """rows= (used by the full-size GPU checks) computes W4-W5 of the selected rows only; CAS
    and PTS stay global, so the subset must equal the same rows of the full computation."""
    wb = synth.weights(512, 1024, 5)
    W = synth.bits_to_f64(wb)
    W[7, :] *= 0.0                       # rows that change nothing globally still select correctly
    full = oq.quantize_weight(W, 1, pack=False)
    rows = np.array([0, 7, 100, 511])
    sub = oq.quantize_weight(W, 1, pack=False, rows=rows)
    assert full.n == sub.n
    assert np.array_equal(full.lam, sub.lam)
    assert np.array_equal(full.codes[rows], sub.codes)
    assert np.array_equal(full.sigma_codes[rows], sub.sigma_codes)
    with pytest.raises(ValueError):
        oq.quantize_weight(W, 1, rows=rows)


# ---------------------------------------------------------- sigma_BF16 variant (R25)
def _bf16_rne_exact(q):
    """Exact-rational round-to-nearest-even of a positive Fraction onto the bf16 grid (normal range)."""
    if q == 0:
        return Fraction(0)
    e = 0
    while q >= 2:
        q /= 2
        e += 1
    while q < 1:
        q *= 2
        e -= 1
    # q in [1, 2): 7 fraction bits
    scaled = q * 128
    lo = scaled.numerator // scaled.denominator
    rem = scaled - lo
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and lo % 2 == 1):
        lo += 1
    return Fraction(lo, 128) * (Fraction(2) ** e)


def test_bf16s_sigma_is_exact_rational_rne():
    """sigma_BF16 = bf16_RN(m / 7): the float64 division then bf16 rounding equals the exact
    rational RNE (no double rounding), on random fp32 group maxima and on m = 7 x bf16 midpoints."""
    rng = np.random.default_rng(2501)
    ms = list(nm.f32(np.exp(rng.uniform(-20, 6, 3000))))
    for v in [1.00390625, 1.01171875, 0.0546875 * 1.00390625]:        # exact ties at m / 7
        ms.append(float(nm.f32(np.array([7.0 * v]))[0]))
    got = nm.bf16_rn(np.array(ms) / 7.0)
    for m, g in zip(ms, got):
        assert Fraction(g) == _bf16_rne_exact(Fraction(m) / 7), m


def test_bf16s_codes_and_closed_form():
    """Codes are the exact-rational RNE of w / sigma clamped to [-8, 7]; a group whose maximum
    is 7 x (a bf16 value) gets exactly that sigma and code 7 there; a zero group gets sigma 0."""
    rng = np.random.default_rng(2502)
    W = nm.bf16_rn(rng.standard_normal((128, 384)) * 0.05)
    W[3, 0] = 7 * 0.25                                  # group (3, 0): sigma = 0.25 exactly
    W[3, 1:128] = np.clip(W[3, 1:128], -1.75, 1.75)
    W[5, 128:256] = 0.0
    q = quant.quantize_weight_bf16s(W, 0)
    Wt = W * 2.0 ** q.n
    assert q.sigma[3, 0] == 0.25 * 2.0 ** q.n and q.codes[3, 0] == 7
    assert q.sigma[5, 1] == 0 and not q.codes[5, 128:256].any()
    for (r, g) in [(0, 0), (3, 0), (77, 2), (127, 1)]:
        sig = Fraction(q.sigma[r, g])
        for k in range(g * 128, g * 128 + 128, 7):
            x = Fraction(Wt[r, k]) / sig
            fl = x.numerator // x.denominator
            rem = x - fl
            rne = fl + (1 if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1) else 0)
            assert q.codes[r, k] == max(-8, min(7, rne))
    # packing: same codes layout as layout v1; scales blocked like the FP8 scale codes
    assert np.array_equal(layout.unpack_codes(q.packed, 128, 384), q.codes)
    assert np.array_equal(q.scales16[layout.scale_index(np.full(3, 3), np.arange(3), 384)], q.sigma_bits[3])


def test_bf16s_reference_vs_fraction():
    """gemm_reference_bf16s against an exact-rational sum on a tiny problem."""
    rng = np.random.default_rng(2503)
    W = nm.bf16_rn(rng.standard_normal((128, 256)) * 0.03)
    X = nm.bf16_rn(rng.standard_normal((2, 256)))
    q = quant.quantize_weight_bf16s(W, 1)
    xq, beta = quant.quantize_act(X, q.c)
    r = gemm.gemm_reference_bf16s(xq, beta, q.codes, q.sigma, q.n)
    xv = nm.E4M3_DECODE[xq]
    for m in range(2):
        for n in (0, 5, 127):
            s = sum(Fraction(xv[m, k]) * int(q.codes[n, k]) * Fraction(q.sigma[n, k // 128]) for k in range(256))
            exact = s * Fraction(beta[m]) / (Fraction(2) ** q.n)
            assert abs(float(exact) - r[m, n]) <= 1e-12 * max(1.0, abs(float(exact)))
