"""Pins for oracle/ffn.py (silu_mul, ffn_reference) against things other than itself.

* SiLU (Step 3 "SiLU and element-wise multiplication") against a 60-digit
  ``decimal`` evaluation of g / (1 + e^-g), rounded to bf16 by an exact-rational
  rounding written here (not the oracle's bf16_rn);
* a hand-derived FFN: identity-structured gate / up / down weights whose INT4
  quantization, LUT dequantization and GEMMs are exact, so every
  intermediate (g, u, the CAS inverse gamma merged into the up half, h, beta_h, h_hat,
  y) is a closed form computed below with Fractions;
* the chained-layer tolerance (R17, 2e-2) calibrated by injected bugs
  (gate / up swapped, gamma on the wrong half, a missing bf16 rounding) against an
  FP32-accumulation positive control, as test_g4_separates_bugs does for G4.
"""
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import ffn as of
from oracle import gemm as og
from oracle import numerics as nm
from oracle import quant as oq

getcontext().prec = 60


# ---------------------------------------------------------------- exact helpers
def round_bits(x: Fraction, p: int, emin: int) -> Fraction:
    """Round x to p significant bits, ties to even; exponent floor emin (subnormals)."""
    if x == 0:
        return Fraction(0)
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    q = Fraction(2) ** (max(e, emin) - (p - 1))
    t = a / q
    n = t.numerator // t.denominator
    rem = t - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    r = n * q
    return -r if x < 0 else r


def bf16(x: Fraction) -> Fraction:
    return round_bits(x, 8, -126)


def f32(x: Fraction) -> Fraction:
    return round_bits(x, 24, -126)


# E4M3 "fn" grid from its definition (bias 7, 3 mantissa bits, S.1111.111 = NaN)
E4M3 = sorted({Fraction(m, 8) * Fraction(2) ** -6 for m in range(8)} |
              {(1 + Fraction(m, 8)) * Fraction(2) ** (e - 7) for e in range(1, 16) for m in range(8)
               if not (e == 15 and m == 7)})
assert E4M3[-1] == 448 and len(E4M3) == 127


def e4m3_rn(x: Fraction) -> Fraction:
    a = min(abs(x), Fraction(448))
    best = min(range(127), key=lambda i: (abs(E4M3[i] - a), i % 2))
    return -E4M3[best] if x < 0 else E4M3[best]


def silu_exact(g: Fraction) -> Fraction:
    ex = (Decimal(-g.numerator) / Decimal(g.denominator)).exp()
    return g / (1 + Fraction(ex))


# ------------------------------------------------------------------ SiLU pin
def test_silu_mul_matches_decimal_exact():
    rng = np.random.default_rng(7)
    gb = synth.to_bf16_bits(rng.normal(0, 3, 1500).astype(np.float32))
    ub = synth.to_bf16_bits(rng.normal(0, 2, 1500).astype(np.float32))
    g = synth.bits_to_f64(gb)
    u = synth.bits_to_f64(ub)
    # special values: 0, the saturating tails, tiny and huge magnitudes
    g = np.concatenate([g, [0.0, -0.0, 1.0, -1.0, 40.0, -40.0, 100.0, -100.0, 2.0 ** -20, 448.0]])
    u = np.concatenate([u, [3.0, 3.0, 1.0, 1.0, 1.0, 1.0, 0.5, 0.5, 1.0, 600.0]])
    h = of.silu_mul(g, u)
    mism = 0
    for gi, ui, hi in zip(g, u, h):
        gf, uf = Fraction(float(gi)), Fraction(float(ui))
        exact = silu_exact(gf) * uf
        ref = bf16(exact)
        if Fraction(float(hi)) != ref:
            # only a near-tie (exact value within 2^-40 relative of a bf16 midpoint) may
            # differ: the fp64 evaluation of exp carries ~1e-16 relative error
            lo, hi2 = sorted([Fraction(float(hi)), ref])
            mid = (lo + hi2) / 2
            assert abs(exact - mid) <= abs(mid) * Fraction(1, 2 ** 40), (gi, ui, hi, float(ref))
            mism += 1
    assert mism <= 2
    # closed forms: silu(0) = 0; silu(g) -> g for large g; -> 0 (from below) for very negative g
    assert of.silu_mul(np.array([0.0]), np.array([5.0]))[0] == 0.0
    assert of.silu_mul(np.array([100.0]), np.array([1.0]))[0] == 100.0
    v = of.silu_mul(np.array([-100.0]), np.array([1.0]))[0]
    assert v == 0.0 and np.signbit(v)      # -3.7e-42 is below bf16's 2^-133: rounds to -0
    v = of.silu_mul(np.array([-40.0]), np.array([1.0]))[0]
    assert v < 0 and abs(v) < 1e-15


# ------------------------------------------------------------------ hand FFN
D = 128
X_ROWS = [
    # token 0: amax 448 -> beta = 1 (x_hat = x); token 1: amax 224 -> beta = 1/2
    [448, 1, -1, 2, 0.5, -3, 0.375, 7, -0.0625, 96, -20, 0.8125],
    [224, -0.25, 3.5, -112, 0, 5, 1.5, -0.5, 40, 0.125, -6, 64],
]


def _hand_weights():
    Wg = np.eye(D)                              # gate: identity
    Wu = 2.0 * np.eye(D)                        # up: 2 * identity
    d_k = np.where(np.arange(D) % 2 == 0, 1.0, 2.0)
    Wd = np.diag(d_k)                           # down: diag(1, 2, 1, 2, ...)
    return Wg, Wu, Wd, d_k


def _hand_expected():
    """y by closed forms (every GEMM here is one exact product per output)."""
    # [gate; up] with CAS: every input column holds one 1 and one 2 -> absmean 3/256
    # everywhere, lambda = 1, c_gu = 1; PTS n = 0 (min nonzero 1 >= 7*2^-9).
    # gate rows: sigma = RZ(1/7) = 9/64, code rint(64/9) = 7, LUT RN(63/64) = 1.
    # up rows:   sigma = RZ(2/7) = 9/32, code 7, LUT RN(63/32) = 2.
    # down (CAS): absmean_k = d_k/128, omega_bar = 1.5/128, lambda_k = 1.5/d_k,
    #   W_bar = diag(1.5); sigma = RZ(1.5/7) = 13/64, code rint(96/13) = 7,
    #   LUT RN(91/64) = RN(1.421875) = 1.375 (1.4375 is the midpoint); PTS n = 0.
    #   gamma_k = c_down_k = bf16(fp32(1 / lambda_k)) multiplies the up half (R20).
    _, _, _, d_k = _hand_weights()
    ys = []
    for row in X_ROWS:
        x = [Fraction(v) for v in row] + [Fraction(0)] * (D - len(row))
        amax = max(abs(v) for v in x)
        beta = bf16(amax / 448)
        xh = [e4m3_rn(v / beta) for v in x]
        h = []
        for k in range(D):
            lam = f32(Fraction(3, 2) / Fraction(d_k[k]).limit_denominator())
            gam = bf16(f32(1 / lam))
            g = bf16(xh[k] * 1 * beta)
            u = bf16(xh[k] * 2 * beta * gam)
            h.append(bf16(silu_exact(g) * u) if g != 0 else Fraction(0))
        hmax = max(abs(v) for v in h)
        bh = bf16(hmax / 448) if hmax > 0 else Fraction(1)
        hh = [e4m3_rn(v / bh) for v in h]
        ys.append([bf16(v * Fraction(11, 8) * bh) for v in hh])
    return ys


def test_hand_ffn_weights_quantize_as_derived():
    Wg, Wu, Wd, _ = _hand_weights()
    q_gu = oq.quantize_weight(np.concatenate([Wg, Wu]), 1)
    q_d = oq.quantize_weight(Wd, 1)
    assert q_gu.n == 0 and q_d.n == 0
    assert np.all(q_gu.lam == 1.0) and np.all(q_gu.c == 1.0)
    deq = og.dequantize_weight(q_gu.packed, q_gu.scales, 2 * D, D)
    assert np.array_equal(deq, np.concatenate([np.eye(D), 2.0 * np.eye(D)]))
    assert np.array_equal(og.dequantize_weight(q_d.packed, q_d.scales, D, D), 1.375 * np.eye(D))
    assert set(np.unique(q_d.sigma)) == {13 / 64}     # K = 128: one group per row


def test_hand_ffn_closed_form():
    Wg, Wu, Wd, _ = _hand_weights()
    q_gu = oq.quantize_weight(np.concatenate([Wg, Wu]), 1)
    q_d = oq.quantize_weight(Wd, 1)
    X = np.array([r + [0.0] * (D - len(r)) for r in X_ROWS], dtype=np.float64)
    y, _ = of.ffn_reference(X, q_gu, q_d, D)
    want = np.array([[float(v) for v in row] for row in _hand_expected()])
    assert np.array_equal(y, want)
    # the derivation is not degenerate: gamma alternates and h uses several FP8 codes
    for row in want:
        assert len(np.unique(np.abs(row[row != 0]))) >= 5


# ------------------------------------------------- chained tolerance calibration
def _ffn_variant(X, q_gu, q_d, dff, bug=None):
    """The FFN chain of oracle/ffn.py with one injected bug (or FP32 accumulation)."""
    N_gu, d = 2 * dff, X.shape[1]
    xq, beta = oq.quantize_act(X, q_gu.c)
    gamma = np.concatenate([np.ones(dff), q_d.c])
    if bug == "gamma_on_gate":
        gamma = np.concatenate([q_d.c, np.ones(dff)])
    wdeq = og.dequantize_weight(q_gu.packed, q_gu.scales, N_gu, d)
    if bug == "fp32_accum":
        acc = (nm.e4m3_decode(xq).astype(np.float32) @ wdeq.T.astype(np.float32)).astype(np.float64)
        r = nm.f32(nm.f32(acc * (beta[:, None] * 2.0 ** -q_gu.n)) * gamma[None, :])
    else:
        r = og.gemm_reference(xq, beta, q_gu.packed, q_gu.scales, N_gu, d, q_gu.n, gamma=gamma, w_deq=wdeq)
    gu = r if bug == "no_bf16_gu" else nm.bf16_rn(r)
    g, u = gu[:, :dff], gu[:, dff:]
    if bug == "swap":
        g, u = u, g
    h = of.silu_mul(g, u)
    hq, hb = oq.quantize_act(h)
    ddeq = og.dequantize_weight(q_d.packed, q_d.scales, d, dff)
    if bug == "fp32_accum":
        acc = (nm.e4m3_decode(hq).astype(np.float32) @ ddeq.T.astype(np.float32)).astype(np.float64)
        return nm.bf16_rn(nm.f32(acc * (hb[:, None] * 2.0 ** -q_d.n)))
    return nm.bf16_rn(og.gemm_reference(hq, hb, q_d.packed, q_d.scales, d, dff, q_d.n, w_deq=ddeq))


@pytest.fixture(scope="module")
def small_ffn():
    M, d, dff = 16, 256, 384
    wg = synth.weights(dff, d, 501)
    wu = synth.weights(dff, d, 502)
    wd = synth.weights(d, dff, 503)
    X = synth.bits_to_f64(synth.activations(M, d, 504))
    q_gu = oq.quantize_weight(synth.bits_to_f64(np.concatenate([wg, wu])), 1)
    q_d = oq.quantize_weight(synth.bits_to_f64(wd), 1)
    _, r = of.ffn_reference(X, q_gu, q_d, dff)
    return X, q_gu, q_d, dff, r


def test_chained_tolerance_accepts_fp32_accumulation(small_ffn):
    X, q_gu, q_d, dff, r = small_ffn
    y = _ffn_variant(X, q_gu, q_d, dff, "fp32_accum")
    assert og.g4_error(y, r) <= 2e-2
    assert og.g4_error(_ffn_variant(X, q_gu, q_d, dff), r) <= 1e-2    # the correct chain, bf16 output


@pytest.mark.parametrize("bug,floor", [("swap", 1.0), ("gamma_on_gate", 1.0), ("no_bf16_gu", 0.1)])
def test_chained_tolerance_rejects_bugs(small_ffn, bug, floor):
    """Each injected bug scores at least 5x the 2e-2 bound (measured: swap 31.7, gamma on
    the gate half 11.7, unrounded g / u 0.79 -- the missing rounding moves FP8 codes of h
    and, through max|h|, beta_h of most tokens)."""
    X, q_gu, q_d, dff, r = small_ffn
    assert og.g4_error(_ffn_variant(X, q_gu, q_d, dff, bug), r) > floor
