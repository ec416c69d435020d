"""FireQ offline weight quantizer and online activation quantizer.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Weight path (offline, "merged with calibration matrices and quantized
offline"), steps W1-W6 of DESIGN.md section "Oracle", in the paper's order:

  W1  CAS      Def. 1: W_bar = W Lambda, lambda^i = omega_bar /
               absmean(omega^i), channel i = input channel (reading A9).
  W2  apply    W_bar[n, k] = fp32(W[n, k]) * lambda_k        (one fp32 rounding)
  W3  PTS      Def. 2: n = smallest n >= 0 meeting
               eq:pts_first_condition or eq:pts_second_condition;
               W_tilde = W_bar * 2^n (exact).
  W4  scale    Eq. 1 with b = 4: sigma = max|w| / 7 encoded in FP8
               toward zero (forced by Lemma 1; reading A2).
  W5  codes    round-half-even(w / sigma) clamped to [-8, 7] (reading A5);
               sigma = 0 -> codes 0 (Lemma 1).
  W6  pack     layout v1 (oracle/layout.py).

Activation path (online), steps A1-A3:
  A1  x' = bf16(x * c_k) when the CAS inverse c = Lambda^-1 is applied to the
      activations, else x' = x.
  A2  beta = bf16_RN(max|x'| / 448) per token (Eq. 2, per-token P:482;
      reading A7), beta = 1 for an all-zero row.
  A3  x_hat = E4M3_RN_sat(x' / beta) (Eq. 2).
"""
import numpy as np

from .numerics import (E4M3_POS_GRID, E4M3_MAX, UNDERFLOW_T, bf16_rn, e4m3_encode,
                       e4m3_rn, f32)
from . import layout

GROUP = 128
PTS_MAX_N = 60


# --------------------------------------------------------------------- W1 / W2
def given_lambda(lam):
    """W1 with a caller-given per-input-channel multiplier (the KV-cache path: CRS divides the
    post-RoPE outlier key channels by t, lambda = fp32(1 / t)): c = bf16(1/lambda)."""
    lam = np.asarray(lam, dtype=np.float32).astype(np.float64)
    c = bf16_rn((np.float32(1.0) / lam.astype(np.float32)).astype(np.float64))
    return lam, c


def cas_lambda(W, cas_mode):
    """W1: per-input-channel lambda (fp32 values as float64) and c = bf16(1/lambda).

    absmean_k = fp32( (sum_{n=0}^{N-1} |W[n,k]|, fp64, ascending n) / N )
    omega_bar = fp32( (sum_{k} absmean_k, fp64, ascending k) / K )
    lambda_k  = fp32( fp64(omega_bar) / fp64(absmean_k) ), or 1 if absmean_k = 0
    cas_mode 0 is the Lambda_1 case "lambda^i is exceptionally set as a
    constant", constant = 1 (reading A10).
    """
    W = np.asarray(W, dtype=np.float64)
    N, K = W.shape
    if cas_mode == 0:
        lam = np.ones(K, dtype=np.float64)
    elif cas_mode == 1:
        acc = np.zeros(K, dtype=np.float64)
        for n in range(N):                 # sequential, ascending n, fp64 RNE adds
            acc = acc + np.abs(W[n])
        absmean = f32(acc / N)
        s = 0.0
        for k in range(K):                 # sequential, ascending k
            s = s + float(absmean[k])
        omega_bar = float(f32(s / K))
        with np.errstate(divide="ignore"):
            lam = np.where(absmean > 0, f32(omega_bar / np.where(absmean > 0, absmean, 1.0)), 1.0)
    else:
        raise ValueError("cas_mode must be 0 or 1")
    c = bf16_rn((np.float32(1.0) / lam.astype(np.float32)).astype(np.float64))
    return lam, c


def cas_apply(W, lam):
    """W2: W_bar = fp32(W) * lambda (IEEE fp32 multiply, one rounding)."""
    return (np.asarray(W, dtype=np.float32) * np.asarray(lam, dtype=np.float32)[None, :]).astype(np.float64)


# ------------------------------------------------------------------------- W3
def pts_exponent(W_bar):
    """W3: Definition 2, searched literally over n = 0, 1, ..., 60.

    Condition 1 (eq:pts_first_condition): S(W 2^n) = S(W 2^{n+i}) for all i,
      S(W) = sum max(0, 7*2^-9 - |w|).  Every term is non-increasing in the
      scale and a nonzero |w| strictly lowers its term when doubled while
      below the threshold, so the condition holds iff every nonzero |w| has
      |w| * 2^n >= 7*2^-9 (zeros contribute the constant 7*2^-9); we test that
      termwise with exact comparisons (reading A12; pinned against an
      exact-rational evaluation of S in tests).
    Condition 2 (eq:pts_second_condition): some w with
      7 * 2^(5-n) <= |w| < 7 * 2^(6-n).
    Returns (n, reason) with reason in {"underflow-stable", "overflow-risk"}.
    Raises ValueError when no n <= 60 qualifies (S:237 guard).
    """
    a = np.abs(np.asarray(W_bar, dtype=np.float64)).ravel()
    nz = a[a > 0]
    mnz = nz.min() if nz.size else None
    for n in range(PTS_MAX_N + 1):
        cond1 = mnz is None or mnz * 2.0 ** n >= UNDERFLOW_T
        lo, hi = 7.0 * 2.0 ** (5 - n), 7.0 * 2.0 ** (6 - n)
        cond2 = bool(np.any((a >= lo) & (a < hi)))
        if cond1 or cond2:
            return n, ("underflow-stable" if cond1 else "overflow-risk")
    raise ValueError("PTS: no exponent n <= 60 (degenerate tensor)")


def underflow_score(W):
    """S(W) of eq:pts_first_condition, in float64 (reporting only)."""
    a = np.abs(np.asarray(W, dtype=np.float64))
    return float(np.sum(np.maximum(0.0, UNDERFLOW_T - a)))


def underflow_group_fraction(W, group=GROUP):
    """Share of 128-groups whose max |w| < 7*2^-9 (App. E.3)."""
    W = np.asarray(W, dtype=np.float64)
    N, K = W.shape
    m = np.abs(W).reshape(N, K // group, group).max(axis=2)
    return float(np.mean(m < UNDERFLOW_T))


# --------------------------------------------------------------------- W4 / W5
SEVEN_GRID = 7.0 * E4M3_POS_GRID       # exact in float64


def group_scale(m):
    """W4: sigma = largest E4M3 value s >= 0 with 7*s <= m (capped at 448).

    This is max|w|/7 rounded toward zero onto the FP8 grid, in exact
    arithmetic (Eq. 1 + Lemma 1).  m: group max-abs values (>= 0).
    """
    m = np.asarray(m, dtype=np.float64)
    idx = np.searchsorted(SEVEN_GRID, m, side="right") - 1
    return E4M3_POS_GRID[np.clip(idx, 0, 126)]


def group_codes(w, sigma):
    """W5: clamp(round_half_even(w / sigma), -8, 7); sigma = 0 -> 0.

    w / sigma is computed in float64: w has a 24-bit and sigma a 4-bit
    significand, so an exact quotient that is not a half-integer lies more
    than 2^-28 (relative to 8) from one, far beyond float64 rounding; np.rint
    is round-half-even.  Pinned against exact rationals in the tests.
    """
    w = np.asarray(w, dtype=np.float64)
    sigma = np.asarray(sigma, dtype=np.float64)
    safe = np.where(sigma > 0, sigma, 1.0)
    q = np.rint(w / safe)
    return np.where(sigma > 0, np.clip(q, -8, 7), 0).astype(np.int8)


def quantize_groups(W_tilde):
    """W4+W5 over a [N][K] matrix: returns (sigma [N][K/128], codes [N][K])."""
    W_tilde = np.asarray(W_tilde, dtype=np.float64)
    N, K = W_tilde.shape
    if K % GROUP:
        raise ValueError("K must be a multiple of 128 (no padding, S:195)")
    G = K // GROUP
    m = np.abs(W_tilde).reshape(N, G, GROUP).max(axis=2)
    sigma = group_scale(m)
    codes = group_codes(W_tilde.reshape(N, G, GROUP), sigma[:, :, None]).reshape(N, K)
    return sigma, codes


# --------------------------------------------------------------------- W1..W6
class QuantizedWeight:
    """Everything fireq_quantize_weight produces, as plain arrays."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


def quantize_weight(W, cas_mode, pack=True, rows=None, lam=None):
    """W1-W6 for a bf16 weight matrix W [N][K] (float64 array of bf16 values).

    pack=False skips W6 (packed/scales are None) for large sampled checks.
    rows (with pack=False): W4-W5 only for those output rows -- CAS (W1) and PTS (W3)
    are still computed over the whole tensor, as their definitions require; W4-W5 act
    on each row independently, so sigma/codes of a row do not depend on the others.

    Returns QuantizedWeight with: lam (fp32 values), c (bf16 values),
    n (PTS exponent), reason, sigma [N][G] (values), sigma_codes [N][G],
    codes [N][K] int8, packed (uint8, layout v1), scales (uint8, layout v1).
    """
    W = np.asarray(W, dtype=np.float64)
    N, K = W.shape
    if N % layout.TILE_N or K % GROUP:
        raise ValueError("N and K must be multiples of 128")
    if not np.all(np.isfinite(W)):
        raise ValueError("non-finite weight")
    lam, c = cas_lambda(W, cas_mode) if lam is None else given_lambda(lam)
    W_bar = cas_apply(W, lam)
    n, reason = pts_exponent(W_bar)
    if rows is not None:
        if pack:
            raise ValueError("rows= needs pack=False")
        W_bar = W_bar[np.asarray(rows)]
    W_tilde = W_bar * 2.0 ** n                     # exact power-of-two scaling
    sigma, codes = quantize_groups(W_tilde)
    sigma_codes = e4m3_encode(sigma)
    return QuantizedWeight(lam=lam, c=c, n=n, reason=reason, W_bar=W_bar,
                           sigma=sigma, sigma_codes=sigma_codes, codes=codes,
                           packed=layout.pack_codes(codes) if pack else None,
                           scales=layout.pack_scales(sigma_codes) if pack else None)


# ---------------------------------------------------------- sigma_BF16 variant
def quantize_weight_bf16s(W, cas_mode, pack=True, rows=None):
    """The paper's comparison variant with BF16 group scales (App. B.1 P:525-527;
    DESIGN reading R25): W1-W3 unchanged (CAS, PTS), then per 128-group

      sigma = bf16_RN(max|W_tilde| / 7)        (no toward-zero step: Lemma 1 concerns FP8)
      code  = clamp(RNE(W_tilde / sigma), -8, 7),  sigma = 0 -> 0

    The dequantized weight is code * sigma exactly (no FP8 re-rounding).  Returns the fields of
    quantize_weight with sigma_bits (uint16 [N][G]) and scales16 (blocked uint16, layout v1
    order) in place of the FP8 codes.
    """
    W = np.asarray(W, dtype=np.float64)
    N, K = W.shape
    if N % layout.TILE_N or K % GROUP:
        raise ValueError("N and K must be multiples of 128")
    lam, c = cas_lambda(W, cas_mode)
    W_bar = cas_apply(W, lam)
    n, reason = pts_exponent(W_bar)
    if rows is not None:
        if pack:
            raise ValueError("rows= needs pack=False")
        W_bar = W_bar[np.asarray(rows)]
    W_tilde = W_bar * 2.0 ** n
    Nr = W_tilde.shape[0]
    m = np.abs(W_tilde).reshape(Nr, K // GROUP, GROUP).max(axis=2)
    sigma = bf16_rn(m / 7.0)
    codes = group_codes(W_tilde.reshape(Nr, K // GROUP, GROUP), sigma[:, :, None]).reshape(Nr, K)
    sigma_bits = (sigma.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    return QuantizedWeight(lam=lam, c=c, n=n, reason=reason, sigma=sigma, sigma_bits=sigma_bits, codes=codes,
                           packed=layout.pack_codes(codes) if pack else None,
                           scales16=layout.pack_scales16(sigma_bits) if pack else None)


# ------------------------------------------------------------------- A1 .. A3
def quantize_act(X, c=None):
    """A1-A3 for X bf16 [M][K] (float64 array of bf16 values).

    Returns (x_codes uint8 [M][K] E4M3, beta float64 [M] (bf16 values)).
    """
    X = np.asarray(X, dtype=np.float64)
    if c is not None:
        Xp = bf16_rn(X * np.asarray(c, dtype=np.float64)[None, :])   # product exact in fp64
    else:
        Xp = X
    amax = np.abs(Xp).max(axis=1)
    beta = np.where(amax > 0, bf16_rn(amax / E4M3_MAX), 1.0)
    xq = e4m3_rn(Xp / beta[:, None])
    return e4m3_encode(xq), beta
