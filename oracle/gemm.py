"""FireQ INT4 x FP8 linear layer: LUT dequantization and fp64 reference GEMM.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

G1  LUT  (Step 1): for each group scale sigma the 16 FP8 entries
         {-8 sigma, ..., 7 sigma}, i.e. LUT[v] = E4M3_RN(v * sigma) -- the
         product v*sigma is exact, then one FP8 rounding (reading A6).
         Indexed here by the 4-bit nibble u = v & 0xF.
G2  reference (Steps 2-3; PTS inverse on the output, P:175;
         Y = X W^T):
         r[m, n] = gamma_n * beta_m * 2^-n_pts * sum_k dec(x_hat[m,k]) * dec(LUT_{n,g(k)}[code[n,k]])
         with the contraction done by a float64 library matmul (products of
         two E4M3 values are exact in float64; only the summation rounds).
G4  criterion: max_{m,n} |y - r| / max(|r|, 0.1 * rms_m(r)) <= 1e-2
         (north_star "max rel err <= 1e-2", floored per row -- reading G4).
"""
import numpy as np

from .numerics import E4M3_DECODE, E4M3_POS_GRID, e4m3_encode, e4m3_rn
from . import layout

NIBBLE_VALUES = np.array([u if u < 8 else u - 16 for u in range(16)], dtype=np.float64)


def lut_for_sigma(sigma):
    """G1: 16 E4M3 codes LUT[u], u = nibble (u >= 8 encodes v = u - 16)."""
    return e4m3_encode(e4m3_rn(NIBBLE_VALUES * float(sigma)))


def lut_of_luts():
    """[127][16] uint8: LUT for every non-negative finite sigma code 0..126."""
    return np.stack([lut_for_sigma(s) for s in E4M3_POS_GRID])


def dequantize_weight(packed, scales, N, K):
    """W_deq [N][K] float64: dec(LUT_{n,g}[code]) (the value the kernel feeds the MMA)."""
    codes = layout.unpack_codes(packed, N, K).astype(np.int64)
    sc = layout.unpack_scales(scales, N, K)                  # [N][G] codes
    table = lut_of_luts()                                    # [127][16]
    nib = codes & 0xF
    sc_full = np.repeat(sc, layout.GROUP, axis=1)
    return E4M3_DECODE[table[sc_full, nib]]


def gemm_reference(x_codes, beta, packed, scales, N, K, pts_n, gamma=None, w_deq=None, residual=None):
    """G2: r [M][N] float64.  residual (values [M][N]): Step 3's element-wise addition fused
    into the epilogue ("activation function, addition ..."), r + R in fp64."""
    x = E4M3_DECODE[np.asarray(x_codes, dtype=np.uint8)]
    if w_deq is None:
        w_deq = dequantize_weight(packed, scales, N, K)
    acc = x @ w_deq.T
    r = acc * np.asarray(beta, dtype=np.float64)[:, None] * 2.0 ** (-pts_n)
    if gamma is not None:
        r = r * np.asarray(gamma, dtype=np.float64)[None, :]
    if residual is not None:
        r = r + np.asarray(residual, dtype=np.float64)
    return r


def reference_rows(x_codes, beta, w_deq_rows, pts_n, gamma_rows=None, residual_cols=None):
    """G2 for a subset of output channels (w_deq_rows [n_sel][K]) -- for sampled checks."""
    x = E4M3_DECODE[np.asarray(x_codes, dtype=np.uint8)]
    r = (x @ np.asarray(w_deq_rows).T) * np.asarray(beta, dtype=np.float64)[:, None] * 2.0 ** (-pts_n)
    if gamma_rows is not None:
        r = r * np.asarray(gamma_rows, dtype=np.float64)[None, :]
    if residual_cols is not None:
        r = r + np.asarray(residual_cols, dtype=np.float64)
    return r


def gemm_reference_bf16s(x_codes, beta, codes, sigma, pts_n):
    """G2 for the sigma_BF16 variant: r = beta 2^-n sum_k dec(x_hat) * code * sigma_{n,g(k)} (fp64; the
    products code * sigma are exact).  codes int [N][K], sigma float64 [N][K/128]."""
    x = E4M3_DECODE[np.asarray(x_codes, dtype=np.uint8)]
    w = np.asarray(codes, dtype=np.float64) * np.repeat(np.asarray(sigma, dtype=np.float64), layout.GROUP, axis=1)
    return (x @ w.T) * np.asarray(beta, dtype=np.float64)[:, None] * 2.0 ** (-pts_n)


def g4_error(y, r):
    """G4: max over (m, n) of |y - r| / max(|r|, 0.1 * rms of row m of r)."""
    y = np.asarray(y, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    rms = np.sqrt(np.mean(r * r, axis=1, keepdims=True))
    den = np.maximum(np.abs(r), 0.1 * rms)
    err = np.abs(y - r)
    ratio = np.where(den > 0, err / np.where(den > 0, den, 1.0), np.where(err > 0, np.inf, 0.0))
    return float(ratio.max()) if ratio.size else 0.0


def rel_frobenius(y, r):
    y = np.asarray(y, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    d = np.linalg.norm(r)
    return float(np.linalg.norm(y - r) / d) if d > 0 else float(np.linalg.norm(y))


def dequant_cost_ops(b, d_in, d_out):
    """App. A.1: dequantization overhead (b + d_in) * d_out."""
    return (b + d_in) * d_out
