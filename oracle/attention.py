"""KV4Q8 attention (FireQ section 3.2) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper quantizes queries to FP8 and keys / values to INT4 (KV4Q8-FP) and
runs the attention score S = Q K^T and the output O = P V through the same INT4 x FP8 kernel
as the linear layers.  Readings (R30-R37):

  RoPE        rotate-half pairing (k_i, k_j), j = i + d/2 -- the pairing Theorem 1 names
              (P:209-215); theta = 10000, positions 0..N-1.
  RPN         Stage 1, pre-RoPE, offline (Theorem 1): s_i = s_j =
              alpha * max_n ||(k_i^n, k_j^n)||_2; K_pre / s, inverse merged into W_q.
  CRS         Stage 2, post-RoPE, online: t_i = beta * max_n |k_i^n| for the
              outlier channels and (separately) their pair channels, 1 elsewhere;
              k' = k / t on the key side (lambda = fp32(1/t) in the INT4 quantizer's W2 step),
              q' = bf16(q * t) on the query side (A1 with c = t).
  K cache     post-RoPE per-token quantization: each (token, head) row of d = 128
              is one 128-group: sigma = RZ_E4M3(max|k'| / 7), codes RNE clamp [-8, 7] --
              the weight quantizer W2-W6 with the given lambda (PTS exponent n_k per head),
              K [N][d] in layout v1 (rows = tokens).
  V cache     groups of 128 consecutive TOKENS of one channel: V^T [d][N] quantized by
              W3-W6 (n_v per head), layout v1 (rows = channels) -- so that O = P V is the
              linear-layer GEMM with V^T as the weight (the paper transposes V on load,
              P:236; here the cache is stored transposed).
  Q           per (token, head) row: A1-A3 (beta_q bf16, E4M3 codes).
  scores      S = G2(Q_hat, K) (LUT re-rounding, fp64 sum), x = tau * S with tau = 1/sqrt(d),
              causal mask (kv > q -> excluded).
  softmax     Alg. 1 with B_c = 128 kv per tile: running max m_i, s_i =
              exp(m_old - m_new), P_ij = exp(x_ij - m_new), l_i = s_i l_i + rowsum(P_ij)
              (fp64 here; the GPU in fp32).
  P_hat       E4M3_RN(448 * P_ij) per tile: P in (0, 1], so beta_P = 1/448 uses the full FP8
              range (the softmax quantized to FP8).
  output      O_i = s_i O_i + G2(P_hat_ij, V_j^T) per tile; O = O_i 2^-n_v / 448 / l_i, BF16.
"""
import numpy as np

from .numerics import bf16_rn, e4m3_rn, e4m3_encode, E4M3_POS_GRID
from . import gemm, quant


def rope(X, theta=10000.0):
    """X [N][d] (float64) -> RoPE(X) with pairs (i, i + d/2), position n = row index."""
    X = np.asarray(X, dtype=np.float64)
    N, d = X.shape
    h = d // 2
    inv = theta ** (-np.arange(h, dtype=np.float64) * 2.0 / d)
    ang = np.arange(N, dtype=np.float64)[:, None] * inv[None, :]
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = X[:, :h], X[:, h:]
    return np.concatenate([x1 * c - x2 * s, x1 * s + x2 * c], axis=1)


def rpn_scales(K_pre, alpha):
    """Theorem 1: s_i = s_j = alpha * max_n ||(k_i^n, k_j^n)||_2, j = i + d/2."""
    K_pre = np.asarray(K_pre, dtype=np.float64)
    d = K_pre.shape[1]
    h = d // 2
    norm = np.sqrt(K_pre[:, :h] ** 2 + K_pre[:, h:] ** 2).max(axis=0)
    s = alpha * norm
    return np.concatenate([s, s])


def crs_scales(K_post, outlier_channels, beta):
    """CRS: t_i = beta * max_n |k_i^n| for each outlier channel i and, separately,
    for its RoPE pair channel; 1 for every other channel."""
    K_post = np.asarray(K_post, dtype=np.float64)
    d = K_post.shape[1]
    t = np.ones(d)
    for i in outlier_channels:
        for c in (i, (i + d // 2) % d):
            m = np.abs(K_post[:, c]).max()
            t[c] = beta * m if m > 0 else 1.0
    return t


class KV4Head:
    """One KV head's quantized cache: K (layout v1, rows = tokens) and V^T (rows = channels)."""

    def __init__(self, K_post, V, t=None):
        K_post = np.asarray(K_post, dtype=np.float64)
        V = np.asarray(V, dtype=np.float64)
        N, d = K_post.shape
        lam = None if t is None else (np.float32(1.0) / np.asarray(t, dtype=np.float32)).astype(np.float64)
        self.k = quant.quantize_weight(K_post, 0, lam=lam)     # W2 (k / t) .. W6 per token row
        self.vt = quant.quantize_weight(V.T.copy(), 0)          # W3 .. W6 per 128-token group
        self.N, self.d = N, d
        self.k_deq = gemm.dequantize_weight(self.k.packed, self.k.scales, N, d)
        self.vt_deq = gemm.dequantize_weight(self.vt.packed, self.vt.scales, d, N)


def e4m3_rounding_ambiguity(v, delta):
    """v = 448 P >= 0 (the FP8 softmax argument).  E4M3_RN(v) is decided by which side of the
    midpoint between its two grid neighbours v lies; an exp evaluated to a relative error
    below delta (the GPU's fp32 argument and ex2.approx, DESIGN R37) may land on the other
    side when |v - midpoint| <= delta * v.  Returns (other neighbour - E4M3_RN(v)) there, 0
    elsewhere -- the largest change of that P_hat code either side may make."""
    v = np.asarray(v, dtype=np.float64)
    c = e4m3_rn(v)
    idx = np.searchsorted(E4M3_POS_GRID, c)
    up = E4M3_POS_GRID[np.minimum(idx + 1, len(E4M3_POS_GRID) - 1)]
    dn = E4M3_POS_GRID[np.maximum(idx - 1, 0)]
    other = np.where(v >= c, up, dn)
    mid = 0.5 * (c + other)
    amb = (other != c) & (np.abs(v - mid) <= delta * v)
    return np.where(amb, other - c, 0.0)


def attention_head(Q, kv, t=None, causal=True, tau=None, bc=128, amb_delta=None):
    """One query head against one KV4 head, Alg. 1 step by step with B_c = bc:
    running row max m, P_j = exp(x_j - m_new) quantized to FP8 per kv tile, O = s * O + P_hat_j V_j,
    l = s * l + rowsum(P_j), s = exp(m_old - m_new).  Q [N][d] bf16 values (post-RoPE).
    Returns (O bf16 values [N][d], O fp64 before the BF16 rounding, dict of intermediates).
    amb_delta: also return dict["ambiguity"] [N][d], the largest |O| change the P_hat codes
    within relative amb_delta of an E4M3 midpoint can make (e4m3_rounding_ambiguity, carried
    through the same recurrence as O with absolute values)."""
    Q = np.asarray(Q, dtype=np.float64)
    N, d = Q.shape
    tau = 1.0 / np.sqrt(d) if tau is None else tau
    c = None if t is None else bf16_rn(np.asarray(t, dtype=np.float64))
    q_codes, beta_q = quant.quantize_act(Q, c)                               # A1..A3
    S = gemm.gemm_reference(q_codes, beta_q, None, None, N, d, kv.k.n, w_deq=kv.k_deq)   # G2
    x = tau * S
    if causal:
        x = np.where(np.arange(N)[None, :] <= np.arange(N)[:, None], x, -np.inf)
    m = np.full(N, -np.inf)
    l = np.zeros(N)
    O = np.zeros((N, d))
    p_codes = np.zeros((N, N), dtype=np.uint8)
    A = np.zeros((N, d)) if amb_delta is not None else None
    with np.errstate(invalid="ignore"):
        for j0 in range(0, N, bc):
            xj = x[:, j0:j0 + bc]
            m_new = np.maximum(m, xj.max(axis=1))
            s = np.where(m_new == m, 1.0, np.exp(m - m_new))                 # exp(-inf) = 0 on tile 0
            Pj = np.exp(xj - m_new[:, None])
            l = s * l + Pj.sum(axis=1)
            pc = e4m3_encode(e4m3_rn(448.0 * Pj))                            # FP8 softmax tile
            p_codes[:, j0:j0 + bc] = pc
            O = s[:, None] * O + gemm.gemm_reference(pc, np.ones(N), None, None, d, bc, 0,
                                                     w_deq=kv.vt_deq[:, j0:j0 + bc])
            if A is not None:
                dP = np.abs(e4m3_rounding_ambiguity(448.0 * Pj, amb_delta))
                A = s[:, None] * A + dP @ np.abs(kv.vt_deq[:, j0:j0 + bc]).T
            m = m_new
    O = O * 2.0 ** (-kv.vt.n) / 448.0 / l[:, None]
    if A is not None:
        A = A * 2.0 ** (-kv.vt.n) / 448.0 / l[:, None]
    return bf16_rn(O), O, dict(q_codes=q_codes, beta_q=beta_q, S=S, m=m, l=l, p_codes=p_codes, ambiguity=A)


def attention_unquantized(Q, K, V, causal=True, tau=None):
    """Textbook softmax attention in fp64 (no quantization) -- the accuracy reference."""
    Q, K, V = (np.asarray(a, dtype=np.float64) for a in (Q, K, V))
    N, d = Q.shape
    tau = 1.0 / np.sqrt(d) if tau is None else tau
    x = tau * (Q @ K.T)
    if causal:
        x = np.where(np.arange(N)[None, :] <= np.arange(N)[:, None], x, -np.inf)
    P = np.exp(x - x.max(axis=1, keepdims=True))
    return (P / P.sum(axis=1, keepdims=True)) @ V
