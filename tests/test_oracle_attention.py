"""Pins of oracle/attention.py (KV4Q8 attention, FireQ section 3.2) against the paper's
Theorem 1, closed forms and special cases -- not against the oracle itself."""
import numpy as np
import pytest

from oracle import attention as oa
from oracle import gemm as og
from oracle import numerics as nm
from oracle import quant as oq


def test_rope_rotates_pairs():
    """RoPE is a rotation of each (i, i + d/2) pair: pair norms are preserved, position 0 is
    the identity, and q_m . k_n depends only on m - n (the relative-position property)."""
    rng = np.random.default_rng(1)
    N, d = 64, 128
    X = rng.standard_normal((N, d))
    R = oa.rope(X)
    h = d // 2
    assert np.allclose(np.hypot(R[:, :h], R[:, h:]), np.hypot(X[:, :h], X[:, h:]), rtol=1e-12)
    assert np.array_equal(R[0], X[0])
    q, k = rng.standard_normal(d), rng.standard_normal(d)
    Rq, Rk = oa.rope(np.tile(q, (N, 1))), oa.rope(np.tile(k, (N, 1)))
    assert np.isclose(Rq[10] @ Rk[3], Rq[40] @ Rk[33], rtol=1e-10)


def test_rpn_theorem1_bound():
    """Theorem 1: with s_i = s_j = alpha max_n ||(k_i, k_j)||, every scaled pair has
    norm <= 1/alpha, with equality for the maximizing token -- before AND after RoPE."""
    rng = np.random.default_rng(2)
    N, d, alpha = 200, 128, 1.7
    K = rng.standard_normal((N, d)) * np.exp(rng.standard_normal(d))     # uneven channel scales
    s = oa.rpn_scales(K, alpha)
    h = d // 2
    assert np.array_equal(s[:h], s[h:])
    for Ks in (K / s, oa.rope(K / s)):
        norms = np.hypot(Ks[:, :h], Ks[:, h:])
        assert norms.max() <= 1 / alpha * (1 + 1e-12)
        assert np.allclose(norms.max(axis=0), 1 / alpha, rtol=1e-12)


def test_crs_scales():
    """CRS: outlier channels and their pairs get t = beta max|k| (so max|k/t| = 1/beta),
    every other channel t = 1."""
    rng = np.random.default_rng(3)
    K = rng.standard_normal((100, 128))
    K[:, 5] *= 40.0
    t = oa.crs_scales(K, [5], beta=2.0)
    assert np.isclose(np.abs(K[:, 5] / t[5]).max(), 0.5) and np.isclose(np.abs(K[:, 69] / t[69]).max(), 0.5)
    assert np.all(t[[c for c in range(128) if c not in (5, 69)]] == 1.0)


def _case(N, seed, outlier=None):
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((N, 128))
    if outlier is not None:
        K[:, outlier] *= 30.0
    return (nm.bf16_rn(rng.standard_normal((N, 128))), nm.bf16_rn(K), nm.bf16_rn(rng.standard_normal((N, 128))))


def test_uniform_scores_average_the_dequantized_values():
    """Q = 0: every logit is 0, so P = 1 and P_hat = E4M3(448) = 448 exactly, l = #visible keys,
    and O_q = mean of the dequantized value rows 0..q (closed form, causal)."""
    N = 256
    _, K, V = _case(N, 4)
    kv = oa.KV4Head(K, V)
    _, O, st = oa.attention_head(np.zeros((N, 128)), kv)
    assert np.all(nm.e4m3_decode(st["p_codes"])[np.tril(np.ones((N, N), bool))] == 448.0)
    v_deq = kv.vt_deq.T * 2.0 ** (-kv.vt.n)                # [N][d] dequantized values
    expect = np.cumsum(v_deq, axis=0) / np.arange(1, N + 1)[:, None]
    assert np.allclose(O, expect, rtol=1e-12, atol=1e-14)


def test_first_query_returns_first_value_row():
    """Causal row 0 sees one key: P = 1, O_0 = the dequantized V row 0 exactly."""
    Q, K, V = _case(128, 5)
    kv = oa.KV4Head(K, V)
    _, O, _ = oa.attention_head(Q, kv)
    assert np.array_equal(O[0], kv.vt_deq[:, 0] * 2.0 ** (-kv.vt.n))


def test_kv_quantization_is_the_weight_quantizer_per_row():
    """K rows are single 128-groups: sigma = RZ(max|k| / 7) per token (W4), V^T groups are 128
    tokens of one channel; both are W2-W6 of the weight quantizer with the given lambda."""
    Q, K, V = _case(256, 6)
    kv = oa.KV4Head(K, V)
    Kt = K * 2.0 ** kv.k.n
    assert np.array_equal(kv.k.sigma[:, 0], oq.group_scale(np.abs(Kt).max(axis=1)))
    assert kv.vt.sigma.shape == (128, 2)


def test_crs_lowers_the_key_quantization_error():
    """The point of CRS: with an outlier key channel, per-token INT4 scales are set
    by the outlier; dividing it out (and multiplying the query channel) lowers the attention
    error against unquantized fp64 attention.  beta = 1/4 brings the outlier channel to
    max |k / t| = 4, the range of the regular N(0, 1) channels."""
    N = 256
    Q, K, V = _case(N, 7, outlier=9)
    ref = oa.attention_unquantized(Q, K, V)
    _, O0, _ = oa.attention_head(Q, oa.KV4Head(K, V))
    t = nm.bf16_rn(oa.crs_scales(K, [9], beta=0.25))
    _, O1, _ = oa.attention_head(Q, oa.KV4Head(K, V, t=t), t=t)
    e0, e1 = (np.linalg.norm(O - ref) / np.linalg.norm(ref) for O in (O0, O1))
    assert e1 < 0.5 * e0, (e0, e1)


def test_kv4q8_accuracy_regression():
    """End-to-end KV4Q8 error on Gaussian inputs vs fp64 attention (pinned regression value,
    INT4 keys/values dominate; informational like G5)."""
    Q, K, V = _case(512, 8)
    _, O, _ = oa.attention_head(Q, oa.KV4Head(K, V))
    ref = oa.attention_unquantized(Q, K, V)
    e = np.linalg.norm(O - ref) / np.linalg.norm(ref)
    assert 0.08 < e < 0.25, e


def _two_pass(S, kv, N, bug=None):
    """Softmax attention from the oracle's scores with the EXACT row max (two passes), optionally
    with a plausible bug -- to calibrate G4 against Alg. 1's running-max tile order."""
    tau = 1.0 / np.sqrt(128)
    x = (S if bug == "no_tau" else tau * S)
    if bug != "no_mask":
        x = np.where(np.tril(np.ones((N, N), bool)), x, -np.inf)
    P = np.exp(x - x.max(axis=1, keepdims=True))
    l = P.sum(axis=1)
    pc = nm.e4m3_encode(nm.e4m3_rn((1.0 if bug == "p_unscaled" else 448.0) * P))
    n_v = kv.vt.n + (1 if bug == "v_pts" else 0)
    return og.gemm_reference(pc, np.full(N, 1.0 / 448.0), None, None, 128, N, n_v, w_deq=kv.vt_deq) / l[:, None]


def test_fp8_softmax_tile_order_is_visible():
    """Two-pass softmax (exact max, one FP8 grid per row) vs Alg. 1's running max (FP8 grid per
    tile) are both "softmax then FP8", but the FP8 decisions differ: a few outputs move by more
    than G4's 1e-2 (Frobenius < 2%).  So the oracle follows Alg. 1's tile order (B_c = 128)
    exactly as the kernel does (DESIGN R36), and G4 would catch a kernel that did not."""
    Q, K, V = _case(512, 9)
    kv = oa.KV4Head(K, V)
    _, O, st = oa.attention_head(Q, kv)
    T = _two_pass(st["S"], kv, 512)
    assert og.g4_error(T, O) > 1e-2 and og.rel_frobenius(T, O) < 2e-2


@pytest.mark.parametrize("bug", ["no_tau", "no_mask", "p_unscaled", "v_pts"])
def test_g4_rejects_attention_bugs(bug):
    """The G4 criterion used for the GPU parity (<= 1e-2) rejects plausible bugs in the softmax /
    scaling path."""
    Q, K, V = _case(256, 9)
    kv = oa.KV4Head(K, V)
    _, O, st = oa.attention_head(Q, kv)
    assert og.g4_error(_two_pass(st["S"], kv, 256, bug), O) > 5e-2


def test_e4m3_rounding_ambiguity_brute_force():
    """Nonzero exactly where v lies within delta * v of the midpoint between E4M3_RN(v) and its
    neighbour on v's side, and then equal to (that neighbour - E4M3_RN(v)): checked against a
    brute-force scan of the grid."""
    rng = np.random.default_rng(5)
    grid = nm.E4M3_POS_GRID
    mids = 0.5 * (grid[1:] + grid[:-1])
    delta = 2.0 ** -15
    # values at, just around and far from every midpoint, plus random values and the ends
    v = np.concatenate([mids, mids * (1 + 0.5 * delta), mids * (1 - 0.5 * delta), mids * (1 + 4 * delta),
                        mids * (1 - 4 * delta), rng.uniform(0, 448, 2000), [0.0, 448.0, 2.0 ** -9]])
    got = oa.e4m3_rounding_ambiguity(v, delta)
    for x, g in zip(v, got):
        c = float(nm.e4m3_rn(np.array([x]))[0])
        near = [m for m in mids if abs(x - m) <= delta * x]
        if not near:
            assert g == 0.0, x
        else:
            m = near[0]
            lo, hi = grid[grid < m].max(), grid[grid > m].min()
            assert {c, c + g} == {lo, hi}, (x, c, g)


def test_attention_ambiguity_bound_is_zero_without_slack_and_covers_code_flips():
    """amb_delta = 0 on random data: no P value sits exactly on a midpoint, so the bound is 0;
    with a slack, flipping every ambiguous code of a one-tile head (recomputing O by hand from
    the oracle's own intermediates) moves O by no more than the bound."""
    rng = np.random.default_rng(8)
    N, d = 128, 128
    Q = nm.bf16_rn(rng.normal(0, 1, (N, d)))
    K = nm.bf16_rn(rng.normal(0, 1, (N, d)))
    V = nm.bf16_rn(rng.normal(0, 1, (N, d)))
    kv = oa.KV4Head(K, V)
    _, _, st0 = oa.attention_head(Q, kv, causal=True, amb_delta=0.0)
    assert np.all(st0["ambiguity"] == 0.0)
    delta = 2.0 ** -6                                  # a large slack: many ambiguous codes
    _, O, st = oa.attention_head(Q, kv, causal=True, amb_delta=delta)
    x = st["S"] / np.sqrt(d)
    x = np.where(np.arange(N)[None, :] <= np.arange(N)[:, None], x, -np.inf)
    P = np.exp(x - st["m"][:, None])                   # one tile: m is the tile's max
    dP = oa.e4m3_rounding_ambiguity(448.0 * P, delta)
    assert np.count_nonzero(dP) > 0
    O_flip = O + (dP @ kv.vt_deq.T) * 2.0 ** (-kv.vt.n) / 448.0 / st["l"][:, None]
    assert np.all(np.abs(O_flip - O) <= st["ambiguity"] * (1 + 1e-12) + 1e-300)
