"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Quantization, packing, LUT and activation encoding must match bit-exactly; the
GEMM must satisfy the G4 criterion (max |y - r| / max(|r|, 0.1 rms_row(r)) <= 1e-2,
DESIGN.md "Tolerance") against the oracle's fp64 reference, and be bit-exact on
the exactness corridor.  All inputs are seeded synthetic (synth/).
"""
import zlib

import numpy as np
import pytest
import torch

import synth
from oracle import gemm as og
from oracle import layout as ol
from oracle import numerics as nm
from oracle import quant as oq

pytestmark = pytest.mark.gpu

G4_TOL = 1e-2
DEV = "cuda"


def to_dev_bf16(bits):
    return synth.bits_to_torch(bits).to(DEV)


def bits_of(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


# ----------------------------------------------------------------- LUT
def test_lut_table_bit_exact(fireq):
    got = fireq.debug_lut_table().cpu().numpy().reshape(127, 16)
    assert np.array_equal(got, og.lut_of_luts())


# ------------------------------------------------------- weight quantizer
def check_weight(fireq, wbits, cas_mode):
    N, K = wbits.shape
    qw = fireq.quantize_weight(to_dev_bf16(wbits), cas_mode=cas_mode)
    torch.cuda.synchronize()
    ref = oq.quantize_weight(synth.bits_to_f64(wbits), cas_mode)
    ps = qw.pts_and_status.cpu().numpy()
    assert ps[1] == 0 and ps[0] == ref.n
    assert np.array_equal(qw.lam.cpu().numpy().astype(np.float64), ref.lam)
    assert np.array_equal(bits_of(qw.c), nm.bf16_to_bits(ref.c))
    assert np.array_equal(qw.scales.cpu().numpy(), ref.scales)
    assert np.array_equal(qw.packed.cpu().numpy(), ref.packed)
    return qw, ref


@pytest.mark.parametrize("N,K,cas", [(128, 128, 0), (256, 512, 1), (384, 1280, 1), (1024, 4096, 0), (4096, 4096, 1)])
def test_quantize_weight_synthetic(fireq, N, K, cas):
    check_weight(fireq, synth.weights(N, K, synth.layer_seed(1, N + K)), cas)


def test_quantize_weight_f_edge(fireq):
    import json, os
    from fractions import Fraction
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "f_edge.json")))
    K = 128 * g["K_groups"]
    W = np.zeros((128, K))
    for i, row in enumerate(g["rows"]):
        W[i, :len(row["values"])] = [float(Fraction(v)) for v in row["values"]]
    qw, ref = check_weight(fireq, nm.bf16_to_bits(W), g["cas_mode"])
    assert ref.n == g["pts_n"]


@pytest.mark.parametrize("case", ["band224", "band448", "tiny", "ones", "neg_near_max", "zero_cols", "subnormal"])
def test_quantize_weight_edges(fireq, case):
    rng = np.random.default_rng(zlib.crc32(case.encode()))
    W = nm.bf16_rn(rng.standard_normal((256, 384)) * 0.02)
    if case == "band224":
        W[3, 7] = 224.0
    elif case == "band448":
        W[5, 9] = 448.0
        W[6, 1] = -447.0
    elif case == "tiny":
        W = nm.bf16_rn(W * 2.0 ** -30)
    elif case == "ones":
        W = np.ones_like(W)
    elif case == "neg_near_max":
        W[:, ::128] = -np.abs(W).max() * 1.01
        W = nm.bf16_rn(W)
    elif case == "zero_cols":
        W[:, 5:40] = 0.0
    elif case == "subnormal":
        W[0, 0] = 2.0 ** -130
        W = nm.bf16_rn(W)
    W = nm.bf16_rn(W)
    for cas in (0, 1):
        check_weight(fireq, nm.bf16_to_bits(W), cas)


def test_quantize_weight_nonfinite_status(fireq):
    W = np.ones((128, 128))
    bits = nm.bf16_to_bits(W)
    bits[3, 3] = 0x7FC0          # NaN
    qw = fireq.quantize_weight(to_dev_bf16(bits), cas_mode=0)
    assert int(qw.pts_and_status.cpu()[1]) == 1   # FIREQ_ERROR_INVALID_VALUE


# ---------------------------------------------------- activation quantizer
@pytest.mark.parametrize("M,K,with_c", [(1, 128, False), (16, 4096, True), (17, 11008, False), (300, 1024, True),
                                        (5, 14336, True),
                                        # M > 64: the persistent TMA-ring kernel (S = 8, 3, 2 stages;
                                        # rows per CTA > S, so every stage is reused)
                                        (2000, 4096, True), (700, 16384, False), (67, 12288, True),
                                        # several rows per stage slot: the ring wraps (phase flips)
                                        (6000, 4096, True), (3000, 11008, False)])
def test_quantize_act(fireq, M, K, with_c):
    xb = synth.activations(M, K, synth.layer_seed(2, M * 7 + K))
    X = synth.bits_to_f64(xb)
    X[0, :5] = [0.0, -0.0, 1e-30, -2.0 ** -130, 0.0]
    xb = nm.bf16_to_bits(nm.bf16_rn(X))
    if M > 2:
        xb[2, :] = 0                                # all-zero row -> beta = 1
    X = synth.bits_to_f64(xb)
    c = None
    cb = None
    if with_c:
        c = nm.bf16_rn(np.exp(np.random.default_rng(K).normal(0, 0.5, K)))
        cb = to_dev_bf16(nm.bf16_to_bits(c))
    xq, beta = fireq.quantize_act(to_dev_bf16(xb), chan_mul=cb)
    rq, rbeta = oq.quantize_act(X, c)
    assert np.array_equal(bits_of(beta), nm.bf16_to_bits(rbeta))
    assert np.array_equal(xq.cpu().numpy(), rq)


def test_quantize_act_exhaustive_bf16(fireq):
    """Every finite bf16 x' below the row amax, for several amax values (so beta = bf16(amax/448)
    spans exponents and mantissas): the reciprocal + residual-FMA quotient of the GPU encode
    must give the oracle's E4M3 codes bit-exactly (DESIGN reading R22)."""
    pos = np.arange(0x0000, 0x7F80, dtype=np.uint32)            # all finite non-negative bf16 patterns
    vals = (pos << 16).astype(np.uint32).view(np.float32).astype(np.float64)
    # ... plus rows whose beta = bf16(amax / 448) is below the fp32 normal range (1/beta
    # overflows: the encoder must fall back to the IEEE quotient)
    amaxes = [448.0, 1.0, 3.140625, 0.0078125 * 1.5, 2.0 ** -100 * 1.75, 57344.0, 1.0e30,
              2.0 ** -120, 2.0 ** -125 * 1.5]
    rows = []
    for A in amaxes:
        A = float(nm.bf16_rn(np.array([A]))[0])
        v = vals[vals <= A]
        rows.append(np.concatenate([v, -v, [A]]))
    K = (max(len(r) for r in rows) + 127) // 128 * 128
    X = np.zeros((len(rows), K))
    for i, r in enumerate(rows):
        X[i, : len(r)] = r
    xb = nm.bf16_to_bits(X)
    xq, beta = fireq.quantize_act(to_dev_bf16(xb))
    rq, rbeta = oq.quantize_act(X)
    assert np.array_equal(bits_of(beta), nm.bf16_to_bits(rbeta))
    assert np.array_equal(xq.cpu().numpy(), rq)


@pytest.mark.parametrize("M,K,ld", [(8, 256, 384), (1500, 4096, 4224), (130, 128, 1024)])
def test_quantize_act_strided(fireq, M, K, ld):
    """Row stride ld > K (M > 64: the row-ring kernel's bulk copies start at m * ld; K = 128:
    most of its threads own no vector)."""
    xb = synth.activations(M, ld, 77)
    Xd = to_dev_bf16(xb)[:, :K]
    xq, beta = fireq.quantize_act(Xd)
    rq, rbeta = oq.quantize_act(synth.bits_to_f64(xb)[:, :K])
    assert np.array_equal(xq.cpu().numpy(), rq)
    assert np.array_equal(bits_of(beta), nm.bf16_to_bits(rbeta))


# ----------------------------------------------------------------- GEMM
def run_case(fireq, M, N, K, cas=1, gamma=False, out_layout=0, seed=0):
    wb = synth.weights(N, K, synth.layer_seed(3, seed))
    xb = synth.activations(M, K, synth.layer_seed(4, seed))
    qw = fireq.quantize_weight(to_dev_bf16(wb), cas_mode=cas)
    xq, beta = fireq.quantize_act(to_dev_bf16(xb), chan_mul=qw.c)
    gam = None
    g_np = None
    if gamma:
        g_np = nm.f32(np.random.default_rng(seed).uniform(0.5, 2.0, N))
        gam = torch.from_numpy(g_np.astype(np.float32)).to(DEV)
    Y = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, gamma=gam, out_layout=out_layout)
    torch.cuda.synchronize()
    y = Y.float().cpu().numpy().astype(np.float64)
    if out_layout == 1:
        y = y.T
    # oracle reference from the oracle's own quantization of the same inputs
    ref = oq.quantize_weight(synth.bits_to_f64(wb), cas)
    rq, rbeta = oq.quantize_act(synth.bits_to_f64(xb), ref.c)
    assert np.array_equal(qw.packed.cpu().numpy(), ref.packed)
    assert np.array_equal(xq.cpu().numpy(), rq)
    r = og.gemm_reference(rq, rbeta, ref.packed, ref.scales, N, K, ref.n, gamma=g_np)
    return y, r, qw, xq, beta


@pytest.mark.parametrize("M,N,K", [
    (1, 128, 128), (7, 256, 512), (16, 512, 1024), (16, 1024, 4096), (17, 384, 640), (32, 256, 2048),
    (64, 640, 1024), (100, 256, 768), (128, 512, 512), (129, 256, 1024), (256, 384, 512), (300, 256, 384),
    (513, 128, 256),
    (2100, 256, 512), (4096, 384, 256),          # prefill tiles of 224 tokens, ragged last m-tile
])
def test_gemm_g4(fireq, M, N, K):
    y, r, *_ = run_case(fireq, M, N, K, seed=M * 131 + N + K)
    err = og.g4_error(y, r)
    assert err <= G4_TOL, f"G4 {err}"
    assert og.rel_frobenius(y, r) < 5e-3


@pytest.mark.parametrize("M,N,K", [
    (16, 10240, 256),        # stream-K (contributors' partials summed by the tile owner)
    (16, 4096, 1280),        # cluster split-K (DSMEM reduction in rank 0)
    (128, 1024, 2048),       # cluster split-K reduce-scatter (each rank emits its token chunks)
    (5, 128, 640),           # one tile over 5 CTAs
    (300, 512, 384),         # whole tiles, ragged m-tile
])
def test_gemm_residual(fireq, M, N, K):
    """fireq_w4a8_gemm_residual (Step 3's addition): G4 against the oracle's
    r + R in fp64; in place (R is Y) equals out of place bit for bit; a zero residual
    leaves every output as the plain GEMM's (x + 0 = x in fp32)."""
    y, r, qw, xq, beta = run_case(fireq, M, N, K, seed=7 * M + N)
    rb = synth.activations(M, N, synth.layer_seed(9, M + N))
    R = to_dev_bf16(rb)
    Y = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, residual=R)
    Y2 = R.clone()
    fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, residual=Y2, out=Y2)
    Y0 = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, residual=torch.zeros_like(R))
    torch.cuda.synchronize()
    rr = r + synth.bits_to_f64(rb)
    yv = Y.float().cpu().numpy().astype(np.float64)
    assert og.g4_error(yv, rr) <= G4_TOL and og.rel_frobenius(yv, rr) < 5e-3
    assert torch.equal(Y, Y2)
    assert np.array_equal(Y0.float().cpu().numpy().astype(np.float64), y)


@pytest.mark.parametrize("M,N,K,mode", [
    (16, 10240, 256, "stream-k"),            # 80 tiles: stream-K remainder over all CTAs
    (16, 4096, 1280, "cluster-split-k"),     # 32 tiles x 4-CTA clusters, ragged K split (10 / 4)
    (32, 256, 2048, "cluster-split-k"),      # NTOK 32: 3-CTA clusters, 16 groups / 3
    (5, 128, 640, "cluster-split-k"),        # one tile, 5 groups over 5 CTAs
])
def test_gemm_schedules(fireq, M, N, K, mode):
    """Each schedule of make_plan against the oracle, all output elements."""
    plan = fireq.gemm_plan(M, N, K)
    assert plan["mode"] == mode, plan          # schedules as chosen on a 148-SM B200
    y, r, *_ = run_case(fireq, M, N, K, seed=N + K)
    assert og.g4_error(y, r) <= G4_TOL
    assert og.rel_frobenius(y, r) < 5e-3


@pytest.mark.parametrize("M,N,K", [(16, 150 * 128, 512), (300, 75 * 128, 512)])
def test_gemm_hybrid_few_remainder_units(fireq, M, N, K):
    """Whole tiles for one full wave plus a remainder of 2 tiles whose 8 K-units are fewer than
    the CTAs: the units are shared by 8 CTAs only (a sharer without units would never publish
    its partial and the tile's owner would wait forever)."""
    plan = fireq.gemm_plan(M, N, K)
    assert plan["mode"] == "stream-k" and plan["ctas"] == 148, plan
    y, r, *_ = run_case(fireq, M, N, K, seed=N + M)
    assert og.g4_error(y, r) <= G4_TOL
    assert og.rel_frobenius(y, r) < 5e-3


@pytest.mark.parametrize("M", [16, 200, 13, 2100])
def test_gemm_transposed_output_and_gamma(fireq, M):
    """Y^T (the column-parallel layout) with gamma; M = 13: ldy = 13 (no 16-B row stores);
    M = 2100: ten 224-token m-tiles, consecutive segments of a CTA in different m-tiles (the
    per-token scales of one segment must not be overwritten by a warp already in the next)."""
    y, r, *_ = run_case(fireq, M, 256, 512, gamma=True, out_layout=1, seed=M)
    assert og.g4_error(y, r) <= G4_TOL


def test_gemm_transposed_many_mtiles_equals_row_major(fireq):
    """Y^T and Y of the same GEMM (same plan) agree bit for bit at many m-tiles per CTA."""
    M, N, K = 4100, 384, 256
    wb = synth.weights(N, K, 901)
    xb = synth.activations(M, K, 902)
    qw = fireq.quantize_weight(to_dev_bf16(wb))
    xq, beta = fireq.quantize_act(to_dev_bf16(xb), chan_mul=qw.c)
    g = torch.rand(N, device=DEV) + 0.5
    y = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, gamma=g)
    yt = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, gamma=g, out_layout=1)
    assert torch.equal(y, yt.t())


def test_gemm_exactness_corridor(fireq):
    """Integer operands, sigma = 1, beta = 1, n = 0, |partial sums| <= 256: bit-exact."""
    rng = np.random.default_rng(5)
    M, N, K = 16, 256, 1024
    codes = rng.integers(-2, 3, size=(N, K)).astype(np.int8)
    sc = np.full((N, K // 128), 56, dtype=np.uint8)           # E4M3 code 56 = 1.0
    sc[7, 3] = 0                                              # a zero-scale group contributes 0
    xi = np.zeros((M, K))
    for m in range(M):
        idx = rng.choice(K, 64, replace=False)
        xi[m, idx] = rng.integers(-2, 3, 64)
    packed = torch.from_numpy(ol.pack_codes(codes)).to(DEV)
    scales = torch.from_numpy(ol.pack_scales(sc)).to(DEV)
    xq = torch.from_numpy(nm.e4m3_encode(xi)).to(DEV)
    beta = torch.ones(M, dtype=torch.bfloat16, device=DEV)
    Y = fireq.w4a8_gemm(xq, beta, packed, scales, N, 0)
    wv = codes.astype(np.float64)
    wv[7, 384:512] = 0
    exact = xi @ wv.T
    assert np.abs(exact).max() <= 256
    assert np.array_equal(Y.float().cpu().numpy().astype(np.float64), exact)


def test_gemm_deterministic(fireq):
    M, N, K = 16, 1024, 4096
    wb = synth.weights(N, K, 11)
    xb = synth.activations(M, K, 12)
    qw = fireq.quantize_weight(to_dev_bf16(wb))
    xq, beta = fireq.quantize_act(to_dev_bf16(xb), chan_mul=qw.c)
    ws = fireq.Workspace(fireq.gemm_workspace_bytes(M, N, K))
    y1 = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, workspace=ws)
    y2 = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, workspace=ws)
    assert torch.equal(y1, y2)
    assert int(ws.t[: 4 * (N // 128)].view(torch.int32).abs().sum()) == 0   # counters left zeroed


@pytest.mark.parametrize("name,M", [("llama2-7b.gate", 16), ("llama2-7b.down", 16), ("llama3-8b.k", 16),
                                    ("llama3-8b.down", 16), ("llama2-7b.up", 1024),
                                    # mid-M (C5 sweep): pure stream-K with the bulk-staged owner fixup
                                    ("llama3-8b.down", 64), ("llama3-8b.down", 128), ("llama3-8b.down", 256),
                                    ("llama3-8b.k", 4096)])
def test_gemm_full_size_sampled(fireq, name, M):
    """BASELINE full shapes in the bench's launch configuration; oracle on sampled channels.

    The oracle quantizes the whole tensor (CAS and PTS are global) and the fp64
    reference is formed for 192 sampled output channels; the GPU packing of those
    rows is also compared bit-exactly with the oracle's codes and scales.
    """
    N, K = synth.SHAPES[name]
    wb = synth.weights(N, K, synth.layer_seed(1, 0))
    xb = synth.activations(M, K, synth.layer_seed(1, 1))
    qw = fireq.quantize_weight(to_dev_bf16(wb), cas_mode=1)
    xq, beta = fireq.quantize_act(to_dev_bf16(xb), chan_mul=qw.c)
    Y = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n)
    torch.cuda.synchronize()
    ref = oq.quantize_weight(synth.bits_to_f64(wb), 1, pack=False)
    assert qw.n == ref.n
    rq, rbeta = oq.quantize_act(synth.bits_to_f64(xb), ref.c)
    assert np.array_equal(xq.cpu().numpy(), rq)
    rows = np.sort(np.random.default_rng(3).choice(N, 192, replace=False))
    # GPU packing of the sampled rows == oracle codes / scale codes
    packed = qw.packed.cpu().numpy()
    scales = qw.scales.cpu().numpy()
    kk = np.arange(K)
    for n in rows[:16]:
        byte, half = ol.packed_byte_index(np.full(K, n), kk, K)
        nib = np.where(half == 0, packed[byte] & 15, packed[byte] >> 4).astype(np.int16)
        assert np.array_equal(np.where(nib >= 8, nib - 16, nib), ref.codes[n])
        assert np.array_equal(scales[ol.scale_index(np.full(K // 128, n), np.arange(K // 128), K)],
                              ref.sigma_codes[n])
    table = og.lut_of_luts()
    wdeq = nm.E4M3_DECODE[table[np.repeat(ref.sigma_codes[rows].astype(np.int64), 128, axis=1),
                                ref.codes[rows].astype(np.int64) & 15]]
    r = og.reference_rows(rq, rbeta, wdeq, ref.n)
    y = Y.float().cpu().numpy().astype(np.float64)[:, rows]
    assert og.g4_error(y, r) <= G4_TOL


def _sampled_parity(fireq, wb, Ms, gamma=False, n_chan=160, n_tok=48, seed=0):
    """Full-size GEMM in the bench's launch configuration vs the oracle on sampled outputs.

    The GPU quantizes the whole weight; the oracle computes CAS lambda and the PTS exponent
    over the whole tensor (global) and W4-W5 for the sampled channels only (per-row
    steps).  For each M in Ms the GPU runs the whole GEMM; the oracle forms the fp64 reference
    for n_tok sampled tokens x n_chan sampled channels (activation rows are quantized
    independently, A1-A3), and the GPU's X_hat / beta of the sampled tokens must equal the
    oracle's bit for bit.
    """
    N, K = wb.shape
    rng = np.random.default_rng(seed)
    chans = np.sort(rng.choice(N, n_chan, replace=False))
    qw = fireq.quantize_weight(to_dev_bf16(wb), cas_mode=1)
    torch.cuda.synchronize()
    ref = oq.quantize_weight(synth.bits_to_f64(wb), 1, pack=False, rows=chans)
    assert qw.n == ref.n
    assert np.array_equal(bits_of(qw.c), nm.bf16_to_bits(ref.c))
    # GPU packing of some sampled rows == oracle codes / scale codes
    packed = qw.packed.cpu().numpy()
    scales = qw.scales.cpu().numpy()
    kk = np.arange(K)
    for i in range(0, n_chan, n_chan // 8):
        n = chans[i]
        byte, half = ol.packed_byte_index(np.full(K, n), kk, K)
        nib = np.where(half == 0, packed[byte] & 15, packed[byte] >> 4).astype(np.int16)
        assert np.array_equal(np.where(nib >= 8, nib - 16, nib), ref.codes[i])
        assert np.array_equal(scales[ol.scale_index(np.full(K // 128, n), np.arange(K // 128), K)],
                              ref.sigma_codes[i])
    del packed
    table = og.lut_of_luts()
    wdeq = nm.E4M3_DECODE[table[np.repeat(ref.sigma_codes.astype(np.int64), 128, axis=1),
                                ref.codes.astype(np.int64) & 15]]
    g_np = gam = None
    if gamma:
        g_np = nm.f32(rng.uniform(0.5, 2.0, N))
        gam = torch.from_numpy(g_np.astype(np.float32)).to(DEV)
    errs = {}
    for M in Ms:
        xb = synth.activations(M, K, synth.layer_seed(5, M))
        xd = to_dev_bf16(xb)
        xq, beta = fireq.quantize_act(xd, chan_mul=qw.c)
        del xd
        Y = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, gamma=gam)
        torch.cuda.synchronize()
        toks = np.arange(M) if M <= n_tok else np.sort(np.concatenate(
            [[0, M - 1], rng.choice(np.arange(1, M - 1), n_tok - 2, replace=False)]))
        tk = torch.from_numpy(toks).to(DEV)
        rq, rbeta = oq.quantize_act(synth.bits_to_f64(xb[toks]), ref.c)
        assert np.array_equal(xq[tk].cpu().numpy(), rq)
        assert np.array_equal(bits_of(beta[tk]), nm.bf16_to_bits(rbeta))
        r = og.reference_rows(rq, rbeta, wdeq, ref.n, gamma_rows=None if g_np is None else g_np[chans])
        y = Y[tk][:, torch.from_numpy(chans).to(DEV)].float().cpu().numpy().astype(np.float64)
        errs[M] = og.g4_error(y, r)
        del Y, xq, beta
        torch.cuda.empty_cache()
    assert all(e <= G4_TOL for e in errs.values()), errs
    return errs


def test_gemm_bench_gate_up_full_size(fireq):
    """The headline bench GEMM exactly: Llama2-7B [gate; up] 22016 x 4096 quantized as ONE
    matrix (reading R20), with a per-channel gamma, at M = 16 (hybrid whole-tile + stream-K
    plan) and at the prefill size M = 16 x 1024."""
    wg = synth.weights(11008, 4096, synth.layer_seed(1, 0))
    wu = synth.weights(11008, 4096, synth.layer_seed(1, 1))
    plan = fireq.gemm_plan(16, 22016, 4096)
    assert plan["mode"] == "stream-k" and plan["ctas"] == 148, plan
    _sampled_parity(fireq, np.concatenate([wg, wu], axis=0), [16, 16384], gamma=True)


@pytest.mark.parametrize("name", ["llama2-70b.gate", "llama2-70b.down", "llama3-8b.down"])
def test_gemm_large_shapes_sampled(fireq, name):
    """BASELINE C4 (Llama2-70B FFN, K up to 28672 -- the longest accumulation) and C3/C5's
    Llama3-8B down_proj, at decode M = 16 and prefill M = 16384."""
    N, K = synth.SHAPES[name]
    _sampled_parity(fireq, synth.weights(N, K, synth.layer_seed(4, N + K)), [16, 16384])


def test_cooperative_launch_same_result(fireq):
    """FIREQ_COOPERATIVE=1 (co-residency guaranteed by a cooperative launch, also inside a
    CUDA graph) gives the same bits as the default launch for a stream-K plan."""
    import os, subprocess, sys
    M, N, K = 16, 22016, 1024
    wb = synth.weights(N, K, 1501)
    xb = synth.activations(M, K, 1502)
    qw = fireq.quantize_weight(to_dev_bf16(wb))
    xq, beta = fireq.quantize_act(to_dev_bf16(xb), chan_mul=qw.c)
    y = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n).cpu()
    assert fireq.gemm_plan(M, N, K)["mode"] == "stream-k"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, torch; sys.path.insert(0, %r)\n"
        "import synth\n"
        "from paper_2505_20839_b200 import fireq as F; F.load()\n"
        "wb = synth.weights(%d, %d, 1501); xb = synth.activations(%d, %d, 1502)\n"
        "qw = F.quantize_weight(synth.bits_to_torch(wb).cuda())\n"
        "xq, beta = F.quantize_act(synth.bits_to_torch(xb).cuda(), chan_mul=qw.c)\n"
        "ws = F.Workspace(F.gemm_workspace_bytes(%d, %d, %d)); out = torch.empty(%d, %d, dtype=torch.bfloat16, device='cuda')\n"
        "s = torch.cuda.Stream()\n"
        "F.w4a8_gemm(xq, beta, qw.packed, qw.scales, %d, qw.n, out=out, workspace=ws, stream=s); torch.cuda.synchronize()\n"
        "g = torch.cuda.CUDAGraph()\n"
        "with torch.cuda.graph(g, stream=s):\n"
        "    F.w4a8_gemm(xq, beta, qw.packed, qw.scales, %d, qw.n, out=out, workspace=ws, stream=s)\n"
        "out.zero_(); g.replay(); torch.cuda.synchronize()\n"
        "torch.save(out.cpu(), sys.argv[1])\n") % (root, N, K, M, K, M, N, K, M, N, N, N)
    tmp = os.path.join(root, "gpurun_out", "coop_y.pt")
    os.makedirs(os.path.dirname(tmp), exist_ok=True)
    r = subprocess.run([sys.executable, "-c", code, tmp], env=dict(os.environ, FIREQ_COOPERATIVE="1"),
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout + r.stderr
    assert torch.equal(torch.load(tmp), y)


@pytest.mark.parametrize("M,N,K", [(16, 448 * 128, 512), (32, 300 * 128, 256)])
def test_gemm_decode_tail_wave_split(fireq, M, N, K):
    """Decode tiles beyond whole waves: 448 tiles = 3 waves of 148 + 4; the 4 remaining tiles
    are split stream-K over all CTAs instead of forming a 4th wave."""
    plan = fireq.gemm_plan(M, N, K)
    assert plan["mode"] == "stream-k" and plan["ctas"] == 148, plan
    y, r, *_ = run_case(fireq, M, N, K, seed=N + 7)
    assert og.g4_error(y, r) <= G4_TOL
