"""GPU tests for the FFN helpers and the transposed (Y^T) activation quantizers."""
import numpy as np
import pytest
import torch

import synth
from oracle import ffn as of
from oracle import gemm as og
from oracle import numerics as nm
from oracle import quant as oq

pytestmark = pytest.mark.gpu
DEV = "cuda"


def bits_of(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("M,K", [(16, 4096), (8, 11008), (3, 128), (300, 1024), (100, 11008), (64, 256)])
def test_quantize_act_transposed_bit_exact(fireq, M, K):
    xb = synth.activations(M, K, 31)
    X = synth.bits_to_torch(xb).to(DEV)
    Xt = X.t().contiguous()                        # [K][M]
    q1, b1 = fireq.quantize_act(X)
    q2, b2 = fireq.quantize_act_t(Xt, M, K)
    rq, rb = oq.quantize_act(synth.bits_to_f64(xb))
    assert torch.equal(q1, q2) and torch.equal(b1, b2)
    assert np.array_equal(q2.cpu().numpy(), rq) and np.array_equal(bits_of(b2), nm.bf16_to_bits(rb))


@pytest.mark.parametrize("M,K,packed", [(16, 11008, False), (5, 256, False), (200, 1408, False),
                                        (1200, 11008, True), (90, 12288, True)])
def test_silu_mul_quantize(fireq, M, K, packed):
    """packed: G and U are the two halves of one [M, 2K] gate_up output (ld = 2K), the prefill
    layout; M > 64 runs the persistent TMA-ring kernel."""
    gb = synth.activations(M, K, 41)
    ub = synth.activations(M, K, 42)
    G, U = synth.bits_to_torch(gb).to(DEV), synth.bits_to_torch(ub).to(DEV)
    if packed:
        GU = torch.cat([G, U], dim=1)
        G, U = GU[:, :K], GU[:, K:]
    q1, b1 = fireq.silu_mul_quantize_act(G, U)
    q2, b2 = fireq.silu_mul_quantize_act_t(G.t().contiguous(), U.t().contiguous(), M, K)
    assert torch.equal(q1, q2) and torch.equal(b1, b2)          # layouts agree bit-exactly
    # vs the oracle: h = bf16(silu(g) u) in fp64; SiLU's exp is not correctly rounded on
    # either side, so compare the dequantized codes within FP8 precision (2^-4 relative)
    h = of.silu_mul(synth.bits_to_f64(gb), synth.bits_to_f64(ub))
    rq, rb = oq.quantize_act(h)
    deq = nm.e4m3_decode(q1.cpu().numpy()) * synth.bits_to_f64(bits_of(b1))[:, None]
    ref = nm.e4m3_decode(rq) * rb[:, None]
    assert np.allclose(synth.bits_to_f64(bits_of(b1)), rb, rtol=2 ** -7)
    err = np.abs(deq - ref) / np.maximum(np.abs(ref), 2 ** -6 * rb[:, None])
    assert err.max() <= 2 ** -3 and np.mean(q1.cpu().numpy() == rq) > 0.99


def test_ffn_decode_vs_oracle(fireq):
    """One Llama2-7B-shaped FFN at M = 16 (reduced d_ff for oracle time) through the CUDA path."""
    M, d, dff = 16, 1024, 2816
    wg = synth.weights(dff, d, 51)
    wu = synth.weights(dff, d, 52)
    wd = synth.weights(d, dff, 53)
    xb = synth.activations(M, d, 54)
    Wgu = np.concatenate([wg, wu], axis=0)
    qgu = fireq.quantize_weight(synth.bits_to_torch(Wgu).to(DEV), 1)
    qd = fireq.quantize_weight(synth.bits_to_torch(wd).to(DEV), 1)
    gamma = torch.cat([torch.ones(dff, device=DEV), qd.c.float()])
    xq, beta = fireq.quantize_act(synth.bits_to_torch(xb).to(DEV), chan_mul=qgu.c)
    gu = fireq.w4a8_gemm(xq, beta, qgu.packed, qgu.scales, 2 * dff, qgu.n, gamma=gamma)
    hq, hb = fireq.silu_mul_quantize_act(gu[:, :dff], gu[:, dff:])
    y = fireq.w4a8_gemm(hq, hb, qd.packed, qd.scales, d, qd.n)
    torch.cuda.synchronize()
    ref_gu = oq.quantize_weight(synth.bits_to_f64(Wgu), 1)
    ref_d = oq.quantize_weight(synth.bits_to_f64(wd), 1)
    yb, r = of.ffn_reference(synth.bits_to_f64(xb), ref_gu, ref_d, dff)
    err = og.g4_error(y.float().cpu().numpy().astype(np.float64), r)
    # two chained quantized layers: the GPU's bf16 gate/up outputs may differ from the
    # oracle's by one bf16 ulp (FP32 vs fp64 accumulation), which can move a few h codes
    # by one FP8 step; the bound is 2x the single-layer G4 tolerance.
    assert err <= 2e-2, err
    assert og.rel_frobenius(y.float().cpu().numpy(), r) < 5e-3


# ------------------------------------------------------------ fused decode FFN
def _ffn_case(fireq, M, d, dff, seed):
    wg = synth.weights(dff, d, seed)
    wu = synth.weights(dff, d, seed + 1)
    wd = synth.weights(d, dff, seed + 2)
    xb = synth.activations(M, d, seed + 3)
    Wg, Wu = synth.bits_to_torch(wg).to(DEV), synth.bits_to_torch(wu).to(DEV)
    Wgu = torch.cat([Wg, Wu])
    qgu = fireq.quantize_weight(Wgu, 1)
    qd = fireq.quantize_weight(synth.bits_to_torch(wd).to(DEV), 1)
    Wil = fireq.interleave_gate_up(Wg, Wu)
    qil = fireq.quantize_weight(Wil, 1)
    x = synth.bits_to_torch(xb).to(DEV)
    return wg, wu, wd, xb, Wgu, Wil, qgu, qil, qd, x


def _unfused(fireq, x, qgu, qd, dff):
    d = x.shape[1]
    gamma = torch.cat([torch.ones(dff, device=DEV), qd.c.float()])
    xq, beta = fireq.quantize_act(x, chan_mul=qgu.c)
    gu = fireq.w4a8_gemm(xq, beta, qgu.packed, qgu.scales, 2 * dff, qgu.n, gamma=gamma)
    hq, hb = fireq.silu_mul_quantize_act(gu[:, :dff], gu[:, dff:])
    y = fireq.w4a8_gemm(hq, hb, qd.packed, qd.scales, d, qd.n)
    return hq, hb, y


def test_interleave_gate_up_is_a_row_permutation(fireq):
    d, dff = 256, 384
    _, _, _, _, Wgu, Wil, qgu, qil, _, _ = _ffn_case(fireq, 1, d, dff, 61)
    n = np.arange(2 * dff)
    t, r = n // 128, n % 128
    src = np.where(r < 64, t * 64 + r, dff + t * 64 + r - 64)
    assert torch.equal(Wil.cpu(), Wgu.cpu()[torch.from_numpy(src)])
    # CAS lambda is per input channel and PTS per tensor: unchanged by the permutation
    assert qil.n == qgu.n and torch.equal(qil.c, qgu.c)


def _check_fused(fireq, M, d, dff, seed, reps=3, residual=True):
    """The fused FFN against its pieces.  Exact: y equals the standalone down GEMM on
    quantize_act(h) (the in-kernel A2..A3 of h is bit for bit fireq_quantize_act's; the
    caller's environment makes the standalone GEMM take the fused path's down plan), and
    repeated calls agree (workspace reset).  Against the unfused 4-kernel chain: G4."""
    *_, qgu, qil, qd, x = _ffn_case(fireq, M, d, dff, seed)
    hq, hb, y_ref = _unfused(fireq, x, qgu, qd, dff)
    ws = fireq.Workspace(fireq.ffn_workspace_bytes(M, d, dff))
    h = torch.empty((M, dff), dtype=torch.bfloat16, device=DEV)
    ys = [fireq.ffn_w4a8_decode(x, qil, qd, h=h, workspace=ws) for _ in range(reps)]
    hq2, hb2 = fireq.quantize_act(h)
    y2 = fireq.w4a8_gemm(hq2, hb2, qd.packed, qd.scales, d, qd.n)
    # the FFN block with its residual connection: y + x in the down GEMM's epilogue
    if residual:
        yr = fireq.ffn_w4a8_decode(x, qil, qd, h=h, workspace=ws, residual=x)
        yr2 = fireq.w4a8_gemm(hq2, hb2, qd.packed, qd.scales, d, qd.n, residual=x)
    torch.cuda.synchronize()
    assert all(torch.equal(v, ys[0]) for v in ys)
    assert torch.equal(ys[0], y2), (ys[0].float() - y2.float()).abs().max().item()
    if residual:
        assert torch.equal(yr, yr2)
    # h of the interleaved gate_up vs the plain one: same up to the fp32 summation order of
    # split tiles (the two paths schedule gate_up differently)
    assert torch.allclose(hb2.float(), hb.float(), rtol=2 ** -7, atol=0)
    assert (hq2 == hq).float().mean().item() > 0.995
    yv, rv = ys[0].float().cpu().numpy().astype(np.float64), y_ref.float().cpu().numpy().astype(np.float64)
    assert og.g4_error(yv, rv) <= 1e-2 and og.rel_frobenius(yv, rv) < 2e-3


def _isolated(call, env):
    """Run `call` (source using F = fireq, T = this module) in a fresh process with `env`
    added: the library reads its FIREQ_* switches once per process."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "from paper_2505_20839_b200 import fireq as F; F.load()\n"
            "import test_gpu_ffn as T\n%s\nprint('ok')\n") % (root, os.path.join(root, "tests"), call)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


FUSED_CASES = [(16, 1024, 2816), (5, 512, 384), (1, 256, 128), (11, 768, 1280), (16, 4096, 11008),
               (200, 512, 768), (1024, 1024, 2816)]             # prefill-sized M: 192/224-token tiles


@pytest.mark.parametrize("M,d,dff", FUSED_CASES)
def test_fused_ffn_default(fireq, M, d, dff):
    """Default fireq_ffn_w4a8_decode: quantize_act(x); gate_up whose epilogue forms h; quantize_act(h);
    down with the standalone GEMM's own plan (cluster split-K at decode) and the residual in its
    epilogue -- y equals fireq_w4a8_gemm[_residual](quantize_act(h)) bit for bit.  (4096 x 11008:
    Llama2-7B, 8 back-to-back calls.)"""
    _check_fused(fireq, M, d, dff, 71 + M, reps=8 if d == 4096 else (1 if M > 16 else 3))


@pytest.mark.parametrize("M,d,dff", [(16, 1024, 2816), (16, 4096, 11008)])
def test_fused_ffn_tail_quant_mode(M, d, dff):
    """FIREQ_FFN_MODE=3: the gate_up kernel quantizes h in its tail (grid barrier, max|h| by
    atomics); same bit-exact checks."""
    _isolated("T._check_fused(F, %d, %d, %d, %d)" % (M, d, dff, 271 + M), {"FIREQ_FFN_MODE": "3"})


@pytest.mark.parametrize("M,d,dff", [(16, 1024, 2816), (5, 512, 384), (16, 4096, 11008)])
def test_fused_ffn_single_launch(M, d, dff):
    """FIREQ_FFN_PERSISTENT=1: ONE persistent launch (x quantized in-kernel behind a grid
    barrier, gate_up + SwiGLU, grid barrier, h quantized in 1/C slices, grid barrier, down by
    stream-K).  FIREQ_NO_CSPLIT=1 gives the standalone down GEMM the same stream-K plan, so y
    must match it bit for bit.  (1024 x 2816: gate_up is pure stream-K, 44 tiles < 148 CTAs: a
    tile owner whose split tile is its last phase-0 segment must not stage partials through
    the weight ring, which already streams phase-1 weights.)"""
    _isolated("T._check_fused(F, %d, %d, %d, %d, reps=%d, residual=False)" % (M, d, dff, 171 + M, 8 if d == 4096 else 3),
              {"FIREQ_NO_CSPLIT": "1", "FIREQ_FFN_PERSISTENT": "1"})


@pytest.mark.parametrize("with_residual,M", [(False, 16), (True, 16), (True, 300)])
def test_fused_ffn_vs_oracle(fireq, with_residual, M):
    d, dff = 1024, 2816
    wg, wu, wd, xb, *_, qil, qd, x = _ffn_case(fireq, M, d, dff, 81)
    y = fireq.ffn_w4a8_decode(x, qil, qd, workspace=fireq.Workspace(fireq.ffn_workspace_bytes(M, d, dff)),
                              residual=x if with_residual else None)
    torch.cuda.synchronize()
    ref_gu = oq.quantize_weight(synth.bits_to_f64(np.concatenate([wg, wu], axis=0)), 1)
    ref_d = oq.quantize_weight(synth.bits_to_f64(wd), 1)
    _, r = of.ffn_reference(synth.bits_to_f64(xb), ref_gu, ref_d, dff,
                            residual=synth.bits_to_f64(xb) if with_residual else None)
    yv = y.float().cpu().numpy().astype(np.float64)
    assert og.g4_error(yv, r) <= 2e-2                        # same bound as the unfused chain
    assert og.rel_frobenius(yv, r) < 5e-3


def test_fused_ffn_headline_size_vs_oracle(fireq):
    """The bench's headline step at its full size (Llama2-7B FFN, batch 16: d = 4096,
    d_ff = 11008) through fireq_ffn_w4a8_decode, every output against the oracle's FFN
    (same bound as the chain)."""
    M, d, dff = 16, 4096, 11008
    wg, wu, wd, xb, *_, qil, qd, x = _ffn_case(fireq, M, d, dff, 91)
    y = fireq.ffn_w4a8_decode(x, qil, qd, workspace=fireq.Workspace(fireq.ffn_workspace_bytes(M, d, dff)))
    torch.cuda.synchronize()
    ref_gu = oq.quantize_weight(synth.bits_to_f64(np.concatenate([wg, wu], axis=0)), 1)
    ref_d = oq.quantize_weight(synth.bits_to_f64(wd), 1)
    _, r = of.ffn_reference(synth.bits_to_f64(xb), ref_gu, ref_d, dff)
    yv = y.float().cpu().numpy().astype(np.float64)
    assert og.g4_error(yv, r) <= 2e-2
    assert og.rel_frobenius(yv, r) < 5e-3


def test_fused_ffn_prefill_size_sampled_vs_oracle(fireq):
    """The prefill FFN block at the bench's size (16 x 1024 tokens, d = 4096, d_ff = 11008:
    224-token tiles, the row-ring quantizers) against the oracle on sampled token rows (every
    step of the FFN is row-independent, so the oracle runs on those rows only)."""
    M, d, dff = 16384, 4096, 11008
    wg, wu, wd, xb, *_, qil, qd, x = _ffn_case(fireq, M, d, dff, 93)
    y = fireq.ffn_w4a8_decode(x, qil, qd, workspace=fireq.Workspace(fireq.ffn_workspace_bytes(M, d, dff)),
                              residual=x)
    torch.cuda.synchronize()
    rows = np.array([0, 1, 223, 224, 5000, 8191, 12345, 16383])
    ref_gu = oq.quantize_weight(synth.bits_to_f64(np.concatenate([wg, wu], axis=0)), 1)
    ref_d = oq.quantize_weight(synth.bits_to_f64(wd), 1)
    xs = synth.bits_to_f64(xb[rows])
    _, r = of.ffn_reference(xs, ref_gu, ref_d, dff, residual=xs)
    yv = y[torch.from_numpy(rows).to(DEV)].float().cpu().numpy().astype(np.float64)
    assert og.g4_error(yv, r) <= 2e-2
    assert og.rel_frobenius(yv, r) < 5e-3


@pytest.mark.gpu
def test_silu_ftz_form_is_bitwise_the_reference_form(tmp_path):
    """The kernels' SiLU (ex2.approx.ftz / rcp.approx.ftz, paired bf16 rounding) must equal
    bf16(__fdividef(g, 1 + __expf(-g)) * u) bit for bit: every bf16 g x 4096 bf16 u
    (scripts/silu_ftz_identity.cu, compiled and run here)."""
    import os
    import shutil
    import subprocess
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    src = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts", "silu_ftz_identity.cu")
    exe = str(tmp_path / "silu_id")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe, src], check=True,
                   capture_output=True, timeout=300)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and " 0 mismatches" in out.stdout, out.stdout + out.stderr
