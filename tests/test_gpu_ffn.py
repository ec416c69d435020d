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


@pytest.mark.parametrize("M,K", [(16, 4096), (8, 11008), (3, 128)])
def test_quantize_act_transposed_bit_exact(fireq, M, K):
    xb = synth.activations(M, K, 31)
    X = synth.bits_to_torch(xb).to(DEV)
    Xt = X.t().contiguous()                        # [K][M]
    q1, b1 = fireq.quantize_act(X)
    q2, b2 = fireq.quantize_act_t(Xt, M, K)
    rq, rb = oq.quantize_act(synth.bits_to_f64(xb))
    assert torch.equal(q1, q2) and torch.equal(b1, b2)
    assert np.array_equal(q2.cpu().numpy(), rq) and np.array_equal(bits_of(b2), nm.bf16_to_bits(rb))


@pytest.mark.parametrize("M,K", [(16, 11008), (5, 256)])
def test_silu_mul_quantize(fireq, M, K):
    gb = synth.activations(M, K, 41)
    ub = synth.activations(M, K, 42)
    G, U = synth.bits_to_torch(gb).to(DEV), synth.bits_to_torch(ub).to(DEV)
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
