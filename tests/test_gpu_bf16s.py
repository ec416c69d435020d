"""sigma_BF16 comparison variant (DESIGN reading R25): the BF16-scale weight
quantizer bit-exact against oracle/quant.py::quantize_weight_bf16s, and the per-group scaled
GEMM (fireq_w4a8_gemm_bf16s) within G4 of oracle/gemm.py::gemm_reference_bf16s."""
import numpy as np
import pytest
import torch

import synth
from oracle import gemm as og
from oracle import numerics as nm
from oracle import quant as oq

pytestmark = pytest.mark.gpu

G4_TOL = 1e-2
DEV = "cuda"


def bits_of(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def check_weight_bf16s(fireq, wb, cas):
    qw = fireq.quantize_weight_bf16s(synth.bits_to_torch(wb).to(DEV), cas_mode=cas)
    torch.cuda.synchronize()
    ref = oq.quantize_weight_bf16s(synth.bits_to_f64(wb), cas)
    ps = qw.pts_and_status.cpu().numpy()
    assert ps[1] == 0 and ps[0] == ref.n
    assert np.array_equal(bits_of(qw.c), nm.bf16_to_bits(ref.c))
    assert np.array_equal(bits_of(qw.scales), ref.scales16)
    assert np.array_equal(qw.packed.cpu().numpy(), ref.packed)
    return qw, ref


@pytest.mark.parametrize("N,K,cas", [(128, 128, 0), (256, 512, 1), (384, 1280, 1), (1024, 4096, 0)])
def test_quantize_weight_bf16s(fireq, N, K, cas):
    check_weight_bf16s(fireq, synth.weights(N, K, synth.layer_seed(11, N + K)), cas)


def test_quantize_weight_bf16s_edges(fireq):
    """Zero groups (sigma = 0), a group whose max is exactly 7 x a bf16 value, and tiny values
    that move the PTS exponent."""
    rng = np.random.default_rng(91)
    W = nm.bf16_rn(rng.standard_normal((256, 384)) * 0.02)
    W[4, 128:256] = 0.0
    W[9, 0] = 7 * 0.0390625
    W[9, 1:128] = np.clip(W[9, 1:128], -0.25, 0.25)
    W[200, 256:384] = nm.bf16_rn(W[200, 256:384] * 2.0 ** -12)
    W = nm.bf16_rn(W)
    for cas in (0, 1):
        check_weight_bf16s(fireq, nm.bf16_to_bits(W), cas)


@pytest.mark.parametrize("M,N,K", [
    (1, 128, 128), (7, 256, 512), (16, 512, 1024), (17, 384, 640), (32, 256, 2048), (64, 384, 2048),
    (300, 256, 512), (16, 4096, 4096),
])
def test_gemm_bf16s_g4(fireq, M, N, K):
    seed = M * 17 + N + K
    wb = synth.weights(N, K, synth.layer_seed(12, seed))
    xb = synth.activations(M, K, synth.layer_seed(13, seed))
    qw, ref = check_weight_bf16s(fireq, wb, 1)
    xq, beta = fireq.quantize_act(synth.bits_to_torch(xb).to(DEV), chan_mul=qw.c)
    Y = fireq.w4a8_gemm_bf16s(xq, beta, qw.packed, qw.scales, N, qw.n)
    torch.cuda.synchronize()
    rq, rbeta = oq.quantize_act(synth.bits_to_f64(xb), ref.c)
    assert np.array_equal(xq.cpu().numpy(), rq)
    r = og.gemm_reference_bf16s(rq, rbeta, ref.codes, ref.sigma, ref.n)
    y = Y.float().cpu().numpy().astype(np.float64)
    err = og.g4_error(y, r)
    assert err <= G4_TOL, f"G4 {err}"
    assert og.rel_frobenius(y, r) < 5e-3


def test_gemm_bf16s_deterministic(fireq):
    M, N, K = 16, 1024, 4096
    wb = synth.weights(N, K, 5)
    qw = fireq.quantize_weight_bf16s(synth.bits_to_torch(wb).to(DEV), cas_mode=1)
    xq, beta = fireq.quantize_act(synth.bits_to_torch(synth.activations(M, K, 6)).to(DEV), chan_mul=qw.c)
    a = fireq.w4a8_gemm_bf16s(xq, beta, qw.packed, qw.scales, N, qw.n)
    b = fireq.w4a8_gemm_bf16s(xq, beta, qw.packed, qw.scales, N, qw.n)
    assert torch.equal(a, b)



@pytest.mark.parametrize("M,N,K", [(16, 22016, 4096), (16, 4096, 11008), (4096, 22016, 4096)])
def test_gemm_bf16s_timed_shapes_sampled(fireq, M, N, K):
    """The shapes scripts/time_bf16s.py times (the Llama2-7B FFN GEMMs at decode and prefill):
    the weight quantizer bit-exact, the GEMM within G4 on sampled token rows (rows are
    independent, so the oracle runs on those rows only)."""
    seed = M + N + K
    wb = synth.weights(N, K, synth.layer_seed(14, seed))
    xb = synth.activations(M, K, synth.layer_seed(15, seed))
    qw, ref = check_weight_bf16s(fireq, wb, 1)
    xq, beta = fireq.quantize_act(synth.bits_to_torch(xb).to(DEV), chan_mul=qw.c)
    Y = fireq.w4a8_gemm_bf16s(xq, beta, qw.packed, qw.scales, N, qw.n)
    torch.cuda.synchronize()
    rows = np.unique(np.array([0, 1, M // 2, M - 1, min(M - 1, 127), min(M - 1, 128)]))
    rq, rbeta = oq.quantize_act(synth.bits_to_f64(xb[rows]), ref.c)
    assert np.array_equal(xq[torch.from_numpy(rows).to(DEV)].cpu().numpy(), rq)
    r = og.gemm_reference_bf16s(rq, rbeta, ref.codes, ref.sigma, ref.n)
    y = Y[torch.from_numpy(rows).to(DEV)].float().cpu().numpy().astype(np.float64)
    assert og.g4_error(y, r) <= G4_TOL
    assert og.rel_frobenius(y, r) < 5e-3
