"""GPU parity of the KV4Q8 attention path (NEXT f4): fireq_quantize_kv bit-exact against the
oracle's K / V^T quantization, the query codes bit-exact, and fireq_kv4q8_attention's output
within G4 <= 1e-2 of the oracle's fp64 attention over the same codes (the FP8 softmax codes
are decided from an fp32 exp on the GPU and an fp64 exp in the oracle: a code flips only
where 448 P lies within ~2^-21 of an E4M3 midpoint, R37)."""
import numpy as np
import pytest
import torch

import synth
from oracle import attention as oa
from oracle import gemm as og
from oracle import numerics as nm

pytestmark = pytest.mark.gpu
DEV = "cuda"
D = 128
# The GPU forms 448 P = ex2(fp32 argument): relative to the oracle's fp64 exp its argument
# carries |x| 2^-24 of rounding (|x| < 2^8 here) and ex2.approx ~2^-22, so a P_hat code may
# round the other way where 448 P lies within 2^-15 (relative) of an E4M3 midpoint (R37).
AMB_DELTA = 2.0 ** -15


def g4_allowing_ambiguous_codes(y, r, amb):
    """G4 after subtracting, per element, the oracle's bound on what the ambiguous P_hat codes
    can change (oracle.attention.attention_head(..., amb_delta) -> dict["ambiguity"])."""
    rms = np.sqrt(np.mean(r * r, axis=1, keepdims=True))
    den = np.maximum(np.abs(r), 0.1 * rms)
    return float((np.maximum(np.abs(y - r) - amb, 0.0) / den).max())


def crs_calibration(K):
    """Offline CRS calibration from one sequence's keys of a kv head: the two channels
    with the largest max|k| are the outliers, beta = 1/4 (oracle/attention.py)."""
    top = np.argsort(-np.abs(K).max(axis=0))[:2]
    return nm.bf16_rn(oa.crs_scales(K, [int(c) % (D // 2) for c in top], beta=0.25))


def run(fireq, B, N, Hq, Hkv, causal, seed, crs=True):
    qb, kb, vb = synth.attention(B, N, Hq, Hkv, seed)
    Q, K, V = synth.bits_to_f64(qb), synth.bits_to_f64(kb), synth.bits_to_f64(vb)
    t = np.stack([crs_calibration(K[0, hk]) if crs else np.ones(D) for hk in range(Hkv)])
    lam = (np.float32(1.0) / t.astype(np.float32))
    Qt, Kt, Vt = (synth.bits_to_torch(x).to(DEV) for x in (qb, kb, vb))
    cache = fireq.KVCache(Kt, Vt, chan_lambda=torch.from_numpy(lam).to(DEV))
    q_fp8 = torch.empty((B, Hq, N, D), dtype=torch.uint8, device=DEV)
    q_scale = torch.empty((B, Hq, N), dtype=torch.bfloat16, device=DEV)
    c_t = synth.bits_to_torch(synth.to_bf16_bits(t)).to(DEV)
    g = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            fireq.quantize_act(Qt[b, h], chan_mul=c_t[h // g], out=(q_fp8[b, h], q_scale[b, h]))
    O = fireq.kv4q8_attention(q_fp8, q_scale, cache, Hq, causal=causal)
    torch.cuda.synchronize()
    return Q, K, V, t, cache, q_fp8, q_scale, O


@pytest.mark.parametrize("B,N,Hq,Hkv,causal", [(1, 256, 2, 1, True), (2, 384, 4, 2, True), (1, 256, 2, 2, False),
                                               (1, 1024, 4, 1, True), (1, 128, 1, 1, True)])
def test_kv4q8_attention_vs_oracle(fireq, B, N, Hq, Hkv, causal):
    Q, K, V, t, cache, q_fp8, q_scale, O = run(fireq, B, N, Hq, Hkv, causal, seed=1000 + N + Hq)
    g = Hq // Hkv
    Og = O.float().cpu().numpy().astype(np.float64)
    for b in range(B):
        for hk in range(Hkv):
            kv = oa.KV4Head(K[b, hk], V[b, hk], t=t[hk])
            x = b * Hkv + hk
            assert np.array_equal(cache.k_packed[x].cpu().numpy(), kv.k.packed)
            assert np.array_equal(cache.k_scales[x].cpu().numpy(), kv.k.scales)
            assert np.array_equal(cache.vt_packed[x].cpu().numpy(), kv.vt.packed)
            assert np.array_equal(cache.vt_scales[x].cpu().numpy(), kv.vt.scales)
            assert cache.k_pts[x, 0].item() == kv.k.n and cache.v_pts[x, 0].item() == kv.vt.n
            for h in range(hk * g, (hk + 1) * g):
                _, r, st = oa.attention_head(Q[b, h], kv, t=t[hk], causal=causal, amb_delta=AMB_DELTA)
                assert np.array_equal(q_fp8[b, h].cpu().numpy(), st["q_codes"])
                y = Og[b * N:(b + 1) * N, h * D:(h + 1) * D]
                e = g4_allowing_ambiguous_codes(y, r, st["ambiguity"])
                assert e <= 1e-2, (b, h, e)
                assert og.rel_frobenius(y, r) < 5e-3


def test_kv4q8_attention_bench_size_sampled(fireq):
    """The bench's attention workload (Llama3-8B prefill: 16 sequences x 1024 tokens, 32 query /
    8 kv heads, causal) in one launch; sampled (sequence, query head) pairs against the oracle."""
    B, N, Hq, Hkv = 16, 1024, 32, 8
    Q, K, V, t, cache, q_fp8, q_scale, O = run(fireq, B, N, Hq, Hkv, True, seed=4242)
    g = Hq // Hkv
    Og = O.float().cpu().numpy().astype(np.float64)
    for b, h in [(0, 0), (3, 9), (7, 13), (12, 22), (15, 31)]:
        hk = h // g
        kv = oa.KV4Head(K[b, hk], V[b, hk], t=t[hk])
        x = b * Hkv + hk
        assert np.array_equal(cache.k_packed[x].cpu().numpy(), kv.k.packed)
        assert np.array_equal(cache.vt_packed[x].cpu().numpy(), kv.vt.packed)
        _, r, st = oa.attention_head(Q[b, h], kv, t=t[hk], causal=True, amb_delta=AMB_DELTA)
        assert np.array_equal(q_fp8[b, h].cpu().numpy(), st["q_codes"])
        y = Og[b * N:(b + 1) * N, h * D:(h + 1) * D]
        assert g4_allowing_ambiguous_codes(y, r, st["ambiguity"]) <= 1e-2, (b, h, og.g4_error(y, r))
        assert og.rel_frobenius(y, r) < 5e-3


def test_kv4q8_attention_repeatable_and_head_layout(fireq):
    """Repeated launches are bit-identical; grouped-query heads sharing a kv head differ only by
    their queries (two q heads with identical queries give identical outputs)."""
    B, N, Hq, Hkv = 1, 256, 4, 2
    Q, K, V, t, cache, q_fp8, q_scale, O = run(fireq, B, N, Hq, Hkv, True, seed=77)
    O2 = fireq.kv4q8_attention(q_fp8, q_scale, cache, Hq)
    q_fp8[0, 1].copy_(q_fp8[0, 0])
    q_scale[0, 1].copy_(q_scale[0, 0])
    O3 = fireq.kv4q8_attention(q_fp8, q_scale, cache, Hq)
    torch.cuda.synchronize()
    assert torch.equal(O, O2)
    assert torch.equal(O3[:, 0:D], O3[:, D:2 * D])
