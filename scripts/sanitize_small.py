"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): weight + activation quantizers, the GEMM under each schedule (whole tiles,
stream-K, cluster split-K, DSMEM reduce-scatter split-K, Y^T, gamma, residual), the SwiGLU
quantizer, the fused FFN block, the sigma_BF16 variant, the KV4 cache quantizer and the KV4Q8
attention.  Prints one line per case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2505_20839_b200 import fireq as F

F.load()
dev = "cuda"


def gemm_case(M, N, K, **kw):
    W = synth.bits_to_torch(synth.weights(N, K, 1)).to(dev)
    X = synth.bits_to_torch(synth.activations(M, K, 2)).to(dev)
    qw = F.quantize_weight(W, 1)
    xq, beta = F.quantize_act(X, chan_mul=qw.c)
    y = F.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, **kw)
    torch.cuda.synchronize()
    print(f"gemm M={M} N={N} K={K} plan={F.gemm_plan(M, N, K)} {kw and list(kw)} ok", flush=True)
    return y


gemm_case(16, 1024, 1024)                       # cluster split-K
gemm_case(16, 150 * 128, 512)                   # stream-K hybrid
gemm_case(7, 256, 512, out_layout=1)            # Y^T
gemm_case(64, 512, 1024)                        # DSMEM reduce-scatter split-K
gemm_case(128, 256, 768, gamma=torch.ones(256, device=dev))
gemm_case(300, 256, 384)                        # 192-token tiles, reduce-scatter
gemm_case(1024, 4096, 512)                      # 224-token tiles, stream-K
gemm_case(2100, 256, 512, out_layout=1)
h = synth.bits_to_torch(synth.activations(20, 2 * 1408, 3)).to(dev)
hq, hb = F.silu_mul_quantize_act(h[:, :1408].contiguous(), h[:, 1408:].contiguous())
torch.cuda.synchronize()
print("silu_mul_quantize_act ok", flush=True)
W16 = synth.bits_to_torch(synth.weights(512, 1024, 4)).to(dev)
q16 = F.quantize_weight_bf16s(W16, 1)
xq, beta = F.quantize_act(synth.bits_to_torch(synth.activations(16, 1024, 5)).to(dev), chan_mul=q16.c)
F.w4a8_gemm_bf16s(xq, beta, q16.packed, q16.scales, 512, q16.n)
torch.cuda.synchronize()
print("sigma_BF16 quantizer + GEMM ok", flush=True)
# residual epilogue (decode prefetch path and a prefill-sized tile), in place
R = synth.bits_to_torch(synth.activations(16, 1024, 6)).to(dev)
gemm_case(16, 1024, 1024, residual=R)
R2 = synth.bits_to_torch(synth.activations(300, 256, 7)).to(dev)
gemm_case(300, 256, 384, residual=R2, out=R2)
# fused FFN block (decode and a prefill-sized M, with the residual)
Wg = synth.bits_to_torch(synth.weights(384, 512, 8)).to(dev)
Wu = synth.bits_to_torch(synth.weights(384, 512, 9)).to(dev)
Wd = synth.bits_to_torch(synth.weights(512, 384, 10)).to(dev)
qil = F.quantize_weight(F.interleave_gate_up(Wg, Wu), 1)
qd = F.quantize_weight(Wd, 1)
for M in (5, 200):
    x = synth.bits_to_torch(synth.activations(M, 512, 11)).to(dev)
    F.ffn_w4a8_decode(x, qil, qd, residual=x)
    torch.cuda.synchronize()
    print(f"fused FFN M={M} ok", flush=True)
# KV4 cache + KV4Q8 attention (GQA, causal and not)
B, N, Hq, Hkv = 1, 256, 2, 1
qb, kb, vb = synth.attention(B, N, Hq, Hkv, 12)
Q, K, V = (synth.bits_to_torch(a).to(dev) for a in (qb, kb, vb))
cache = F.KVCache(K, V)
xq, beta = F.quantize_act(Q.reshape(B * Hq * N, 128))
for causal in (True, False):
    F.kv4q8_attention(xq.reshape(B, Hq, N, 128), beta.reshape(B, Hq, N), cache, Hq, causal=causal)
    torch.cuda.synchronize()
    print(f"kv4q8 attention causal={causal} ok", flush=True)
print("SANITIZE DRIVER DONE")
