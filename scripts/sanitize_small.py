"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): weight + activation quantizers, the GEMM under each schedule (whole tiles,
stream-K, cluster split-K, DSMEM reduce-scatter split-K, Y^T, gamma), the SwiGLU quantizer,
the fused decode FFN and the sigma_BF16 variant.  Prints one line per case."""
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
print("SANITIZE DRIVER DONE")
