"""Determinism of the stream-K gate_up GEMM (M=16, N=22016, K=4096) and of the silu kernel."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2505_20839_b200 import fireq as F
F.load()
DEV = "cuda"
M, d, dff = 16, 4096, 11008
seed = 91
wg = synth.weights(dff, d, seed); wu = synth.weights(dff, d, seed + 1)
xb = synth.activations(M, d, seed + 3)
Wg, Wu = synth.bits_to_torch(wg).to(DEV), synth.bits_to_torch(wu).to(DEV)
qgu = F.quantize_weight(torch.cat([Wg, Wu]), 1)
x = synth.bits_to_torch(xb).to(DEV)
xq, beta = F.quantize_act(x, chan_mul=qgu.c)
outs = []
for it in range(20):
    gu = F.w4a8_gemm(xq, beta, qgu.packed, qgu.scales, 2 * dff, qgu.n)
    outs.append(gu.clone())
torch.cuda.synchronize()
for it in range(1, 20):
    d_ = (outs[it].float() - outs[0].float()).abs()
    if d_.max().item() > 0:
        idx = d_.nonzero().cpu().numpy()
        print("run", it, "differs at", len(idx), "elements; tiles", np.unique(idx[:, 1] // 128)[:20], "tokens", np.unique(idx[:, 0]))
print("done")
