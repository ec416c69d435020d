import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2505_20839_b200 import fireq as F
F.load()
DEV = "cuda"
M, d, dff = 16, 4096, 11008
seed = 91
wg = synth.weights(dff, d, seed); wu = synth.weights(dff, d, seed + 1); wd = synth.weights(d, dff, seed + 2)
xb = synth.activations(M, d, seed + 3)
Wg, Wu = synth.bits_to_torch(wg).to(DEV), synth.bits_to_torch(wu).to(DEV)
qgu = F.quantize_weight(torch.cat([Wg, Wu]), 1)
qd = F.quantize_weight(synth.bits_to_torch(wd).to(DEV), 1)
qil = F.quantize_weight(F.interleave_gate_up(Wg, Wu), 1)
x = synth.bits_to_torch(xb).to(DEV)
gamma = torch.cat([torch.ones(dff, device=DEV), qd.c.float()])
xq, beta = F.quantize_act(x, chan_mul=qgu.c)
gu = F.w4a8_gemm(xq, beta, qgu.packed, qgu.scales, 2 * dff, qgu.n, gamma=gamma)
hq, hb = F.silu_mul_quantize_act(gu[:, :dff], gu[:, dff:])
torch.cuda.synchronize()
hb_c, gu_c, hq_c = hb.clone(), gu.clone(), hq.clone()
print("silu beta*448 before fused", (hb.float() * 448).cpu().numpy())
ws = F.Workspace(F.ffn_workspace_bytes(M, d, dff))
h = torch.empty((M, dff), dtype=torch.bfloat16, device=DEV)
y = F.ffn_w4a8_decode(x, qil, qd, h=h, workspace=ws)
torch.cuda.synchronize()
print("hb changed by fused:", not torch.equal(hb, hb_c), " gu changed:", not torch.equal(gu, gu_c), "hq changed", not torch.equal(hq, hq_c))
hq3, hb3 = F.silu_mul_quantize_act(gu[:, :dff], gu[:, dff:])
print("silu beta*448 after", (hb3.float() * 448).cpu().numpy())
g, u = gu[:, :dff].float(), gu[:, dff:].float()
h_ref = (g / (1 + torch.exp(-g)) * u).to(torch.bfloat16).float()
print("torch amax", h_ref.abs().max(1).values.cpu().numpy())
