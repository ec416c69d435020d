"""Compare the fused FFN's h with the unfused chain's (torch silu on the GEMM's bf16 g, u)."""
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
g, u = gu[:, :dff].float(), gu[:, dff:].float()
h_ref = (g / (1 + torch.exp(-g)) * u).to(torch.bfloat16).float()
ws = F.Workspace(F.ffn_workspace_bytes(M, d, dff))
h = torch.zeros((M, dff), dtype=torch.bfloat16, device=DEV)
y = F.ffn_w4a8_decode(x, qil, qd, h=h, workspace=ws)
torch.cuda.synchronize()
hf = h.float()
diff = (hf - h_ref).abs()
rel = diff / h_ref.abs().clamp_min(1e-3)
bad = (rel > 0.02).nonzero().cpu().numpy()
print("max rel", rel.max().item(), "n bad", len(bad))
tiles = bad[:, 1] // 64
print("bad tiles (interleaved) histogram:", np.unique(tiles, return_counts=True))
print("bad tokens:", np.unique(bad[:, 0], return_counts=True))
for m, j in bad[:10]:
    print(m, j, hf[m, j].item(), h_ref[m, j].item(), g[m, j].item(), u[m, j].item())
print("amax fused per token", hf.abs().max(1).values.cpu().numpy())
print("amax ref   per token", h_ref.abs().max(1).values.cpu().numpy())
hq, hb = F.silu_mul_quantize_act(gu[:, :dff], gu[:, dff:])
torch.cuda.synchronize()
print("silu kernel beta*448", (hb.float() * 448).cpu().numpy())
print("ref amax/448 -> bf16*448", ((h_ref.abs().max(1).values / 448).to(torch.bfloat16).float() * 448).cpu().numpy())
am = h_ref.abs()
j = am[9].argmax().item()
print("token 9 argmax channel", j, am[9, j].item())
# recompute with contiguous copies
hq2, hb2 = F.silu_mul_quantize_act(gu[:, :dff].contiguous(), gu[:, dff:].contiguous())
print("contiguous beta*448", (hb2.float() * 448).cpu().numpy())
