import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch, synth
from paper_2505_20839_b200 import fireq as F
F.load()
import test_gpu_ffn as T
M, d, dff = 16, 4096, 11008
*_, qgu, qil, qd, x = T._ffn_case(F, M, d, dff, 91)
gamma = torch.cat([torch.ones(dff, device="cuda"), qd.c.float()])
xq, beta = F.quantize_act(x, chan_mul=qgu.c)
gu = F.w4a8_gemm(xq, beta, qgu.packed, qgu.scales, 2 * dff, qgu.n, gamma=gamma)
hq, hb = F.silu_mul_quantize_act(gu[:, :dff], gu[:, dff:])
torch.cuda.synchronize()
print("A", (hb.float() * 448).cpu().numpy()[8:11])
y = F.w4a8_gemm(hq, hb, qd.packed, qd.scales, d, qd.n)
torch.cuda.synchronize()
print("B", (hb.float() * 448).cpu().numpy()[8:11])
hq, hb, y_ref = T._unfused(F, x, qgu, qd, dff)
torch.cuda.synchronize()
print("C", (hb.float() * 448).cpu().numpy()[8:11])
g, u = gu[:, :dff].float(), gu[:, dff:].float()
h_ref = (g / (1 + torch.exp(-g)) * u).to(torch.bfloat16).float()
print("torch amax", h_ref.abs().max(1).values.cpu().numpy()[8:11])
