import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch, synth
from paper_2505_20839_b200 import fireq
fireq.load()
import test_gpu_ffn as T
DEV = "cuda"
M, d, dff = 16, 4096, 11008
*_, qgu, qil, qd, x = T._ffn_case(fireq, M, d, dff, 91)
hq, hb, y_ref = T._unfused(fireq, x, qgu, qd, dff)
if len(sys.argv) > 1:
    torch.cuda.synchronize()
    print("unfused hb*448", (hb.float() * 448).cpu().numpy()[8:11])
ws = fireq.Workspace(fireq.ffn_workspace_bytes(M, d, dff))
h = torch.empty((M, dff), dtype=torch.bfloat16, device=DEV)
y = fireq.ffn_w4a8_decode(x, qil, qd, h=h, workspace=ws)
torch.cuda.synchronize()
print("unfused hb*448 after fused", (hb.float() * 448).cpu().numpy()[8:11])
hq2, hb2 = fireq.quantize_act(h)
torch.cuda.synchronize()
print("fused hb2*448", (hb2.float() * 448).cpu().numpy()[8:11])
print("h amax", h.float().abs().max(1).values.cpu().numpy()[8:11])
