"""One quantize_act(c) and one silu_mul_quantize_act launch at M (default 16384) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_20839_b200 import fireq as F
F.load()
M = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
gu = synth.bits_to_torch(synth.activations(M, 22016, 3)).cuda()
x = synth.bits_to_torch(synth.activations(M, 4096, 4)).cuda()
c = torch.ones(4096, dtype=torch.bfloat16, device="cuda")
for _ in range(2):
    F.quantize_act(x, chan_mul=c)
    F.silu_mul_quantize_act(gu[:, :11008], gu[:, 11008:])
torch.cuda.synchronize()
