"""Llama2-7B FFN block at decode batch 16 through fireq_ffn_w4a8_decode, a few steps (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2505_20839_b200 import fireq as F
F.load()
ffn = bench.FusedFFN(F, 16, 2, torch.device("cuda"))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for i in range(4):
        ffn.step(i % 2, s)
torch.cuda.synchronize()
print("ok")
