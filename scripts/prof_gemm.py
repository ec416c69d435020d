"""Run one fireq_w4a8_gemm configuration a few times (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2505_20839_b200 import fireq as F

M, N, K = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
F.load()
W = synth.bits_to_torch(synth.weights(N, K, 1)).cuda()
X = synth.bits_to_torch(synth.activations(M, K, 2)).cuda()
qw = F.quantize_weight(W, 1)
xq, beta = F.quantize_act(X, chan_mul=qw.c)
ws = F.Workspace(F.gemm_workspace_bytes(M, N, K))
out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
n = qw.n
print(F.gemm_plan(M, N, K))
for _ in range(reps):
    F.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, n, out=out, workspace=ws)
torch.cuda.synchronize()
