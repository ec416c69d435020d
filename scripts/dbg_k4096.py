import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2505_20839_b200 import fireq as F
F.load()
M, (N, K) = 4096, synth.SHAPES["llama3-8b.k"]
W = synth.bits_to_torch(synth.weights(N, K, 1)).cuda(); X = synth.bits_to_torch(synth.activations(M, K, 2)).cuda()
qw = F.quantize_weight(W, 1); xq, beta = F.quantize_act(X, chan_mul=qw.c)
print(F.gemm_plan(M, N, K), flush=True)
for i in range(3):
    torch.cuda.synchronize(); t = time.time()
    Y = F.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n)
    torch.cuda.synchronize(); print(f"gemm {1e6*(time.time()-t):.0f} us", flush=True)
