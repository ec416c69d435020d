import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import synth
from paper_2505_20839_b200 import fireq as F
F.load()
for (M, N, K) in [(16, 1024, 4096), (16, 22016, 4096), (16, 4096, 11008)]:
    wb = synth.weights(N, K, 11); xb = synth.activations(M, K, 12)
    qw = F.quantize_weight(synth.bits_to_torch(wb).cuda())
    xq, beta = F.quantize_act(synth.bits_to_torch(xb).cuda(), chan_mul=qw.c)
    ws = F.Workspace(F.gemm_workspace_bytes(M, N, K))
    torch.cuda.synchronize()
    yref = F.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, workspace=ws); torch.cuda.synchronize()
    ys = [F.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, workspace=ws) for _ in range(4)]
    torch.cuda.synchronize()
    yref2 = F.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, workspace=ws); torch.cuda.synchronize()
    print(M, N, K, "ref==ref2", torch.equal(yref, yref2), [torch.equal(yref, y) for y in ys],
          "counters", int(ws.t[:4*(N//128)].view(torch.int32).abs().sum()))
    diff = (yref.float() - ys[0].float()).abs()
    bad = (diff > 0).any(dim=0).nonzero().flatten()
    print("  bad cols", bad.numel(), bad[:20].tolist())
