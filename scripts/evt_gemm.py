"""Per-stage event log of CTA 0 (profile build): where does a pipeline stage spend time?
ROT=r cycles r weight copies (r x 46 MB > L2 for the HBM-resident case; ROT=1: L2-resident)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2505_20839_b200 import fireq as F
F.load(os.path.join(os.path.dirname(F.LIB_PATH), 'libfireq_prof.so'))
M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (16, 22016, 4096)
ROT = int(os.environ.get("ROT", "4"))
W = synth.bits_to_torch(synth.weights(N, K, 1)).cuda(); X = synth.bits_to_torch(synth.activations(M, K, 2)).cuda()
qw = F.quantize_weight(W, 1); xq, beta = F.quantize_act(X, chan_mul=qw.c)
rot = [(qw.packed.clone(), qw.scales.clone()) for _ in range(ROT)]
ws = F.Workspace(F.gemm_workspace_bytes(M, N, K)); out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
plan = F.gemm_plan(M, N, K); C = plan["ctas"]
tr = torch.zeros(C * 16 + 64 * 8 + 512 + C * 16, dtype=torch.int64, device="cuda")
for it in range(2 * ROT + 1):
    p, s = rot[it % ROT]
    F.debug_set_trace(tr if it == 2 * ROT else None)
    F.w4a8_gemm(xq, beta, p, s, N, qw.n, out=out, workspace=ws)
torch.cuda.synchronize()
F.debug_set_trace(None)
ev = tr.cpu().numpy()[C * 16:C * 16 + 512].reshape(64, 8).astype(np.int64)
t0 = ev[0, 0]
names = ["prodW", "conv_fullW", "conv_Aok", "conv_arrive", "mma_afull", "mma_fullX", "mma_issued"]
print(f"M={M} N={N} K={K} ROT={ROT} plan={plan} (cycles from CTA 0's first weight issue)")
print("stage " + " ".join(f"{n:>11s}" for n in names))
for i in range(64):
    if ev[i, 0] == 0 and ev[i, 6] == 0: break
    print(f"{i:5d} " + " ".join(f"{(ev[i, j] - t0) if ev[i, j] else -1:11d}" for j in range(7)))
