import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2505_20839_b200 import fireq as F
F.load()
DEV = "cuda"
M, d, dff = 16, 4096, 11008
wg = synth.weights(dff, d, 91); wu = synth.weights(dff, d, 92)
Wg, Wu = synth.bits_to_torch(wg).to(DEV), synth.bits_to_torch(wu).to(DEV)
qgu = F.quantize_weight(torch.cat([Wg, Wu]), 1)
x = synth.bits_to_torch(synth.activations(M, d, 94)).to(DEV)
gamma = torch.cat([torch.ones(dff, device=DEV), torch.rand(dff, device=DEV) + 0.5])
xq, beta = F.quantize_act(x, chan_mul=qgu.c)
for mode in ["gamma-sync", "gamma-nosync", "nogamma-nosync", "gamma-nosync-ws"]:
    outs = []
    ws = F.Workspace(F.gemm_workspace_bytes(M, 2 * dff, d))
    for it in range(30):
        g = gamma if mode.startswith("gamma") else None
        gu = F.w4a8_gemm(xq, beta, qgu.packed, qgu.scales, 2 * dff, qgu.n, gamma=g,
                         workspace=ws if mode.endswith("ws") else None)
        outs.append(gu)
        if "nosync" not in mode:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    nbad = [i for i in range(1, 30) if not torch.equal(outs[i], outs[0])]
    print(mode, "mismatch iterations vs first:", nbad[:20])
    if nbad:
        dz = (outs[nbad[0]].float() - outs[0].float()).abs().nonzero()
        print("   tiles", sorted(set((dz[:, 1] // 128).tolist()))[:20], "tokens", sorted(set(dz[:, 0].tolist())))
