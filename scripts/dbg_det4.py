"""Synced repeated gate_up GEMMs: how many results differ from the most common one?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_20839_b200 import fireq as F
F.load()
DEV = "cuda"
M, d, dff = 16, 4096, 11008
N = int(os.environ.get("DBG_N", 2 * dff))
Wgu = synth.bits_to_torch(synth.weights(N, d, 91)).to(DEV)
qgu = F.quantize_weight(Wgu, 1)
x = synth.bits_to_torch(synth.activations(M, d, 94)).to(DEV)
gamma = torch.rand(N, device=DEV) + 0.5
xq, beta = F.quantize_act(x, chan_mul=qgu.c)
torch.cuda.synchronize()
outs = []
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 200):
    outs.append(F.w4a8_gemm(xq, beta, qgu.packed, qgu.scales, N, qgu.n, gamma=gamma))
    torch.cuda.synchronize()
ref = outs[len(outs) // 2]
cnt = sum(torch.equal(o, ref) for o in outs)
tiles = {}
for o in outs:
    if not torch.equal(o, ref):
        dz = (o.float() - ref.float()).abs().nonzero()
        for t in set((dz[:, 1] // 128).tolist()):
            tiles[t] = tiles.get(t, 0) + 1
print(f"cfg={os.environ.get('FIREQ_CFG16', '0')} N={N}: {len(outs) - cnt} of {len(outs)} differ from the middle result; tiles {sorted(tiles.items())[:10]}")
