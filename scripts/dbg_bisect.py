"""Count wrong gate_up results in the unfused decode chain (no syncs) for a given libfireq build."""
import sys, os
os.environ["FIREQ_LOAD_PARTIAL"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_20839_b200 import fireq as F
F.load(sys.argv[1])
DEV = "cuda"
M, d, dff = 16, 4096, 11008
wg = synth.weights(dff, d, 91); wu = synth.weights(dff, d, 92); wd = synth.weights(d, dff, 93)
Wg, Wu = synth.bits_to_torch(wg).to(DEV), synth.bits_to_torch(wu).to(DEV)
qgu = F.quantize_weight(torch.cat([Wg, Wu]), 1)
qd = F.quantize_weight(synth.bits_to_torch(wd).to(DEV), 1)
x = synth.bits_to_torch(synth.activations(M, d, 94)).to(DEV)
gamma = torch.cat([torch.ones(dff, device=DEV), qd.c.float()])
S = torch.cuda.synchronize
xq, beta = F.quantize_act(x, chan_mul=qgu.c); S()
refs = []
for _ in range(3):
    refs.append(F.w4a8_gemm(xq, beta, qgu.packed, qgu.scales, 2 * dff, qgu.n, gamma=gamma)); S()
assert all(torch.equal(r, refs[0]) for r in refs)
ref = refs[0]
hq_r, hb_r = F.silu_mul_quantize_act(ref[:, :dff], ref[:, dff:]); S()
yref = F.w4a8_gemm(hq_r, hb_r, qd.packed, qd.scales, d, qd.n); S()
bad_gu, bad_y, tiles = 0, 0, {}
outs = []
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 150):
    xq, beta = F.quantize_act(x, chan_mul=qgu.c)
    gu = F.w4a8_gemm(xq, beta, qgu.packed, qgu.scales, 2 * dff, qgu.n, gamma=gamma)
    hq, hb = F.silu_mul_quantize_act(gu[:, :dff], gu[:, dff:])
    y = F.w4a8_gemm(hq, hb, qd.packed, qd.scales, d, qd.n)
    outs.append((gu, y))
S()
for gu, y in outs:
    if not torch.equal(gu, ref):
        bad_gu += 1
        dz = (gu.float() - ref.float()).abs().nonzero()
        for t in set((dz[:, 1] // 128).tolist()):
            tiles[t] = tiles.get(t, 0) + 1
    if not torch.equal(y, yref):
        bad_y += 1
print(os.path.basename(sys.argv[1]), "bad gu", bad_gu, "bad y", bad_y, "of", len(outs), "tiles", sorted(tiles.items())[:12])
