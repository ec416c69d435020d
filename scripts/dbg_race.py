"""Race hunt: unfused chain + fused FFN back to back without syncs, vs. synced references."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from paper_2505_20839_b200 import fireq as F
F.load()
import test_gpu_ffn as T
M, d, dff = 16, 4096, 11008
*_, qgu, qil, qd, x = T._ffn_case(F, M, d, dff, 91)
gamma = torch.cat([torch.ones(dff, device="cuda"), qd.c.float()])
S = torch.cuda.synchronize


def unfused(sync):
    xq, beta = F.quantize_act(x, chan_mul=qgu.c); sync()
    gu = F.w4a8_gemm(xq, beta, qgu.packed, qgu.scales, 2 * dff, qgu.n, gamma=gamma); sync()
    hq, hb = F.silu_mul_quantize_act(gu[:, :dff], gu[:, dff:]); sync()
    y = F.w4a8_gemm(hq, hb, qd.packed, qd.scales, d, qd.n); sync()
    return xq, beta, gu, hq, hb, y


def fused(sync, ws):
    h = torch.empty((M, dff), dtype=torch.bfloat16, device="cuda")
    y = F.ffn_w4a8_decode(x, qil, qd, h=h, workspace=ws); sync()
    return h, y


snap = {"gamma": gamma.clone(), "gu.packed": qgu.packed.clone(), "gu.scales": qgu.scales.clone(), "x": x.clone(),
        "gu.c": qgu.c.clone(), "il.packed": qil.packed.clone(), "il.scales": qil.scales.clone(),
        "d.packed": qd.packed.clone(), "d.scales": qd.scales.clone(), "d.c": qd.c.clone()}
live = {"gamma": gamma, "gu.packed": qgu.packed, "gu.scales": qgu.scales, "x": x, "gu.c": qgu.c,
        "il.packed": qil.packed, "il.scales": qil.scales, "d.packed": qd.packed, "d.scales": qd.scales, "d.c": qd.c}
def check(tag):
    S()
    for k in snap:
        if not torch.equal(snap[k], live[k]):
            dz = (snap[k].float() - live[k].float()).abs().nonzero()
            print(tag, "CORRUPTED", k, dz.shape[0], dz[:4].flatten().tolist(), "ptr", hex(live[k].data_ptr()), "numel", live[k].numel())
ref_u = unfused(S)
check("after ref_u")
ws = F.Workspace(F.ffn_workspace_bytes(M, d, dff))
ref_f = fused(S, ws)
check("after ref_f")
names_u = ["xq", "beta", "gu", "hq", "hb", "y"]
bad = {}
for it in range(40):
    u = unfused(lambda: None)
    f = fused(lambda: None, ws)
    S()
    for nm, a, b in zip(names_u, u, ref_u):
        if not torch.equal(a, b):
            bad.setdefault("unfused." + nm, []).append(it)
    for nm, a, b in zip(["h", "y"], f, ref_f):
        if not torch.equal(a, b):
            bad.setdefault("fused." + nm, []).append(it)
print("mismatches:", {k: v[:10] for k, v in bad.items()})
check("after loop")
print("ws ptr", hex(ws.t.data_ptr()), ws.t.numel())
if "unfused.gu" in bad:
    u = unfused(lambda: None); S()
    diff = (u[2].float() - ref_u[2].float()).abs().nonzero()
    print("gu diff count", diff.shape[0], "first", diff[:5].tolist())
# detail: unfused chain only, 60 iterations, report y mismatches by (token, tile)
cnt = 0
for it in range(200):
    u = unfused(lambda: None)
    S()
    if not torch.equal(u[5], ref_u[5]):
        cnt += 1
        same_in = all(torch.equal(a, b) for a, b in zip(u[:5], ref_u[:5]))
        dd = (u[5].float() - ref_u[5].float()).abs()
        nz = dd.nonzero()
        toks = sorted(set(nz[:, 0].tolist())); tiles = sorted(set((nz[:, 1] // 128).tolist()))
        print(f"it {it}: inputs identical={same_in} n={nz.shape[0]} tokens={toks[:16]} tiles={tiles[:16]} maxdiff={dd.max().item():.4g}")
        for nm, a, b in zip(names_u[:5], u[:5], ref_u[:5]):
            if not torch.equal(a, b):
                dz = (a.float() - b.float()).abs().nonzero()
                print("   ", nm, "differs at", dz.shape[0], "first", dz[:6].tolist())
print("unfused-only y mismatches:", cnt)
# down GEMM alone on fixed inputs
cnt = 0
for it in range(100):
    y = F.w4a8_gemm(ref_u[3], ref_u[4], qd.packed, qd.scales, d, qd.n)
    if not torch.equal(y, ref_u[5]):
        cnt += 1
S()
print("down-alone mismatches (async check, may be 0):", cnt)
ys = [F.w4a8_gemm(ref_u[3], ref_u[4], qd.packed, qd.scales, d, qd.n) for _ in range(100)]
S()
print("down-alone mismatches:", sum(not torch.equal(y, ref_u[5]) for y in ys))
