"""Per-CTA timelines of the gate_up and down GEMMs INSIDE the decode FFN chain (profile build).

Graph of 3 FFN steps; the middle step's two GEMMs record per-CTA traces, all kernels record
spans; times are relative to the middle step's act_quant start (ns -> us)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_20839_b200 import fireq as F
F.load(os.path.join(os.path.dirname(F.LIB_PATH), 'libfireq_prof.so'))
import bench
dev = torch.device("cuda", 0)
M = 16
ffn = bench.FFN(F, M, 4, dev)
stream = torch.cuda.Stream()
for r in range(8):
    with torch.cuda.stream(stream):
        ffn.step(r % 4, stream)
torch.cuda.synchronize()
D_FF, D_MODEL = bench.D_FF, bench.D_MODEL
pg = F.gemm_plan(M, 2 * D_FF, D_MODEL)
pd = F.gemm_plan(M, D_MODEL, D_FF)
trg = torch.zeros(pg["ctas"] * 32 + 512, dtype=torch.int64, device=dev)
trd = torch.zeros(pd["ctas"] * 32 + 512, dtype=torch.int64, device=dev)
spans = torch.zeros((12, 2), dtype=torch.int64, device=dev)


def step(r, traced):
    p_gu, s_gu, p_d, s_d = ffn.rot[r]
    nxt = ffn.rot[(r + 1) % 4]
    F.quantize_act(ffn.x, chan_mul=ffn.c_gu, out=(ffn.xq, ffn.beta), stream=stream)
    F.debug_set_trace(trg if traced else None)
    F.w4a8_gemm(ffn.xq, ffn.beta, p_gu, s_gu, 2 * D_FF, ffn.n_gu, gamma=ffn.gamma, out=ffn.gu, workspace=ffn.ws1,
                stream=stream, prefetch=(p_d, s_d))
    F.debug_set_trace(None)
    F.silu_mul_quantize_act(ffn.gu[:, :D_FF], ffn.gu[:, D_FF:], out=(ffn.hq, ffn.hbeta), stream=stream)
    F.debug_set_trace(trd if traced else None)
    F.w4a8_gemm(ffn.hq, ffn.hbeta, p_d, s_d, D_MODEL, ffn.n_d, out=ffn.y, workspace=ffn.ws2, stream=stream,
                prefetch=(nxt[0], nxt[1]))
    F.debug_set_trace(None)


F.debug_set_spans(spans)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    for r in range(3):
        step(r, r == 1)
F.debug_set_spans(None)
names = ["act_quant(x)", "gemm gate_up", "silu_mul_quant", "gemm down"]
for trial in range(3):
    spans[:, 0] = -1
    spans[:, 1] = 0
    trg.zero_(); trd.zero_()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
sp = spans.cpu().numpy().astype(np.uint64).astype(np.float64)
t0 = sp[4, 0]
for i in range(4, 12):
    print(f"   {names[i % 4]:16s} start {(sp[i,0]-t0)/1e3:8.2f}  end {(sp[i,1]-t0)/1e3:8.2f} us")
tl = ["start", "setup", "first_data", "mma_done", "epi_done", "end", "drained", "fixup_done"]
for name, tr, plan in (("gate_up", trg, pg), ("down", trd, pd)):
    C = plan["ctas"]
    a = tr.cpu().numpy()
    t16 = a[: C * 16].reshape(-1, 16)[:, :8].astype(np.float64)
    rel = np.where(t16 > 0, (t16 - t0) / 1e3, np.nan)
    print(f"{name}: {plan}")
    for j, nm in enumerate(tl):
        col = rel[:, j]
        col = col[~np.isnan(col)]
        if col.size:
            print(f"   {nm:10s} min={col.min():7.2f} med={np.median(col):7.2f} max={col.max():7.2f}  (n={col.size})")
    t2 = a[C * 16 + 512: C * 32 + 512].reshape(-1, 16).astype(np.float64)
    rel2 = np.where(t2 > 0, (t2 - t0) / 1e3, np.nan)
    order = np.argsort(-np.nan_to_num(rel[:, 5]))
    print("   slowest CTAs: start setup first mma_done epi_done end | per segment: accfull arrived done")
    for c in order[:8]:
        print(f"   {c:4d} " + " ".join(f"{v:6.2f}" for v in rel[c, [0, 1, 2, 3, 4, 5]]) + " | " +
              " ".join(f"{v:6.2f}" for v in rel2[c, :13]))
