"""Fused decode FFN (fireq_ffn_w4a8_decode) inside a graph of 3 steps: kernel spans and the
per-CTA timeline of gate_up (FIREQ_TRACE_WHICH=1) or down (=2) of the middle step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_20839_b200 import fireq as F
F.load(os.path.join(os.path.dirname(F.LIB_PATH), 'libfireq_prof.so'))
import bench
dev = torch.device("cuda", 0)
M = 16
ffn = bench.FusedFFN(F, M, 4, dev)
stream = torch.cuda.Stream()
for r in range(8):
    with torch.cuda.stream(stream):
        ffn.step(r % 4, stream)
torch.cuda.synchronize()
which = int(os.environ.get("FIREQ_TRACE_WHICH", "1"))
D_FF, D_MODEL = bench.D_FF, bench.D_MODEL
plan = F.gemm_plan(M, 2 * D_FF, D_MODEL) if which == 1 else F.gemm_plan(M, D_MODEL, D_FF)
tr = torch.zeros(plan["ctas"] * 32 + 512, dtype=torch.int64, device=dev)
NK = 3
spans = torch.zeros((3 * NK, 2), dtype=torch.int64, device=dev)
F.debug_set_spans(spans)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    for r in range(3):
        F.debug_set_trace(tr if r == 1 else None)
        ffn.step(r, stream)
        F.debug_set_trace(None)
F.debug_set_spans(None)
for trial in range(3):
    spans[:, 0] = -1
    spans[:, 1] = 0
    tr.zero_()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
sp = spans.cpu().numpy().astype(np.uint64).astype(np.float64)
t0 = sp[NK, 0]
names = ["act_quant(x)", "ffn(gate_up|down)", "(unused slot)"] if os.environ.get("PERSIST", "1") == "1" else ["act_quant(x)", "gate_up+swiglu+hq", "down"]
for i in range(3 * NK):
    print(f"   {names[i % NK]:20s} start {(sp[i,0]-t0)/1e3:8.2f}  end {(sp[i,1]-t0)/1e3:8.2f} us")
C = plan["ctas"]
a = tr.cpu().numpy()
t16 = a[: C * 16].reshape(-1, 16)[:, :8].astype(np.float64)
rel = np.where(t16 > 0, (t16 - t0) / 1e3, np.nan)
print(f"phase {which}: {plan}")
for j, nm in enumerate(["start", "setup", "first_data", "mma_done", "epi_done", "end", "drained", "fixup_done"]):
    col = rel[:, j]
    col = col[~np.isnan(col)]
    if col.size:
        print(f"   {nm:10s} min={col.min():7.2f} med={np.median(col):7.2f} max={col.max():7.2f}  (n={col.size})")
t2 = a[C * 16 + 512: C * 32 + 512].reshape(-1, 16).astype(np.float64)
rel2 = np.where(t2 > 0, (t2 - t0) / 1e3, np.nan)
for slot, nm in ((15, "grid_bar"),):
    col = rel2[:, slot]
    col = col[~np.isnan(col)]
    if col.size:
        print(f"   {nm:10s} min={col.min():7.2f} med={np.median(col):7.2f} max={col.max():7.2f}")
order = np.argsort(-np.nan_to_num(rel[:, 5]))
print("   slowest: start setup first mma_done epi_done end | accfull arrived done ...")
for c in order[:6]:
    print(f"   {c:4d} " + " ".join(f"{v:6.2f}" for v in rel[c, [0, 1, 2, 3, 4, 5]]) + " | " +
          " ".join(f"{v:6.2f}" for v in rel2[c, :9]))
if os.environ.get("EVT"):
    ev = a[C * 16: C * 16 + 512].reshape(64, 8).astype(np.int64)
    base = ev[0, 0]
    print("CTA0 stage events (cycles from stage-0 weight issue): prodW conv_fullW conv_Aok conv_arrive mma_afull mma_fullX mma_issued")
    for i in range(64):
        if ev[i, 0] == 0 and ev[i, 6] == 0:
            break
        print(f"{i:3d} " + " ".join(f"{(ev[i, j] - base) if ev[i, j] else -1:9d}" for j in range(7)))
