"""Per-CTA timeline of the fused decode FFN (profile build): FIREQ_FFN_PERSISTENT=1 runs gate_up
and down in one grid (NPH = 2); prints phase milestones (us from the first CTA start)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_20839_b200 import fireq as F
F.load(os.path.join(os.path.dirname(F.LIB_PATH), 'libfireq_prof.so'))
import bench
dev = torch.device("cuda", 0)
ffn = bench.FusedFFN(F, 16, 4, dev)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for r in range(8):
        ffn.step(r % 4, s)
torch.cuda.synchronize()
C = 148
tr = torch.zeros(C * 48 + 512 + 64, dtype=torch.int64, device=dev)
for it in range(9):
    F.debug_set_trace(tr if it == 8 else None)
    with torch.cuda.stream(s):
        ffn.step(it % 4, s)
F.debug_set_trace(None)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.int64)
t1 = t[:C * 16].reshape(C, 16)
t2 = t[C * 16 + 512: C * 16 + 512 + C * 16].reshape(C, 16)
t0 = t1[:, 0][t1[:, 0] > 0].min()
def col(a, j):
    v = a[:, j]
    v = v[v > 0]
    return (v - t0) / 1e3
for nm, a, j in [("start", t1, 0), ("setup", t1, 1), ("first_data", t1, 2), ("mma_done", t1, 3), ("epi_done", t1, 4),
                 ("end", t1, 5), ("seg0 accfull", t2, 0), ("seg0 done", t2, 2), ("seg1 accfull", t2, 3), ("seg1 done", t2, 5),
                 ("seg2 accfull", t2, 6), ("seg2 done", t2, 8), ("seg3 accfull", t2, 9),
                 ]:
    c = col(a, j)
    if c.size:
        print(f"  {nm:18s} min={c.min():7.2f} med={np.median(c):7.2f} max={c.max():7.2f}  n={c.size}")
t3 = t[C * 32 + 512: C * 32 + 512 + C * 16].reshape(C, 16)
for nm, j in [("epi after pdl_wait", 0), ("phase A done", 1), ("G1 passed", 2), ("X prod ph0 start", 3),
              ("W prod ph0 last issue", 9), ("G2 passed", 4), ("phase C slice done", 5), ("G3 passed", 8), ("X prod ph1 start", 6),
              ("MMA ph1 first stage", 7), ("W prod ph1 first issue", 10), ("W prod done", 11)]:
    c = col(t3, j)
    if c.size:
        print(f"  {nm:22s} min={c.min():7.2f} med={np.median(c):7.2f} max={c.max():7.2f}  n={c.size}")
