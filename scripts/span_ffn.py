"""Timeline of one decode FFN step (profile build): kernel spans in a PDL chain."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_20839_b200 import fireq as F
F.load(os.path.join(os.path.dirname(F.LIB_PATH), 'libfireq_prof.so'))
import bench
dev = torch.device("cuda", 0)
FUSED = os.environ.get("FUSED") == "1"
ffn = bench.FusedFFN(F, 16, 4, dev) if FUSED else bench.FFN(F, 16, 4, dev)
stream = torch.cuda.Stream()
for r in range(8):
    with torch.cuda.stream(stream):
        ffn.step(r % 4, stream)
torch.cuda.synchronize()
names = (["act_quant(x)", "gemm gate_up+SwiGLU", "act_quant(h)", "gemm down"] if FUSED else
         ["act_quant(x)", "gemm gate_up", "silu_mul_quant", "gemm down"])
buf = torch.zeros((4 * 3, 2), dtype=torch.int64, device=dev)
F.debug_set_spans(buf)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    for r in range(3):
        ffn.step(r, stream)
F.debug_set_spans(None)
for trial in range(3):
    buf[:, 0] = -1
    buf[:, 1] = 0
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    sp = buf.cpu().numpy().astype(np.uint64).astype(np.float64)
    t0 = sp[4, 0]
    print(f"trial {trial}: step 2 and 3 (ns relative to step-2 start)")
    for i in range(4, 12):
        print(f"   {names[i % 4]:16s} start {sp[i,0]-t0:9.0f}  end {sp[i,1]-t0:9.0f}  dur {sp[i,1]-sp[i,0]:8.0f}")
