# A/B of the decode FFN step (bench.FFN, graph of PDL-chained steps): current vs libfireq_prev.so
cd $GRAFT_REPO_ROOT
cat > /tmp/ffn_ab.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2505_20839_b200 import fireq as F
F.load(os.environ["LIB"])
import bench
dev = torch.device("cuda", 0)
ffn = bench.FFN(F, 16, 4, dev)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for r in range(4): ffn.step(r, s)
torch.cuda.synchronize()
gm = bench.capture(lambda: [ffn.step(r, s) for r in range(4)], s)
gs = [bench.capture(lambda r=r: ffn.step(r, s), s) for r in range(4)]
ms = bench.time_steps(gm, gs, 2000, 50, s)
print(f"{os.path.basename(os.environ['LIB'])}: FFN {ms * 1e3 / 2000:.3f} us/step")
PY
for i in 1 2; do for lib in libfireq_prev.so libfireq.so; do LIB=paper_2505_20839_b200/$lib timeout 120 python /tmp/ffn_ab.py; done; done 2>&1 | grep FFN
