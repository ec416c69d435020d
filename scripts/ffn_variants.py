import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2505_20839_b200 import fireq as F
F.load(os.environ["LIB"]) if os.environ.get("LIB") else F.load()
import bench
dev = torch.device("cuda", 0)
for name, cls in [("chain4", bench.FFN), ("fused", bench.FusedFFN)]:
    ffn = cls(F, 16, 4, dev)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for r in range(4): ffn.step(r, s)
    torch.cuda.synchronize()
    gm = bench.capture(lambda: [ffn.step(r, s) for r in range(4)], s)
    gs = [bench.capture(lambda r=r: ffn.step(r, s), s) for r in range(4)]
    ms = bench.time_steps(gm, gs, 2000, 50, s)
    print(f"{name} persistent={os.environ.get('FIREQ_FFN_PERSISTENT', '0')}: {ms * 1e3 / 2000:.3f} us/step", flush=True)
    del ffn, gm, gs
    torch.cuda.empty_cache()
