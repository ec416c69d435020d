"""Decode FFN step timings (Llama2-7B, batch 16): the 4-kernel chain, fireq_ffn_w4a8_decode,
each with and without the residual connection (chain: y += x as its own kernel; fused: in the
down GEMM's epilogue).  env LIB: alternative .so; FIREQ_FFN_MODE / FIREQ_FFN_PERSISTENT select
the fused path's variant."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2505_20839_b200 import fireq as F
F.load(os.environ["LIB"]) if os.environ.get("LIB") else F.load()
import bench
dev = torch.device("cuda", 0)
tag = f"mode={os.environ.get('FIREQ_FFN_MODE', '4')} persistent={os.environ.get('FIREQ_FFN_PERSISTENT', '0')}"
for name, cls in [("chain4", bench.FFN), ("fused", bench.FusedFFN)]:
    ffn = cls(F, 16, 4, dev)
    s = torch.cuda.Stream()
    for res in (False, True):
        if cls is bench.FFN:
            def step(r, res=res):
                ffn.step(r, s)
                if res:
                    ffn.y.add_(ffn.x)
        else:
            def step(r, res=res):
                ffn.step(r, s, residual=res)
        with torch.cuda.stream(s):
            for r in range(4): step(r)
        torch.cuda.synchronize()
        gm = bench.capture(lambda: [step(r) for r in range(4)], s)
        gs = [bench.capture(lambda r=r: step(r), s) for r in range(4)]
        ms = bench.time_steps(gm, gs, 2000, 50, s)
        print(f"{name:7s} residual={int(res)} {tag}: {ms * 1e3 / 2000:.3f} us/step", flush=True)
        del gm, gs
    del ffn
    torch.cuda.empty_cache()
