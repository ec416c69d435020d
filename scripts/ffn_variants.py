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
    for res in ((0, 1, 2) if cls is bench.FFN else (0, 1)):
        if cls is bench.FFN:
            def step(r, res=res):
                if res == 2:                 # the down GEMM with the residual in its epilogue
                    F.quantize_act(ffn.x, chan_mul=ffn.c_gu, out=(ffn.xq, ffn.beta), stream=s)
                    p_gu, s_gu, p_d, s_d = ffn.rot[r]
                    F.w4a8_gemm(ffn.xq, ffn.beta, p_gu, s_gu, 2 * bench.D_FF, ffn.n_gu, gamma=ffn.gamma, out=ffn.gu,
                                workspace=ffn.ws1, stream=s)
                    F.silu_mul_quantize_act(ffn.gu[:, :bench.D_FF], ffn.gu[:, bench.D_FF:], out=(ffn.hq, ffn.hbeta),
                                            stream=s)
                    F.w4a8_gemm(ffn.hq, ffn.hbeta, p_d, s_d, bench.D_MODEL, ffn.n_d, out=ffn.y, workspace=ffn.ws2,
                                stream=s, residual=ffn.x)
                    return
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
