"""Time fireq_w4a8_gemm launches (CUDA graph of back-to-back launches over ROT weight copies).
usage: time_gemm.py M N K [M N K ...]   env: ROT (default 4), LIB (alternative .so)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2505_20839_b200 import fireq as F

F.load(os.environ["LIB"]) if os.environ.get("LIB") else F.load()
ROT = int(os.environ.get("ROT", "4"))
args = [int(v) for v in sys.argv[1:]]
for M, N, K in zip(args[0::3], args[1::3], args[2::3]):
    W = synth.bits_to_torch(synth.weights(N, K, 1)).cuda()
    X = synth.bits_to_torch(synth.activations(M, K, 2)).cuda()
    qw = F.quantize_weight(W, 1)
    xq, beta = F.quantize_act(X, chan_mul=qw.c)
    del W
    rot = [(qw.packed.clone(), qw.scales.clone()) for _ in range(ROT)]
    ws = F.Workspace(F.gemm_workspace_bytes(M, N, K))
    out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    gam = torch.rand(N, device="cuda") + 0.5 if os.environ.get("GAMMA") else None
    res = torch.randn((M, N), device="cuda").bfloat16() if os.environ.get("RESIDUAL") else None
    s = torch.cuda.Stream()
    def run():
        for p, sc in rot:
            F.w4a8_gemm(xq, beta, p, sc, N, qw.n, gamma=gam, out=out, workspace=ws, stream=s, residual=res)
    with torch.cuda.stream(s):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(max(1, 32 // ROT)):
            run()
    nl = max(1, 32 // ROT) * ROT
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * nl)
    b = N * K // 2 + N * K // 128 + M * K + 2 * M + 2 * M * N
    print(f"M={M:6d} N={N:6d} K={K:6d} plan={F.gemm_plan(M, N, K)} {us:9.2f} us  {b / us / 1e3:8.1f} GB/s  "
          f"{2 * M * N * K / us / 1e6:8.1f} TFLOP/s", flush=True)
    del rot, qw, out, ws, g
    torch.cuda.empty_cache()
