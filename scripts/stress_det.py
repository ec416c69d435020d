"""Determinism stress: repeated launches of each GEMM schedule must be bit-identical
(R23: fixed reduction orders; a race would show up as rare differing tiles).
usage: stress_det.py [repeats]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_20839_b200 import fireq as F
F.load()
R = int(sys.argv[1]) if len(sys.argv) > 1 else 200
cases = [(16, 22016, 4096), (16, 4096, 11008), (16, 1024, 4096), (16, 150 * 128, 512), (32, 4096, 14336),
         (64, 4096, 14336), (128, 4096, 14336), (256, 4096, 14336), (100, 256, 768), (300, 256, 384), (300, 9600, 512), (1024, 4096, 14336), (4096, 1024, 4096),
         (16384, 4096, 4096)]
bad = 0
for M, N, K in cases:
    W = synth.bits_to_torch(synth.weights(N, K, 5)).cuda()
    X = synth.bits_to_torch(synth.activations(M, K, 6)).cuda()
    qw = F.quantize_weight(W, 1)
    xq, beta = F.quantize_act(X, chan_mul=qw.c)
    ws = F.Workspace(F.gemm_workspace_bytes(M, N, K))
    ref = F.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, workspace=ws).clone()
    out = torch.empty_like(ref)
    reps = R if M <= 1024 else max(5, R // 20)
    diff = 0
    for i in range(reps):
        F.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, out=out, workspace=ws)
        if i % 4 == 3 or i == reps - 1:
            torch.cuda.synchronize()
        if not torch.equal(out, ref):
            diff += 1
    torch.cuda.synchronize()
    pl = F.gemm_plan(M, N, K)
    tiles = (-(-M // pl["ntok"])) * (N // 128)
    zero = int(ws.t[: 4 * tiles].view(torch.int32).abs().sum())   # per-tile arrival counters
    print(f"M={M:6d} N={N:6d} K={K:6d} {F.gemm_plan(M, N, K)['mode']:16s} repeats={reps:4d} differing={diff} counters_left={zero}", flush=True)
    bad += diff + (zero != 0)
    del W, X, qw, xq, beta, ws, ref, out
    torch.cuda.empty_cache()
print("STRESS", "OK" if bad == 0 else f"FAILED ({bad})")
