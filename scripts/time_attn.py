"""Time fireq_kv4q8_attention (CUDA events over a graph of launches): Llama3-8B prefill attention
(B sequences x N tokens, Hq = 32 query heads, Hkv = 8 kv heads, d = 128, causal).
usage: time_attn.py [B N Hq Hkv ...]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2505_20839_b200 import fireq as F

F.load(os.environ["LIB"]) if os.environ.get("LIB") else F.load()
args = [int(v) for v in sys.argv[1:]] or [16, 1024, 32, 8, 1, 4096, 32, 8]
res = []
for B, N, Hq, Hkv in zip(args[0::4], args[1::4], args[2::4], args[3::4]):
    qb, kb, vb = synth.attention(B, N, Hq, Hkv, 5)
    Q, K, V = (synth.bits_to_torch(x).cuda() for x in (qb, kb, vb))
    cache = F.KVCache(K, V)
    xq, beta = F.quantize_act(Q.reshape(B * Hq * N, 128))
    q_fp8, q_scale = xq.reshape(B, Hq, N, 128), beta.reshape(B, Hq, N)
    out = torch.empty((B * N, Hq * 128), dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        F.kv4q8_attention(q_fp8, q_scale, cache, Hq, out=out, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    per = 10
    with torch.cuda.graph(g, stream=s):
        for _ in range(per):
            F.kv4q8_attention(q_fp8, q_scale, cache, Hq, out=out, stream=s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    with torch.cuda.stream(s):
        g.replay()
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * per)
    flops = 4.0 * 128 * B * Hq * N * (N + 1) / 2          # causal: S and O, 2 flop per MAC
    kernel_flops = 0
    T = N // 128
    for i in range(T):
        kernel_flops += B * Hq * (3 * (i + 1)) * 2 * 128 * 128 * 128   # pass-1 S, pass-2 S and O per kv tile
    r = {"B": B, "N": N, "Hq": Hq, "Hkv": Hkv, "us": round(us, 2), "tflops_algorithmic": round(flops / us / 1e6, 1),
         "tflops_issued": round(kernel_flops / us / 1e6, 1)}
    print(json.dumps(r), flush=True)
    res.append(r)
