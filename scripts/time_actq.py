"""Per-launch time of the activation quantizers (graph of back-to-back PDL launches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2505_20839_b200 import fireq as F
F.load()
M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
gu = synth.bits_to_torch(synth.activations(M, 22016, 3)).cuda()
x = synth.bits_to_torch(synth.activations(M, 4096, 4)).cuda()
c = torch.ones(4096, dtype=torch.bfloat16, device="cuda")
hq = torch.empty((M, 11008), dtype=torch.uint8, device="cuda"); hb = torch.empty(M, dtype=torch.bfloat16, device="cuda")
xq = torch.empty((M, 4096), dtype=torch.uint8, device="cuda"); xb = torch.empty(M, dtype=torch.bfloat16, device="cuda")
s = torch.cuda.Stream()
for name, fn in [("silu_mul_quantize_act 16x11008", lambda: F.silu_mul_quantize_act(gu[:, :11008], gu[:, 11008:], out=(hq, hb), stream=s)),
                 ("quantize_act(c) 16x4096", lambda: F.quantize_act(x, chan_mul=c, out=(xq, xb), stream=s)),
                 ("quantize_act 16x11008 (h)", lambda: F.quantize_act(gu[:, :11008], out=(hq, hb), stream=s))]:
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(20):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 400
    nbytes = M * 22016 * 2 + M * 11008 if "silu" in name else (M * 11008 * 3 if "(h)" in name else M * 4096 * 3)
    print(f"{name.replace('16x', str(M) + 'x')}: {us:.2f} us per launch, {nbytes / us / 1e3:.0f} GB/s")
