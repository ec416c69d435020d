"""Per-kernel times of the Llama2-70B FFN at P = 1 (decode M = 16 or prefill M from argv)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2505_20839_b200 import fireq as F
F.load()
M = int(sys.argv[1]) if len(sys.argv) > 1 else 16
d, dff = 8192, 28672
dev = torch.device("cuda")
Wgu = synth.bits_to_torch(np.concatenate([synth.weights(dff, d, 1), synth.weights(dff, d, 2)])).to(dev)
q_gu = F.quantize_weight(Wgu, 1); del Wgu
Wd = synth.bits_to_torch(synth.weights(d, dff, 3)).to(dev)
q_d = F.quantize_weight(Wd, 1); del Wd
x = synth.bits_to_torch(synth.activations(M, d, 4)).to(dev)
xq, beta = F.quantize_act(x, chan_mul=q_gu.c)
gam = torch.cat([torch.ones(dff, device=dev), q_d.c.float()])
ws1 = F.Workspace(F.gemm_workspace_bytes(M, 2 * dff, d)); ws2 = F.Workspace(F.gemm_workspace_bytes(M, d, dff))
gt = torch.empty((2 * dff, M), dtype=torch.bfloat16, device=dev); g = torch.empty((M, 2 * dff), dtype=torch.bfloat16, device=dev)
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
print("plan gate_up", F.gemm_plan(M, 2 * dff, d), "down", F.gemm_plan(M, d, dff))
print(f"quantize_act x        {t(lambda: F.quantize_act(x, chan_mul=q_gu.c, out=(xq, beta))):9.1f} us")
print(f"gate_up Y^T           {t(lambda: F.w4a8_gemm(xq, beta, q_gu.packed, q_gu.scales, 2 * dff, q_gu.n, gamma=gam, out=gt, out_layout=1, workspace=ws1)):9.1f} us")
print(f"gate_up Y             {t(lambda: F.w4a8_gemm(xq, beta, q_gu.packed, q_gu.scales, 2 * dff, q_gu.n, gamma=gam, out=g, workspace=ws1)):9.1f} us")
hq, hb = F.silu_mul_quantize_act_t(gt[:dff], gt[dff:], M, dff)
print(f"silu_mul_quant_t      {t(lambda: F.silu_mul_quantize_act_t(gt[:dff], gt[dff:], M, dff, out=(hq, hb))):9.1f} us")
print(f"silu_mul_quant (row)  {t(lambda: F.silu_mul_quantize_act(g[:, :dff], g[:, dff:], out=(hq, hb))):9.1f} us")
yt = torch.empty((d, M), dtype=torch.bfloat16, device=dev)
print(f"down Y^T              {t(lambda: F.w4a8_gemm(hq, hb, q_d.packed, q_d.scales, d, q_d.n, out=yt, out_layout=1, workspace=ws2)):9.1f} us")
wb = (2 * dff * d + d * dff) * (0.5 + 1 / 128)
print(f"weights {wb / 1e6:.1f} MB")
