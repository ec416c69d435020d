"""sigma_BF16 vs sigma_FP8 GEMM time on the same shapes (the paper reports the
BF16-scale kernel at about 0.6x the FP8-scale throughput).  Prints one JSON line."""
import json
import sys

import torch

sys.path.insert(0, ".")
import synth
from paper_2505_20839_b200 import fireq as F


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    out = {}
    for (M, N, K) in [(16, 22016, 4096), (16, 4096, 11008), (128, 22016, 4096), (4096, 22016, 4096)]:
        wb = synth.weights(N, K, 1)
        Wd = synth.bits_to_torch(wb).cuda()
        q8 = F.quantize_weight(Wd, cas_mode=1)
        q16 = F.quantize_weight_bf16s(Wd, cas_mode=1)
        xq, beta = F.quantize_act(synth.bits_to_torch(synth.activations(M, K, 2)).cuda(), chan_mul=q8.c)
        ws8 = F.Workspace(F.gemm_workspace_bytes(M, N, K), "cuda")
        ws16 = F.Workspace(F.lib().fireq_w4a8_gemm_bf16s_workspace_bytes(M, N, K), "cuda")
        y8 = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
        y16 = torch.empty_like(y8)
        reps = 200 if M <= 128 else 20
        t8 = timed(lambda: F.w4a8_gemm(xq, beta, q8.packed, q8.scales, N, q8.n, out=y8, workspace=ws8), reps)
        t16 = timed(lambda: F.w4a8_gemm_bf16s(xq, beta, q16.packed, q16.scales, N, q16.n, out=y16, workspace=ws16),
                    reps)
        out[f"{M}x{N}x{K}"] = {"fp8_scales_us": round(t8, 2), "bf16_scales_us": round(t16, 2),
                               "bf16_over_fp8_throughput": round(t8 / t16, 3)}
        del Wd, q8, q16, ws8, ws16
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
