"""Per-CTA timeline of one fireq_w4a8_gemm launch (debug trace) + event timing."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2505_20839_b200 import fireq as F

F.load(os.path.join(os.path.dirname(F.LIB_PATH), 'libfireq_prof.so'))
for (M, N, K) in [(16, 22016, 4096), (16, 4096, 11008), (16, 4096, 4096), (16384, 22016, 4096)]:
    W = synth.bits_to_torch(synth.weights(N, K, 1)).cuda()
    X = synth.bits_to_torch(synth.activations(M, K, 2)).cuda()
    qw = F.quantize_weight(W, 1)
    xq, beta = F.quantize_act(X, chan_mul=qw.c)
    ws = F.Workspace(F.gemm_workspace_bytes(M, N, K))
    out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    n = qw.n
    plan = F.gemm_plan(M, N, K)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    tr = torch.zeros(plan["ctas"] * 32 + 512, dtype=torch.int64, device="cuda")
    for it in range(3):
        flush.fill_(it)
        F.debug_set_trace(tr if it == 2 else None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, n, out=out, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
    F.debug_set_trace(None)
    t16 = tr.cpu().numpy()[: plan["ctas"] * 16].reshape(-1, 16).astype(np.int64)
    t = t16[:, :8]
    t0 = t[:, 0].min()
    rel = np.where(t > 0, (t - t0) / 1000.0, np.nan)
    print(f"M={M} N={N} K={K} plan={plan} event={e0.elapsed_time(e1)*1e3:.1f}us")
    names = ["start", "setup", "first_data", "mma_done", "epi_done", "end", "drained", "fixup_done"]
    for j, nm in enumerate(names):
        col = rel[:, j]
        col = col[~np.isnan(col)]
        if col.size:
            print(f"   {nm:10s} min={col.min():8.2f} med={np.median(col):8.2f} max={col.max():8.2f} us  (n={col.size})")
    cyc = t16[:, 8:16]
    cn = ["prod_wait_empty", "mma_wait_afull", "mma_wait_full", "mma_total", "conv_wait_full", "conv_wait_aempty", "conv_total", "mma_issue"]
    for j, nm in enumerate(cn):
        print(f"   cyc {nm:18s} med={np.median(cyc[:, j]):9.0f}")
    del W, X, qw, flush
    torch.cuda.empty_cache()
    if os.environ.get("TRACE_SLOW"):
        order = np.argsort(-np.nan_to_num(rel[:, 5]))
        print("   slowest CTAs: cta " + " ".join(f"{n:>10s}" for n in names))
        for c in order[:12]:
            print(f"   {c:4d} " + " ".join(f"{v:10.2f}" for v in rel[c]))
        t2 = tr.cpu().numpy()[plan["ctas"] * 16 + 512:].reshape(-1, 16).astype(np.int64)
        rel2 = np.where(t2 > 0, (t2 - t0) / 1000.0, np.nan)
        print("   epilogue per segment: accfull seen / arrived (stream-K) / segment done")
        for c in order[:12]:
            print(f"   {c:4d} " + " ".join(f"{v:7.2f}" for v in rel2[c, :12]))
