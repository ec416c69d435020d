"""Per-CTA timeline of one fireq_w4a8_gemm launch (debug trace) + event timing."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2505_20839_b200 import fireq as F

F.load(os.path.join(os.path.dirname(F.LIB_PATH), 'libfireq_prof.so'))
SHAPES = [(16, 22016, 4096), (16, 4096, 11008), (16, 4096, 4096), (16384, 22016, 4096)]
if len(sys.argv) > 3:
    a = [int(v) for v in sys.argv[1:]]
    SHAPES = list(zip(a[0::3], a[1::3], a[2::3]))
for (M, N, K) in SHAPES:
    W = synth.bits_to_torch(synth.weights(N, K, 1)).cuda()
    X = synth.bits_to_torch(synth.activations(M, K, 2)).cuda()
    qw = F.quantize_weight(W, 1)
    xq, beta = F.quantize_act(X, chan_mul=qw.c)
    ws = F.Workspace(F.gemm_workspace_bytes(M, N, K))
    out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    n = qw.n
    plan = F.gemm_plan(M, N, K)
    # ROT weight copies launched back to back (HBM-resident, no L2 flush write-back in flight);
    # the last launch is traced
    ROT = int(os.environ.get("ROT", "4"))
    rot = [(qw.packed.clone(), qw.scales.clone()) for _ in range(ROT)]
    tr = torch.zeros(plan["ctas"] * 32 + 512, dtype=torch.int64, device="cuda")
    for it in range(2 * ROT + 1):
        F.debug_set_trace(tr if it == 2 * ROT else None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F.w4a8_gemm(xq, beta, rot[it % ROT][0], rot[it % ROT][1], N, n, out=out, workspace=ws)
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
    fw = np.where(t16[:, 8] > 0, (t16[:, 8] - t0) / 1000.0, np.nan)
    print(f"   first_W_issue min={np.nanmin(fw):8.2f} med={np.nanmedian(fw):8.2f} max={np.nanmax(fw):8.2f} us")
    if os.environ.get("FIREQ_DEBUG_MODE", "0") == "64":
        for j, nm in [(9, "bar_init_done"), (10, "tmem_alloc_done"), (12, "lut_done_t0"), (13, "after_syncthreads"), (11, "prod_role_start"), (14, "prod_after_init"), (15, "prod_after_next")]:
            v = np.where(t16[:, j] > 0, (t16[:, j] - t0) / 1000.0, np.nan)
            print(f"   {nm:16s} min={np.nanmin(v):8.2f} med={np.nanmedian(v):8.2f} max={np.nanmax(v):8.2f} us")
    cyc = t16[:, 8:16]
    cn = ["(first_W_issue)", "mma_wait_afull", "mma_wait_full", "mma_total", "conv_wait_full", "conv_wait_aempty", "conv_total", "mma_issue"]
    for j, nm in enumerate(cn):
        print(f"   cyc {nm:18s} med={np.median(cyc[:, j]):9.0f}")
    t2all = tr.cpu().numpy()[plan["ctas"] * 16 + 512:].reshape(-1, 16).astype(np.int64)
    if os.environ.get("ACC_WAIT") and plan["mode"] != "split-k-dsmem":
        print(f"   cyc {'mma_wait_accempty':18s} med={np.median(t2all[:plan['ctas'], 15]):9.0f}")
        print(f"   cyc {'mma_fence_after':18s} med={np.median(t2all[:plan['ctas'], 13]):9.0f}")
        print(f"   cyc {'mma_iter_sum':18s} med={np.median(t2all[:plan['ctas'], 14]):9.0f}")
    del W, X, qw, rot
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
            print(f"   {c:4d} " + " ".join(f"{v:7.2f}" for v in rel2[c, :16]))
        if os.environ.get("RAW_COLS"):
            cols = [int(v) for v in os.environ["RAW_COLS"].split(",")]
            print("   raw values (cycles) of trace2 cols", cols)
            for c in order[:12]:
                print(f"   {c:4d} " + " ".join(f"{t2[c, j]:10d}" for j in cols))
