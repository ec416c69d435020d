"""BASELINE configs C1, C3 and C5 on one B200: rooflines of fireq_w4a8_gemm.

  C1  q_proj shape M=16, N=K=4096: quantize_weight + quantize_act + GEMM, single-shot and graph
  C3  Llama3-8B linear layers (q, k, v, o, gate, up, down) at prefill M = 16 x 1024
  C5  M sweep 1 .. 16384 on the Llama3-8B down_proj (N=4096, K=14336)

Each GEMM is timed as a CUDA graph of back-to-back launches over rotating weight copies
(> 2 x L2 for the HBM-bound shapes), CUDA events.  Writes one JSON document to stdout.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2505_20839_b200 import fireq as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 7672.0, "bf16_tflops": 2250.0}
HBM = peaks["hbm_gbs"]
FP8 = 2.0 * peaks["bf16_tflops"]


def gemm_bytes(M, N, K):
    return N * K // 2 + N * K // 128 + M * K + 2 * M + 2 * M * N


_wcache = {}


def weights(N, K):
    if (N, K) not in _wcache:
        _wcache.clear()
        torch.cuda.empty_cache()
        W = synth.bits_to_torch(synth.weights(N, K, synth.layer_seed(5, N % 97))).cuda()
        _wcache[(N, K)] = F.quantize_weight(W, 1)
        del W
    return _wcache[(N, K)]


def time_gemm(M, N, K, launches=24):
    qw = weights(N, K)
    X = synth.bits_to_torch(synth.activations(M, K, synth.layer_seed(5, 1000 + M % 89))).cuda()
    xq, beta = F.quantize_act(X, chan_mul=qw.c)
    wbytes = N * K // 2
    rot_n = max(1, min(8, -(-300_000_000 // wbytes))) if M <= 1024 else 1
    rot = [(qw.packed, qw.scales)] + [(qw.packed.clone(), qw.scales.clone()) for _ in range(rot_n - 1)]
    ws = F.Workspace(F.gemm_workspace_bytes(M, N, K))
    out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.Stream()
    n_rep = max(1, launches // rot_n) if M <= 1024 else 3
    def run():
        for p, sc in rot:
            F.w4a8_gemm(xq, beta, p, sc, N, qw.n, out=out, workspace=ws, stream=s)
    with torch.cuda.stream(s):
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n_rep):
            run()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10 if M <= 1024 else 2
    e0.record()                      # replay() launches on the current stream
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * n_rep * rot_n)
    b, fl = gemm_bytes(M, N, K), 2.0 * M * N * K
    t_mem, t_fp8 = b / (HBM * 1e3), fl / (FP8 * 1e6)          # us at 100 %
    bound = "hbm" if t_mem >= t_fp8 else "tensor"
    r = {"M": M, "N": N, "K": K, "us": round(us, 3), "gbs": round(b / us / 1e3, 1),
         "tflops": round(fl / us / 1e6, 1), "bound": bound,
         "frac": round(max(t_mem, t_fp8) / us, 4), "plan": F.gemm_plan(M, N, K), "weight_copies": rot_n}
    del rot, ws, out, g, X, xq, beta
    return r


def c1():
    M, N, K = 16, 4096, 4096
    W = synth.bits_to_torch(synth.weights(N, K, synth.layer_seed(1, 7))).cuda()
    X = synth.bits_to_torch(synth.activations(M, K, synth.layer_seed(1, 8))).cuda()
    for _ in range(2):
        qw = F.quantize_weight(W, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    qw = F.quantize_weight(W, 1)
    e1.record()
    torch.cuda.synchronize()
    qw_us = e0.elapsed_time(e1) * 1e3
    xq, beta = F.quantize_act(X, chan_mul=qw.c)
    out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    ws = F.Workspace(F.gemm_workspace_bytes(M, N, K))
    n = qw.n
    # single shot: act quant + GEMM, cold weights (L2 flushed by a 256 MB write first)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    shots = []
    for i in range(5):
        flush.fill_(i)
        torch.cuda.synchronize()
        e0.record()
        F.quantize_act(X, chan_mul=qw.c, out=(xq, beta))
        F.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, n, out=out, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        shots.append(e0.elapsed_time(e1) * 1e3)
    del flush
    g = time_gemm(M, N, K)
    return {"config": "C1 q_proj M=16 N=K=4096", "quantize_weight_us": round(qw_us, 1),
            "act_quant_plus_gemm_single_shot_us_median": round(sorted(shots)[2], 2),
            "gemm_graph": g}


def main():
    torch.cuda.init()
    doc = {"device": torch.cuda.get_device_name(0), "hbm_gbs_peak": HBM, "fp8_tflops_peak": FP8,
           "peak_source": "MEASURED_PEAKS.json (hbm_gbs; fp8 = 2 x bf16_tflops burst)",
           "timing": "CUDA graph of back-to-back launches over rotating weight copies, CUDA events"}
    doc["C1"] = c1()
    print(json.dumps(doc["C1"]), file=sys.stderr, flush=True)
    layers = [("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
              ("gate", 14336, 4096), ("up", 14336, 4096), ("down", 4096, 14336)]
    M = 16384
    c3, tot_us, tot_fl = [], 0.0, 0.0
    for name, N, K in layers:
        r = time_gemm(M, N, K)
        r["layer"] = name
        c3.append(r)
        tot_us += r["us"]
        tot_fl += 2.0 * M * N * K
        print(json.dumps(r), file=sys.stderr, flush=True)
    doc["C3"] = {"config": "Llama3-8B linear layers, prefill M = 16 x 1024", "layers": c3,
                 "layer_total_us": round(tot_us, 1), "layer_tflops": round(tot_fl / tot_us / 1e6, 1),
                 "layer_frac_fp8": round(tot_fl / tot_us / 1e6 / FP8, 4)}
    c5 = []
    for e in range(15):
        r = time_gemm(2 ** e, 4096, 14336)
        c5.append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
    doc["C5"] = {"config": "M sweep on Llama3-8B down_proj N=4096 K=14336", "points": c5}
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
