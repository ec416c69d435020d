"""Column-parallel FFN across the GPUs of one node (bench.py --gpus N, launched by torchrun).

One process per GPU.  Every rank quantizes the full FFN weights with
fireq_quantize_weight (deterministic, so CAS lambda and PTS n are identical on all
ranks) and keeps its N-shard (sharding.py).  A decode step on rank r:

  fireq_quantize_act(x, c_gu)                         replicated (bit-identical on all ranks)
  fireq_w4a8_gemm_colpar_p2p(W_gu shard r) -> GU^T    the epilogue stores the rank's slice into
                                                      every rank's symmetric buffer (NVLink)
  fireq_silu_mul_quantize_act_t(GU^T)                 replicated
  fireq_w4a8_gemm_colpar_p2p(W_down shard r) -> Y^T   same

The only data-path exchange is the output gather (north_star (d)), fused into the GEMM
epilogue; the same step with the NCCL in-place all-gather
(fireq_w4a8_gemm_colpar, libfireq's own NCCL communicator) is timed alongside.
torch.distributed is plumbing only: handle exchange, barriers, max-over-ranks timing.
"""
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

from . import sharding

D_MODEL, D_FF = 4096, 11008


def run_colpar_bench(args, rank, world, dev, F, stream, peaks, peak_src, clock_cls=None):
    import synth
    M = 16
    R = 4
    uid = F.Comm.unique_id() if rank == 0 else None
    box = [uid]
    dist.broadcast_object_list(box, src=0)
    comm = F.Comm(world, rank, box[0])

    wg = synth.weights(D_FF, D_MODEL, synth.layer_seed(1, 0))
    wu = synth.weights(D_FF, D_MODEL, synth.layer_seed(1, 1))
    wd = synth.weights(D_MODEL, D_FF, synth.layer_seed(1, 2))
    W_gu = synth.bits_to_torch(np.concatenate([wg, wu], axis=0)).to(dev)
    W_d = synth.bits_to_torch(wd).to(dev)
    q_gu = F.quantize_weight(W_gu, cas_mode=1)
    q_d = F.quantize_weight(W_d, cas_mode=1)
    n_gu, n_d = q_gu.n, q_d.n
    del W_gu, W_d
    plan_gu = sharding.ShardPlan(2 * D_FF, world)
    plan_d = sharding.ShardPlan(D_MODEL, world)
    zeros_u8 = lambda n: torch.zeros(n, dtype=torch.uint8, device=dev)
    gamma_full = torch.cat([torch.ones(D_FF, device=dev), q_d.c.float()])
    gamma_l = sharding.shard_vector(gamma_full, plan_gu, rank, lambda n: torch.ones(n, device=dev))
    rot = []
    for _ in range(R):
        pg, sg = sharding.shard_quantized(q_gu.packed, q_gu.scales, plan_gu, rank, D_MODEL, zeros_u8)
        pd, sd = sharding.shard_quantized(q_d.packed, q_d.scales, plan_d, rank, D_FF, zeros_u8)
        rot.append((pg, sg, pd, sd))
    def exchange(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    symm_gu = F.Symmetric(world, rank, plan_gu.N_local, M, exchange, device=dev)
    symm_d = F.Symmetric(world, rank, plan_d.N_local, M, exchange, device=dev)
    x = synth.bits_to_torch(synth.activations(M, D_MODEL, synth.layer_seed(1, 3))).to(dev)
    xq = torch.empty((M, D_MODEL), dtype=torch.uint8, device=dev)
    beta = torch.empty(M, dtype=torch.bfloat16, device=dev)
    gut = torch.empty((plan_gu.N_pad, M), dtype=torch.bfloat16, device=dev)
    hq = torch.empty((M, D_FF), dtype=torch.uint8, device=dev)
    hbeta = torch.empty(M, dtype=torch.bfloat16, device=dev)
    yt = torch.empty((plan_d.N_pad, M), dtype=torch.bfloat16, device=dev)
    ws1 = F.Workspace(F.gemm_workspace_bytes(M, plan_gu.N_local, D_MODEL), dev)
    ws2 = F.Workspace(F.gemm_workspace_bytes(M, plan_d.N_local, D_FF), dev)

    def step_nccl(r):
        pg, sg, pd, sd = rot[r]
        F.quantize_act(x, chan_mul=q_gu.c, out=(xq, beta), stream=stream)
        F.w4a8_gemm_colpar(xq, beta, pg, sg, plan_gu.N_local, n_gu, comm, gut, ws1, gamma_local=gamma_l,
                           stream=stream)
        F.silu_mul_quantize_act_t(gut[:D_FF], gut[D_FF:2 * D_FF], M, D_FF, out=(hq, hbeta), stream=stream)
        F.w4a8_gemm_colpar(hq, hbeta, pd, sd, plan_d.N_local, n_d, comm, yt, ws2, stream=stream)

    def step(r, xin=None):
        pg, sg, pd, sd = rot[r]
        F.quantize_act(x if xin is None else xin, chan_mul=q_gu.c, out=(xq, beta), stream=stream)
        g = F.w4a8_gemm_colpar_p2p(xq, beta, pg, sg, plan_gu.N_local, n_gu, symm_gu, ws1, gamma_local=gamma_l,
                                   stream=stream)
        F.silu_mul_quantize_act_t(g[:D_FF], g[D_FF:2 * D_FF], M, D_FF, out=(hq, hbeta), stream=stream)
        F.w4a8_gemm_colpar_p2p(hq, hbeta, pd, sd, plan_d.N_local, n_d, symm_d, ws2, stream=stream)

    with torch.cuda.stream(stream):
        for r in range(R):
            step(r)
    torch.cuda.synchronize()
    graphed = True
    try:
        g_multi = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_multi, stream=stream):
            for r in range(R):
                step(r)
        replay = lambda: g_multi.replay()
        per_call = R
    except Exception as e:                      # NCCL capture unsupported: eager launches
        graphed = False
        print(f"[rank {rank}] graph capture failed ({e}); timing eager launches", file=sys.stderr)
        replay = lambda: [step(r) for r in range(R)]
        per_call = R
    calls = max(1, args.steps // per_call)
    steps = calls * per_call
    for _ in range(max(1, args.warmup // per_call)):
        with torch.cuda.stream(stream):
            replay()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = clock_cls(dev.index or 0) if (clock_cls is not None and rank == 0) else None
    if clocks:
        # a longer pass under the clock sampler (nvidia-smi polls every ~0.1 s), then the timed K
        clocks.start()
        time.sleep(0.25)
        with torch.cuda.stream(stream):
            for _ in range(max(calls, 20000 // per_call)):
                replay()
        torch.cuda.synchronize()
        clocks.stop()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(calls):
            replay()
        e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    us_per_step = float(ms.item()) * 1e3 / steps

    # end to end through host buffers: pinned H2D of each step's x and D2H of the gathered y
    # every step.  The uploads run ahead on their own stream into per-step device buffers (x is
    # rank-local); the download stays on the compute stream: peers write this rank's Y^T in
    # the next step, so it must be read before that step starts.
    x_hosts = [(x * (1 + 0.25 * r)).cpu().pin_memory() for r in range(R)]
    xds = [torch.empty_like(x) for _ in range(R)]
    y_host = torch.empty_like(yt, device="cpu").pin_memory()
    s_h2d = torch.cuda.Stream(device=dev)

    def e2e_steps(rs):
        fork = torch.cuda.Event()
        fork.record(stream)
        s_h2d.wait_event(fork)
        done = []
        with torch.cuda.stream(s_h2d):
            for i, r in enumerate(rs):
                xds[i].copy_(x_hosts[r], non_blocking=True)
                done.append(torch.cuda.Event())
                done[i].record(s_h2d)
        for i, r in enumerate(rs):
            stream.wait_event(done[i])
            step(r, xds[i])
            y_host.copy_(symm_d.yt, non_blocking=True)
        stream.wait_stream(s_h2d)

    def e2e_step(r):
        e2e_steps([r])

    with torch.cuda.stream(stream):
        for r in range(R):
            e2e_step(r)
    torch.cuda.synchronize()
    e2e_graphed = False
    if graphed:
        # the same R steps with their copies as one CUDA graph (as the device timing)
        try:
            g_e2e = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_e2e, stream=stream):
                e2e_steps(list(range(R)))
            e2e_graphed = True
        except Exception as e:
            print(f"[rank {rank}] e2e graph capture failed ({e}); timing eager launches", file=sys.stderr)
    dist.barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e2.record(stream)
        if e2e_graphed:
            for _ in range(steps // R):
                g_e2e.replay()
        else:
            for i in range(steps):
                e2e_step(i % R)
        e3.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms2 = torch.tensor([e2.elapsed_time(e3)], device=dev)
    dist.all_reduce(ms2, op=dist.ReduceOp.MAX)
    e2e_us = float(ms2.item()) * 1e3 / steps

    # the same step with the NCCL in-place all-gathers (fireq_w4a8_gemm_colpar), for comparison
    nccl_us = None
    try:
        g_n = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            for r in range(R):
                step_nccl(r)
        torch.cuda.synchronize()
        with torch.cuda.graph(g_n, stream=stream):
            for r in range(R):
                step_nccl(r)
        with torch.cuda.stream(stream):
            g_n.replay()
        torch.cuda.synchronize()
        dist.barrier()
        e6, e7 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e6.record(stream)
            for _ in range(calls):
                g_n.replay()
            e7.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        ms3 = torch.tensor([e6.elapsed_time(e7)], device=dev)
        dist.all_reduce(ms3, op=dist.ReduceOp.MAX)
        nccl_us = float(ms3.item()) * 1e3 / steps
        del g_n
    except Exception as e:
        print(f"[rank {rank}] NCCL comparison skipped: {e}", file=sys.stderr)
    # BASELINE configs[3]: Llama2-70B FFN column-parallel at M = 16 and M = 16384
    from .c4 import c4_figures
    c4 = c4_figures(F, dev, stream, rank, world, comm, exchange=exchange) if not getattr(args, "no_c4", False) else None
    comm.destroy()
    symm_gu.close()
    symm_d.close()

    # dominant kernel: this rank's gate_up shard GEMM alone (no collective), rotating copies
    gu_out = torch.empty((M, plan_gu.N_local), dtype=torch.bfloat16, device=dev)

    def gu_only(r):
        pg, sg, _, _ = rot[r]
        F.w4a8_gemm(xq, beta, pg, sg, plan_gu.N_local, n_gu, gamma=gamma_l, out=gu_out, workspace=ws1, stream=stream)

    with torch.cuda.stream(stream):
        for r in range(R):
            gu_only(r)
    torch.cuda.synchronize()
    g_gu = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_gu, stream=stream):
        for r in range(R):
            gu_only(r)
    with torch.cuda.stream(stream):
        g_gu.replay()
    torch.cuda.synchronize()
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    with torch.cuda.stream(stream):
        e4.record(stream)
        for _ in range(reps):
            g_gu.replay()
        e5.record(stream)
    torch.cuda.synchronize()
    gu_us = e4.elapsed_time(e5) * 1e3 / (reps * R)
    Nl = plan_gu.N_local
    gu_bytes = Nl * D_MODEL // 2 + Nl * D_MODEL // 128 + M * D_MODEL + 2 * M + 2 * M * Nl
    if rank == 0:
        line = {
            "metric": "Llama2-7B FFN latency at batch 16 (W4A8-FP: INT4 weights + FP8 g128 scales, FP8 activations)",
            "value": round(us_per_step, 3), "unit": "us", "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": round(us_per_step / 1e3, 6), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp8e4m3 x int4 -> f32 acc -> bf16", "data": "synthetic",
            "config": {"workload": "llama2-7b-ffn-decode-b16", "tokens": M, "d_model": D_MODEL, "d_ff": D_FF,
                       "parallelism": f"column-parallel tp{world} (N-sharded gate_up + down; Y^T gathered by the "
                                      "GEMM epilogue's NVLink stores into every rank's buffer, CUDA IPC)",
                       "l2": f"{R} rotating weight-shard copies", "graph": "captured" if graphed else "eager"},
            "gpu_launches": 4 * steps,
            "e2e": {"value": round(e2e_us, 3), "unit": "us", "h2d_bytes_per_step": x.numel() * 2,
                    "d2h_bytes_per_step": yt.numel() * 2,
                    "timing": ("CUDA graph of the steps with their copies (uploads on their own stream)"
                               if e2e_graphed else "eager launches")
                              + ", max over ranks"},
        }
        if clocks:
            line["clocks"] = clocks.summary()
        if c4:
            line["c4_llama2_70b_ffn"] = c4
        if nccl_us is not None:
            line["nccl_allgather_variant_us"] = round(nccl_us, 3)
        hbm = peaks["hbm_gbs"]
        line["roofline"] = {"bound": "hbm", "kernel": f"fireq_w4a8_gemm gate_up shard M={M} N={Nl} K={D_MODEL} (per rank)",
                            "achieved": round(gu_bytes / gu_us / 1e3, 1), "peak": hbm, "unit": "GB/s",
                            "frac": round(gu_bytes / gu_us / 1e3 / hbm, 4), "traffic": None,
                            "algorithmic_bytes": gu_bytes, "launch_us": round(gu_us, 3),
                            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})"}
        print(json.dumps(line), flush=True)
