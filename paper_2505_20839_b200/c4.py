"""BASELINE configs[3]: the Llama2-70B FFN (gate/up 8192 -> 28672,
down 28672 -> 8192) column-parallel over the P ranks of one node, at decode M = 16 and
prefill M = 16384.

Per P (= world size) and M it reports, from rank 0 (times are max over ranks):
  gemm_only_us   the rank's two shard GEMMs (gate_up shard with gamma, down shard) plus the
                 replicated activation quantizers, without the collectives
  gemm_ag_us     the full column-parallel FFN step: the same kernels plus the two in-place
                 NCCL all-gathers of Y^T (fireq_w4a8_gemm_colpar)
  gemm_p2p_us    the step with the gathers fused into the GEMM epilogues (NVLink stores into
                 every rank's symmetric buffer + epoch flags, fireq_w4a8_gemm_colpar_p2p)
  ag_busbw_gbs   the two all-gathers alone (same sizes, NCCL): bus bandwidth
                 bytes * (P - 1) / P / time
  vs_p1          rank 0 computes the single-GPU FFN output from the full weights (every rank
                 quantizes the full weight, so CAS lambda / PTS n are global) and compares it
                 with the gathered output: bitwise when every tile is reduced whole (prefill),
                 else the G4 distance (K-split points depend on N / P, DESIGN reading R24)
The weights are synthetic (synth/), the shards byte slices of the full packing (sharding.py).
"""
import numpy as np
import torch

from . import sharding

D_MODEL, D_FF = 8192, 28672


def _events(stream, fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        fn()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def _max_over_ranks(v, dev, world):
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _g4(y, r):
    rms = np.sqrt(np.mean(r * r, axis=1, keepdims=True))
    den = np.maximum(np.abs(r), 0.1 * rms)
    return float(np.max(np.abs(y - r) / np.where(den > 0, den, 1.0)))


def c4_figures(F, dev, stream, rank, world, comm=None, Ms=(16, 16384), exchange=None):
    import synth
    wg = synth.weights(D_FF, D_MODEL, synth.layer_seed(3, 0))
    wu = synth.weights(D_FF, D_MODEL, synth.layer_seed(3, 1))
    W_gu = synth.bits_to_torch(np.concatenate([wg, wu], axis=0)).to(dev)
    del wg, wu
    q_gu = F.quantize_weight(W_gu, cas_mode=1)
    del W_gu
    W_d = synth.bits_to_torch(synth.weights(D_MODEL, D_FF, synth.layer_seed(3, 2))).to(dev)
    q_d = F.quantize_weight(W_d, cas_mode=1)
    del W_d
    torch.cuda.empty_cache()
    n_gu, n_d = q_gu.n, q_d.n
    P = world
    pg_plan, pd_plan = sharding.ShardPlan(2 * D_FF, P), sharding.ShardPlan(D_MODEL, P)
    z8 = lambda n: torch.zeros(n, dtype=torch.uint8, device=dev)
    gamma_full = torch.cat([torch.ones(D_FF, device=dev), q_d.c.float()])
    gamma_l = sharding.shard_vector(gamma_full, pg_plan, rank, lambda n: torch.ones(n, device=dev))
    pg, sg = sharding.shard_quantized(q_gu.packed, q_gu.scales, pg_plan, rank, D_MODEL, z8)
    pd, sd = sharding.shard_quantized(q_d.packed, q_d.scales, pd_plan, rank, D_FF, z8)
    out = {"workload": "llama2-70b-ffn-column-parallel", "d_model": D_MODEL, "d_ff": D_FF, "tp": P,
           "N_local": {"gate_up": pg_plan.N_local, "down": pd_plan.N_local}}
    for M in Ms:
        x = synth.bits_to_torch(synth.activations(M, D_MODEL, synth.layer_seed(3, 3 + M))).to(dev)
        xq = torch.empty((M, D_MODEL), dtype=torch.uint8, device=dev)
        beta = torch.empty(M, dtype=torch.bfloat16, device=dev)
        gut = torch.empty((pg_plan.N_pad, M), dtype=torch.bfloat16, device=dev)
        hq = torch.empty((M, D_FF), dtype=torch.uint8, device=dev)
        hbeta = torch.empty(M, dtype=torch.bfloat16, device=dev)
        yt = torch.empty((pd_plan.N_pad, M), dtype=torch.bfloat16, device=dev)
        ws1 = F.Workspace(F.gemm_workspace_bytes(M, pg_plan.N_local, D_MODEL), dev)
        ws2 = F.Workspace(F.gemm_workspace_bytes(M, pd_plan.N_local, D_FF), dev)
        gl = gut[rank * pg_plan.N_local:(rank + 1) * pg_plan.N_local]
        yl = yt[rank * pd_plan.N_local:(rank + 1) * pd_plan.N_local]

        def gemm_only():
            F.quantize_act(x, chan_mul=q_gu.c, out=(xq, beta), stream=stream)
            F.w4a8_gemm(xq, beta, pg, sg, pg_plan.N_local, n_gu, gamma=gamma_l, out=gl, out_layout=1,
                        workspace=ws1, stream=stream)
            F.silu_mul_quantize_act_t(gut[:D_FF], gut[D_FF:2 * D_FF], M, D_FF, out=(hq, hbeta), stream=stream)
            F.w4a8_gemm(hq, hbeta, pd, sd, pd_plan.N_local, n_d, out=yl, out_layout=1, workspace=ws2,
                        stream=stream)

        def gemm_ag():
            F.quantize_act(x, chan_mul=q_gu.c, out=(xq, beta), stream=stream)
            F.w4a8_gemm_colpar(xq, beta, pg, sg, pg_plan.N_local, n_gu, comm, gut, ws1, gamma_local=gamma_l,
                               stream=stream)
            F.silu_mul_quantize_act_t(gut[:D_FF], gut[D_FF:2 * D_FF], M, D_FF, out=(hq, hbeta), stream=stream)
            F.w4a8_gemm_colpar(hq, hbeta, pd, sd, pd_plan.N_local, n_d, comm, yt, ws2, stream=stream)

        reps = 20 if M <= 64 else 3
        rec = {}
        ex = exchange if exchange is not None else (lambda obj: [obj])
        symm_gu = F.Symmetric(world, rank, pg_plan.N_local, M, ex, device=dev)
        symm_d = F.Symmetric(world, rank, pd_plan.N_local, M, ex, device=dev)

        def gemm_p2p():
            F.quantize_act(x, chan_mul=q_gu.c, out=(xq, beta), stream=stream)
            g = F.w4a8_gemm_colpar_p2p(xq, beta, pg, sg, pg_plan.N_local, n_gu, symm_gu, ws1, gamma_local=gamma_l,
                                       stream=stream)
            F.silu_mul_quantize_act_t(g[:D_FF], g[D_FF:2 * D_FF], M, D_FF, out=(hq, hbeta), stream=stream)
            F.w4a8_gemm_colpar_p2p(hq, hbeta, pd, sd, pd_plan.N_local, n_d, symm_d, ws2, stream=stream)

        rec["gemm_only_us"] = round(_max_over_ranks(_events(stream, gemm_only, reps), dev, world), 2)
        if comm is not None:
            rec["gemm_ag_us"] = round(_max_over_ranks(_events(stream, gemm_ag, reps), dev, world), 2)
        rec["gemm_p2p_us"] = round(_max_over_ranks(_events(stream, gemm_p2p, reps), dev, world), 2)
        with torch.cuda.stream(stream):
            gemm_p2p()
        torch.cuda.synchronize()
        p2p_y = symm_d.yt[:D_MODEL].clone()
        if world > 1:
            import torch.distributed as dist

            def ag_only():
                dist.all_gather_into_tensor(gut, gl.contiguous(), async_op=False)
                dist.all_gather_into_tensor(yt, yl.contiguous(), async_op=False)

            t = _max_over_ranks(_events(stream, ag_only, reps), dev, world)
            nbytes = (gut.numel() + yt.numel()) * 2
            rec["ag_us"] = round(t, 2)
            rec["ag_busbw_gbs"] = round(nbytes * (P - 1) / P / (t * 1e-6) / 1e9, 1)
            # the same collectives timed above: recompute the outputs through the fireq path
            with torch.cuda.stream(stream):
                gemm_ag()
        else:
            with torch.cuda.stream(stream):
                gemm_only()
        torch.cuda.synchronize()
        flops = 2 * M * (2 * D_FF * D_MODEL + D_MODEL * D_FF)
        wbytes = (2 * D_FF * D_MODEL + D_MODEL * D_FF) * (0.5 + 1 / 128) / P
        rec["per_rank_weight_mb"] = round(wbytes / 1e6, 1)
        rec["tflops_total"] = round(flops / (rec.get("gemm_ag_us", rec["gemm_only_us"]) * 1e-6) / 1e12, 1)
        if rank == 0 and P > 1:
            # single-GPU reference from the full quantized weights (same inputs)
            ws_a = F.Workspace(F.gemm_workspace_bytes(M, 2 * D_FF, D_MODEL), dev)
            ws_b = F.Workspace(F.gemm_workspace_bytes(M, D_MODEL, D_FF), dev)
            with torch.cuda.stream(stream):
                F.quantize_act(x, chan_mul=q_gu.c, out=(xq, beta), stream=stream)
                g1 = F.w4a8_gemm(xq, beta, q_gu.packed, q_gu.scales, 2 * D_FF, n_gu, gamma=gamma_full,
                                 out_layout=1, workspace=ws_a, stream=stream)
                F.silu_mul_quantize_act_t(g1[:D_FF], g1[D_FF:], M, D_FF, out=(hq, hbeta), stream=stream)
                y1 = F.w4a8_gemm(hq, hbeta, q_d.packed, q_d.scales, D_MODEL, n_d, out_layout=1, workspace=ws_b,
                                 stream=stream)
            torch.cuda.synchronize()
            yg = yt[:D_MODEL]
            same = bool(torch.equal(yg, y1))
            rec["vs_p1_bitwise"] = same
            rec["p2p_equals_nccl"] = bool(torch.equal(p2p_y, yg))
            if not same:
                rows = torch.arange(0, M, max(1, M // 64), device=dev)
                a = yg[:, rows].t().float().cpu().numpy().astype(np.float64)
                b = y1[:, rows].t().float().cpu().numpy().astype(np.float64)
                rec["vs_p1_g4"] = round(_g4(a, b), 5)
            del ws_a, ws_b, g1, y1
        out[f"M{M}"] = rec
        symm_gu.close()
        symm_d.close()
        del x, xq, gut, hq, yt, ws1, ws2, p2p_y
        torch.cuda.empty_cache()
    return out
