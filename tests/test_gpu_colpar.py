"""GPU tests of the column-parallel layer (north_star (d)) on one B200.

* fireq_w4a8_gemm_colpar through a real NCCL communicator of world size 1 (the in-place
  all-gather is still issued) equals the single-GPU GEMM's Y^T bit for bit.
* P "ranks" simulated on one GPU: each shard (byte slices of the full packing,
  sharding.shard_quantized) runs the same Y^T GEMM into its slot of the full Y^T, exactly
  what a rank does before the all-gather.  When every tile is reduced whole (prefill
  plans), the gathered Y^T equals the 1-GPU result bit for bit (SURVEY 8(e) invariant);
  at decode the K-split of a tile depends on N_local (stream-K / cluster split-K), so the
  shards agree with the 1-GPU result up to FP32 summation order (DESIGN reading R24) and
  both satisfy G4 against the oracle.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import gemm as og
from oracle import quant as oq
from paper_2505_20839_b200 import sharding

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _setup(fireq, M, N, K, seed):
    wb = synth.weights(N, K, seed)
    xb = synth.activations(M, K, seed + 1)
    qw = fireq.quantize_weight(synth.bits_to_torch(wb).to(DEV), cas_mode=1)
    xq, beta = fireq.quantize_act(synth.bits_to_torch(xb).to(DEV), chan_mul=qw.c)
    return wb, xb, qw, xq, beta


@pytest.mark.parametrize("M", [16, 5])
def test_colpar_nccl_world1(fireq, M):
    N, K = 1024, 2048
    _, _, qw, xq, beta = _setup(fireq, M, N, K, 1201)
    comm = fireq.Comm(1, 0, fireq.Comm.unique_id())
    try:
        ws = fireq.Workspace(fireq.gemm_workspace_bytes(M, N, K))
        yt_full = torch.full((N, M), float("nan"), dtype=torch.bfloat16, device=DEV)
        fireq.w4a8_gemm_colpar(xq, beta, qw.packed, qw.scales, N, qw.n, comm, yt_full, ws)
        ref = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, out_layout=1)
        torch.cuda.synchronize()
        assert torch.equal(yt_full, ref)
    finally:
        comm.destroy()


def _simulated_ranks(fireq, qw, xq, beta, N, K, P, gamma=None):
    M = xq.shape[0]
    plan = sharding.ShardPlan(N, P)
    yt = torch.empty((plan.N_pad, M), dtype=torch.bfloat16, device=DEV)
    for r in range(P):
        pl, sl = sharding.shard_quantized(qw.packed, qw.scales, plan, r, K,
                                          lambda n: torch.zeros(n, dtype=torch.uint8, device=DEV))
        g = None
        if gamma is not None:
            g = sharding.shard_vector(gamma, plan, r, lambda n: torch.ones(n, dtype=torch.float32, device=DEV))
        fireq.w4a8_gemm(xq, beta, pl, sl, plan.N_local, qw.n, gamma=g,
                        out=yt[r * plan.N_local:(r + 1) * plan.N_local], out_layout=1)
    return yt[:N]


@pytest.mark.parametrize("P", [2, 4, 8])
def test_shards_bitwise_equal_single_gpu_prefill(fireq, P):
    """M = 8192: every plan (P = 1 and each shard) reduces whole tiles, so the gathered Y^T
    is the 1-GPU Y^T bit for bit; N = 8192 with P = 8 leaves N_local = 1024."""
    M, N, K = 8192, 8192, 512
    _, _, qw, xq, beta = _setup(fireq, M, N, K, 1301)
    gamma = torch.rand(N, device=DEV) + 0.5
    assert fireq.gemm_plan(M, N // P, K)["mode"] == "tiles"
    assert fireq.gemm_plan(M, N, K)["mode"] == "tiles"
    full = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, gamma=gamma, out_layout=1)
    got = _simulated_ranks(fireq, qw, xq, beta, N, K, P, gamma)
    torch.cuda.synchronize()
    assert torch.equal(got, full)


@pytest.mark.parametrize("P,N", [(2, 3072), (4, 3072), (8, 8192), (3, 1280)])
def test_shards_decode_vs_oracle(fireq, P, N):
    """Decode M = 16: shards (zero-padded when N/128 is not a multiple of P) against the
    oracle (G4) and against the 1-GPU result (same tolerance)."""
    M, K = 16, 1024
    wb, xb, qw, xq, beta = _setup(fireq, M, N, K, 1401 + P)
    full = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, out_layout=1)
    got = _simulated_ranks(fireq, qw, xq, beta, N, K, P)
    torch.cuda.synchronize()
    ref = oq.quantize_weight(synth.bits_to_f64(wb), 1)
    rq, rbeta = oq.quantize_act(synth.bits_to_f64(xb), ref.c)
    r = og.gemm_reference(rq, rbeta, ref.packed, ref.scales, N, K, ref.n)
    y = got.t().float().cpu().numpy().astype(np.float64)
    yf = full.t().float().cpu().numpy().astype(np.float64)
    assert og.g4_error(y, r) <= 1e-2
    assert og.g4_error(y, yf) <= 1e-2


# ----------------------------------------------- comm-fused column parallelism (f2)
def test_colpar_p2p_world1(fireq):
    """fireq_w4a8_gemm_colpar_p2p at one rank: the epilogue's Y^T in the symmetric buffer equals the
    plain GEMM's Y^T bit for bit (no signalling at world size 1)."""
    M, N, K = 16, 1024, 2048
    _, _, qw, xq, beta = _setup(fireq, M, N, K, 1601)
    symm = fireq.Symmetric(1, 0, N, M, exchange=lambda obj: [obj])
    try:
        ws = fireq.Workspace(fireq.gemm_workspace_bytes(M, N, K))
        yt = fireq.w4a8_gemm_colpar_p2p(xq, beta, qw.packed, qw.scales, N, qw.n, symm, ws)
        ref = fireq.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, out_layout=1)
        torch.cuda.synchronize()
        assert torch.equal(yt, ref)
    finally:
        symm.close()


def _p2p_rank(rank, world, port, M, N, K, out_dir):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from paper_2505_20839_b200 import fireq as F
    from paper_2505_20839_b200 import sharding as sh
    F.load()
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        wb = synth.weights(N, K, 1701)
        xb = synth.activations(M, K, 1702)
        qw = F.quantize_weight(synth.bits_to_torch(wb).cuda(), cas_mode=1)
        xq, beta = F.quantize_act(synth.bits_to_torch(xb).cuda(), chan_mul=qw.c)
        plan = sh.ShardPlan(N, world)
        pl, sl = sh.shard_quantized(qw.packed, qw.scales, plan, rank, K,
                                    lambda n: torch.zeros(n, dtype=torch.uint8, device="cuda"))

        def exchange(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out

        symm = F.Symmetric(world, rank, plan.N_local, M, exchange)
        ws = F.Workspace(F.gemm_workspace_bytes(M, plan.N_local, K))
        ref = F.w4a8_gemm(xq, beta, qw.packed, qw.scales, N, qw.n, out_layout=1)
        s = torch.cuda.Stream()
        ok = []
        for it in range(3):                       # repeated calls: the epochs advance
            with torch.cuda.stream(s):
                symm.yt.zero_()
                torch.cuda.synchronize()          # zeroed before the peer's stores can arrive
                dist.barrier()
                yt = F.w4a8_gemm_colpar_p2p(xq, beta, pl, sl, plan.N_local, qw.n, symm, ws, stream=s)
            torch.cuda.synchronize()
            ok.append(yt[:N].clone())
            dist.barrier()
        # graph capture: replays advance the device-side epochs
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            F.w4a8_gemm_colpar_p2p(xq, beta, pl, sl, plan.N_local, qw.n, symm, ws, stream=s)
        for it in range(2):
            symm.yt.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            g.replay()
            torch.cuda.synchronize()
            ok.append(symm.yt[:N].clone())
            dist.barrier()
        whole = F.gemm_plan(M, N, K)["mode"] == "tiles" and F.gemm_plan(M, plan.N_local, K)["mode"] == "tiles"
        res = []
        for y in ok:
            if whole:
                res.append(bool(torch.equal(y, ref)))
            else:
                a = y.t().float().cpu().numpy().astype(np.float64)
                b = ref.t().float().cpu().numpy().astype(np.float64)
                res.append(og.g4_error(a, b) <= 1e-2 and not torch.isnan(y.float()).any().item())
        symm.close()
        with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as f:
            f.write("ok" if all(res) else f"fail {res}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,N,K", [(16, 3072, 1024), (8192, 4096, 256)])
def test_colpar_p2p_two_ranks_one_gpu(fireq, tmp_path, M, N, K):
    """Two processes on one GPU (CUDA IPC works between processes of the same device): each rank's
    epilogue stores its Y^T slice into both symmetric buffers and the flags complete the exchange;
    both ranks hold the single-GPU Y^T (bitwise for whole-tile plans, else G4), across repeated
    calls and CUDA-graph replays."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_p2p_rank, args=(r, 2, port, M, N, K, str(tmp_path))) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    for r in range(2):
        assert (tmp_path / f"rank{r}.txt").read_text() == "ok"
