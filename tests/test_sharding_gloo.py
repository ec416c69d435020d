"""Column-parallel host logic (sharding.py) on CPU, including a world_size-2 gloo run.

The CUDA GEMM cannot run here; each rank computes its shard's Y^T with the CPU oracle
(test infrastructure) and the shards are all-gathered with torch.distributed/gloo in
the same rank-major order the in-place NCCL all-gather uses on the GPUs.  The gathered
Y^T must equal the oracle's unsharded result exactly (same arithmetic per element), and
shard bytes must be byte slices of the full layout-v1 packing.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import gemm as og
from oracle import layout as ol
from oracle import quant as oq
from paper_2505_20839_b200 import sharding


def test_shard_plan():
    p = sharding.ShardPlan(22016, 8)           # 172 tiles -> 22 per rank, 4 padded
    assert p.N_local == 22 * 128 and p.N_pad == 176 * 128
    assert p.rows(7) == (7 * 2816, 22016)
    p = sharding.ShardPlan(4096, 4)
    assert p.N_local == 1024 and p.rows(3) == (3072, 4096)
    p = sharding.ShardPlan(256, 4)             # fewer tiles than ranks -> empty shards
    assert p.rows(3) == (256, 256)
    with pytest.raises(ValueError):
        sharding.ShardPlan(100, 2)


@pytest.mark.parametrize("N,K,P", [(512, 256, 2), (640, 384, 4), (384, 128, 8)])
def test_shard_bytes_are_slices_of_full_packing(N, K, P):
    W = synth.bits_to_f64(synth.weights(N, K, 5))
    q = oq.quantize_weight(W, 1)
    plan = sharding.ShardPlan(N, P)
    zeros = lambda n: torch.zeros(n, dtype=torch.uint8)
    for r in range(P):
        pl, sl = sharding.shard_quantized(torch.from_numpy(q.packed), torch.from_numpy(q.scales), plan, r, K, zeros)
        a, b = plan.rows(r)
        if b > a:
            # packing the row slice on its own (same codes, same scales) gives the same bytes
            assert np.array_equal(pl.numpy()[: (b - a) * K // 2], ol.pack_codes(q.codes[a:b]))
            assert np.array_equal(sl.numpy()[: (b - a) * K // 128], ol.pack_scales(q.sigma_codes[a:b]))
        assert not pl.numpy()[(b - a) * K // 2:].any() and not sl.numpy()[(b - a) * K // 128:].any()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, N, K, M, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = synth.bits_to_f64(synth.weights(N, K, 9))
        X = synth.bits_to_f64(synth.activations(M, K, 10))
        q = oq.quantize_weight(W, 1)                      # full tensor on every rank (global CAS / PTS)
        xq, beta = oq.quantize_act(X, q.c)                # replicated activations
        plan = sharding.ShardPlan(N, world)
        zeros = lambda n: torch.zeros(n, dtype=torch.uint8)
        pl, sl = sharding.shard_quantized(torch.from_numpy(q.packed), torch.from_numpy(q.scales), plan, rank, K,
                                          zeros)
        # this rank's Y^T slice [N_local][M] (oracle stands in for the CUDA GEMM)
        r_local = og.gemm_reference(xq, beta, pl.numpy(), sl.numpy(), plan.N_local, K, q.n)
        yt_local = torch.from_numpy(np.ascontiguousarray(r_local.T))
        yt_full = torch.empty((plan.N_pad, M), dtype=torch.float64)
        dist.all_gather_into_tensor(yt_full, yt_local)
        if rank == 0:
            ref = og.gemm_reference(xq, beta, q.packed, q.scales, N, K, q.n)
            out.put((yt_full[:N].numpy().T.copy(), ref, yt_full[N:].numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,world", [(384, 2), (640, 2)])
def test_colpar_gather_gloo_world2(N, world):
    K, M = 256, 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, K, M, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, ref, pad = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got, ref)
    assert not pad.any()                                   # padded rows produce zeros
