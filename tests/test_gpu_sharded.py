"""The tree-sharded multi-GPU path end to end on one GPU: two
ranks (gloo over the same cuda:0 — NCCL refuses two ranks on one device)
each traverse, bucket and sketch their half of the trees; the (n, k) sketch
partials are all-reduced once per pass (proximity._Sketch.apply).  The
factorisation on the shards must reproduce the single-process result: the
same reconstruction P ~ Q Q^T and pmax within 1e-5 (shards regroup the f32
per-batch partial sums of the sketch), and dense row shards must concatenate
to the whole triangle bit for bit."""

import os
import socket

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_19493_b200 import _lib
        from paper_2511_19493_b200 import distributed as D
        from paper_2511_19493_b200 import proximity as P
        from paper_2511_19493_b200.dataset import from_arrays, make_synthetic
        from oracle.trainer import train
        from paper_2511_19493_b200.forest import TrainConfig
        X, y = make_synthetic(3000, 20, seed=2)
        ds = from_arrays(X, y)
        forest = train(ds, TrainConfig(ntree=24, iseed=3))
        lo, hi = D.tree_shard(forest.ntree, rank, world)
        shard = P.leaf_membership(forest, ds, trees=(lo, hi))
        lr = P.lowrank_proximity(shard, rank=8, mode="f32", seed=1)
        whole = P.leaf_membership(forest, ds)
        rlo, rhi = D.row_shard(ds.n, rank, world)
        rows = P.pair_counts_device(whole, _lib.UPPER_I32, rlo, rhi).cpu().numpy()
        out[rank] = (lr.dequantized(), lr.pmax, rows)
        if rank == 0:
            ref = P.lowrank_proximity(whole, rank=8, mode="f32", seed=1)
            full = P.pair_counts_device(whole, _lib.UPPER_I32).cpu().numpy()
            out["ref"] = (ref.dequantized(), ref.pmax, full)
    finally:
        dist.destroy_process_group()


def test_tree_sharded_lowrank_and_row_sharded_dense():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_rank, args=(2, _port(), out), nprocs=2, join=True, start_method="spawn")
    A_ref, pmax_ref, full = out["ref"]
    for r in (0, 1):
        A, pmax, _ = out[r]
        R = A_ref
        rel = np.linalg.norm(A @ A.T - R @ R.T) / np.linalg.norm(R @ R.T)
        assert rel <= 1e-5, rel
        assert abs(pmax - pmax_ref) <= 1e-5 * abs(pmax_ref)
    assert np.array_equal(np.concatenate([out[0][2], out[1][2]]), full)
