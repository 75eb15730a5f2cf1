"""Multi-process host logic of the sharded path on CPU with the
gloo backend, world_size 2: tree shards of the sketch summed by all_reduce
equal the whole-forest sketch (the only collective of the path), shard leaf
totals, and row shards of the dense triangle.  The per-rank compute is the
CPU oracle's restatement of M (M^T X) (oracle/rfx_oracle.c, test
infrastructure) — on GPUs the same partition runs rfxc_sketch_pass + NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_2511_19493_b200.distributed import all_reduce_int, row_shard, tree_shard
        g = golden("synth2k.npz")
        codes, lc = g["codes"], g["leaf_counts"]
        n, B = codes.shape
        X = np.random.default_rng(7).normal(size=(n, 6))
        lo, hi = tree_shard(B, rank, world)
        Yl = np.empty_like(X)
        part = np.ascontiguousarray(codes[:, lo:hi])
        orc.lib().orc_sketch_pass(orc._p(part), n, hi - lo, orc._p(np.ascontiguousarray(lc[lo:hi])),
                                  orc._p(np.ascontiguousarray(X)), X.shape[1], orc._p(Yl), 1)
        Yl *= (hi - lo) / B  # the oracle scales by its own tree count; shards use the global B
        t = torch.from_numpy(Yl)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        total = all_reduce_int(int(lc[lo:hi].sum()))
        rlo, rhi = row_shard(n, rank, world)
        if rank == 0:
            Yw = np.empty_like(X)
            orc.lib().orc_sketch_pass(orc._p(np.ascontiguousarray(codes)), n, B,
                                      orc._p(np.ascontiguousarray(lc)), orc._p(np.ascontiguousarray(X)),
                                      X.shape[1], orc._p(Yw), 1)
            out["err"] = float(np.abs(t.numpy() - Yw).max() / np.abs(Yw).max())
            out["total"] = total
            out["want_total"] = int(lc.sum())
        out[f"rows{rank}"] = (rlo, rhi)
    finally:
        dist.destroy_process_group()


def test_tree_shards_allreduce_to_whole_sketch(built):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["err"] <= 1e-12
    assert out["total"] == out["want_total"]
    n = golden("synth2k.npz")["codes"].shape[0]
    (a0, b0), (a1, b1) = out["rows0"], out["rows1"]
    assert a0 == 0 and b0 == a1 and b1 == n
