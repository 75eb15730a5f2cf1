"""Multi-GPU partitioning of the proximity path.

One process per GPU (torch.distributed, NCCL on GPUs / gloo in CPU tests):
  * sketch (K4): trees are sharded; every rank builds the leaf codes and
    leaf buckets of its own trees only and the (n, k) sketch partials are
    summed with one all-reduce per pass (proximity._Sketch.apply).  QR,
    eigh, quantisation and MDS are replicated (identical inputs after the
    all-reduce, so identical outputs).
  * dense counts (K3): output rows are sharded into blocks of equal
    upper-triangle area; no reduction (every rank needs all codes, which it
    recomputes locally — traversal is cheap next to the counts).
"""

from __future__ import annotations


def env_rank_world():
    import os
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def tree_shard(B: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced tree range of ``rank`` (sizes differ by <= 1)."""
    if not 0 <= rank < world or B < world:
        raise ValueError(f"cannot shard {B} trees over {world} ranks")
    return B * rank // world, B * (rank + 1) // world


def _row_start(n: int, i: int) -> int:
    return i * (2 * n - i - 1) // 2


def row_shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [lo, hi) whose packed upper-triangle area is ~1/world of the
    total (row i holds n - i - 1 pairs), contiguous and covering [0, n)."""
    total = _row_start(n, n)

    def boundary(q: int) -> int:
        if q <= 0:
            return 0
        if q >= world:
            return n
        target = total * q / world
        a, b = 0, n
        while a < b:  # smallest i with area(0..i) >= target
            mid = (a + b) // 2
            if _row_start(n, mid) >= target:
                b = mid
            else:
                a = mid + 1
        return a

    return boundary(rank), boundary(rank + 1)


def all_reduce_int(value: int, group=None) -> int:
    """Sum of a Python int over the ranks (device tensor under NCCL)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return int(value)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([int(value)], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def all_reduce_sum(tensor, group=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor


def gather_codes(membership, group=None):
    """Full (n, B) host codes of a tree-sharded membership (all-gather of the
    local (n, Bl) blocks)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    d = membership.device()
    world = dist.get_world_size(group)
    sizes = [tree_shard(d.B, r, world) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    local = torch.zeros((d.n, width), dtype=torch.int32, device=d.codes_nb.device)
    local[:, :d.Bl] = d.codes_nb
    bufs = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(bufs, local, group=group)
    return np.concatenate([b[:, :hi - lo].cpu().numpy() for b, (lo, hi) in zip(bufs, sizes)],
                          axis=1)
