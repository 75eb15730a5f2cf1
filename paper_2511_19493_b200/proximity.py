"""Proximity backends — drop-in for the reference's proximity.py hot path.

Same function names, signatures, defaults, dataclasses and error behaviour as
``rfx.proximity`` (proximity.py:68-420); the bodies call the sm_100a kernels
of librfxc.so through the C ABI (include/rfxc.h).  There is no CPU fallback:
without a CUDA device or the built library every call raises RfxError.

Results stay on the device between calls (``LeafMembership`` keeps its codes
and leaf buckets in HBM; ``FullTriangle.packed`` / ``LeafMembership.codes``
are copied to the host only when read), so
``lowrank_proximity(leaf_membership(forest, ds), ...)`` never round-trips the
(n, B) codes through the host.

Tree sharding (multi-GPU): ``leaf_membership(..., trees=(lo, hi))``
builds a shard; ``lowrank_proximity`` on a shard all-reduces the (n, k)
sketch partials with torch.distributed (NCCL) — the only collective.
"""

from __future__ import annotations

import logging
import os
from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .device import DeviceForest, DeviceMembership, DeviceValues, host_copy, traverse
from .errors import BudgetError, DataError, RfxError
from .profiling import region
from .quantize import (BYTES_PER_ELEMENT, MODES, QuantFactor, dequantize,
                       device_dequantize, factor_quantize)

logger = logging.getLogger(__name__)

ZERO_TIER = 1e-6          # proximity.py:39
DEFAULT_TAU = 1e-4        # proximity.py:43
DEFAULT_BUDGET = 32 * 2**30
DEFAULT_RETENTION = 0.8
_OVERSAMPLE = 8           # proximity.py:51
_POWER_ITERS = 2          # proximity.py:52
SEQ_FACTOR, SEQ_PMAX = 3, 4


def _packed_len(n: int) -> int:
    return n * (n - 1) // 2


def _row_start(n: int, i: int) -> int:
    """Packed index of (i, i+1); _row_start(n, n) == n(n-1)/2."""
    return i * (2 * n - i - 1) // 2


def packed_index(n: int, i, j):
    """Index of (i, j), i < j, in the row-major packed upper triangle."""
    return i * (2 * n - i - 1) // 2 + (j - i - 1)


def _check_pair(n, i, j):
    i, j = int(i), int(j)
    if not (0 <= i < n and 0 <= j < n):
        raise IndexError(f"pair ({i}, {j}) out of range for n={n}")
    return (j, i) if i > j else (i, j)


# ---------------------------------------------------------------- membership
class LeafMembership:
    """Terminal-leaf code of every sample in every tree (proximity.py:68-97).

    Constructible from host arrays exactly like the reference dataclass;
    when produced by ``leaf_membership`` the codes live on the GPU and
    ``codes`` is materialised on first read."""

    def __init__(self, codes=None, leaf_counts=None, *, _dev: DeviceMembership | None = None):
        self._codes = None if codes is None else np.asarray(codes)
        self.leaf_counts = np.asarray(leaf_counts, dtype=np.int32)
        self._dev = _dev

    @property
    def codes(self) -> np.ndarray:
        if self._codes is None:
            d = self._dev
            if d.is_shard:
                raise RfxError("codes of a tree shard: gather with "
                               "distributed.gather_codes(membership)")
            self._codes = host_copy(d.codes_nb)
        return self._codes

    @codes.setter
    def codes(self, value):
        self._codes = np.asarray(value)
        self._dev = None

    @property
    def n(self) -> int:
        return self._dev.n if self._dev is not None else self._codes.shape[0]

    @property
    def tree_count(self) -> int:
        return self._dev.B if self._dev is not None else self._codes.shape[1]

    @property
    def total_leaves(self) -> int:
        """Leaves over the whole forest (all-reduced over the ranks when this
        membership is a tree shard)."""
        return _total_leaves(self)

    @property
    def tree_range(self):
        d = self._dev
        return (0, self.tree_count) if d is None else (d.tree_lo, d.tree_hi)

    def device(self) -> DeviceMembership:
        if self._dev is None:
            self._dev = DeviceMembership.from_host(self._codes, self.leaf_counts)
        return self._dev

    def onehot(self):
        """Host CSR one-hot (proximity.py:88-97) for API parity; the device
        path never builds it."""
        import scipy.sparse as sp
        codes = self.codes
        n, B = codes.shape
        off = np.zeros(B + 1, dtype=np.int64)
        off[1:] = np.cumsum(self.leaf_counts)
        cols = (codes.astype(np.int64) + off[:B][None, :]).reshape(-1)
        rows = np.repeat(np.arange(n, dtype=np.int64), B)
        return sp.csr_matrix((np.full(n * B, 1.0 / np.sqrt(B)), (rows, cols)),
                             shape=(n, int(off[B])))

    def __repr__(self):
        return f"LeafMembership(n={self.n}, tree_count={self.tree_count})"


def leaf_membership(forest, dataset, trees: tuple | None = None) -> LeafMembership:
    """Classify every sample down every tree on the GPU (proximity.py:100-116).

    Tree shards (multi-GPU): ``trees=(lo, hi)`` restricts the work to that
    range of ``forest``; a forest grown as a shard (``train(...,
    trees=(lo, hi))``, carrying ``tree_range``) is a shard by itself.  The
    membership of a shard keeps the forest-wide tree count B (the 1/B of
    every proximity) and its own trees' leaf counts."""
    if forest.n != dataset.n or forest.p != dataset.p:
        raise DataError("forest and dataset shapes disagree")
    grown = getattr(forest, "tree_range", None)
    if grown is not None:
        lo, hi, B = grown
        local = (0, forest.ntree)
    else:
        B = forest.ntree
        lo, hi = (0, B) if trees is None else (int(trees[0]), int(trees[1]))
        if not 0 <= lo < hi <= B:
            raise DataError(f"tree range {trees} outside [0, {B})")
        local = (lo, hi)
    dvals = DeviceValues(dataset.values, defer=True)
    layout = None if dvals.exact_f32 else _lib.NODES_F64
    dforest = DeviceForest(forest, *local, layout=layout, defer=True)
    # PCIe order: the first half of the samples, the first two tree chunks
    # (the first one small), the other samples, the other chunks — traverse()
    # walks the first two chunks sample block by sample block, so the first
    # launch waits for ~1/4 of the bytes instead of all values + a full chunk
    n = dvals.n
    split = (n // 2) // 128 * 128 if dvals.exact_f32 and n >= 256 else 0
    if split:
        dvals.upload_rows(0, split)
    first = min(2, len(dforest._spans)) if split else 1
    for j in range(first):
        dforest.upload_chunk(j)
    if dvals.exact_f32:
        dvals.upload_rows(split, n)
    for j in range(first, len(dforest._spans)):
        dforest.upload_chunk(j)
    nb, tm, chunks = traverse(dforest, dvals)
    dev = DeviceMembership(nb, tm, dforest.leaf_counts, lo, hi, B, chunks)
    return LeafMembership(leaf_counts=dforest.leaf_counts, _dev=dev)


# ------------------------------------------------------------- full triangle
def oob_votes(forest, dataset, membership: "LeafMembership | None" = None) -> np.ndarray:
    """Out-of-bag class votes (n, C) int64 recomputed on the GPU from the K1
    leaf codes — the accumulation the trainer does per tree
    (oob_votes_tree, _kernels.py:377-385; forest.py:287-290), so it must
    equal ``forest.oob_votes`` exactly."""
    import torch
    mem = membership if membership is not None else leaf_membership(forest, dataset)
    d = mem.device()
    if d.is_shard:
        raise DataError("oob votes need every tree of the forest")
    counts = np.ascontiguousarray(forest.bootstrap.counts, dtype=np.int32)
    if counts.shape != (d.B, d.n):
        raise DataError(f"bootstrap counts {counts.shape} do not match (B, n) = ({d.B}, {d.n})")
    leaf_class = np.concatenate([np.asarray(t.node_class)[np.asarray(t.status) == 1]
                                 for t in forest.trees]).astype(np.int32)
    if leaf_class.size != d.total_leaves:
        raise DataError("leaf classes do not match the membership's leaf counts")
    C = int(forest.class_count)
    dev = d.codes_tm.device
    lc = torch.from_numpy(leaf_class).to(dev)
    inbag = torch.from_numpy(counts).to(dev)
    votes = torch.empty((d.n, C), dtype=torch.int64, device=dev)
    _lib.call("rfxc_oob_votes", _lib.ptr(d.codes_tm), d.n, d.B, _lib.ptr(d.leaf_base),
              _lib.ptr(lc), _lib.ptr(inbag), C, _lib.ptr(votes), _lib.stream_handle())
    return votes.cpu().numpy()


@dataclass
class FullTriangle:
    """Exact proximities, packed upper triangle, implicit unit diagonal
    (proximity.py:123-146)."""

    n: int
    tree_count: int
    packed: np.ndarray
    _packed_dev: object = field(default=None, repr=False, compare=False)  # HBM copy (K3 output)

    def entry(self, i: int, j: int) -> float:
        i, j = _check_pair(self.n, i, j)
        if i == j:
            return 1.0
        return float(self.packed[packed_index(self.n, i, j)])

    def packed_device(self):
        """The packed triangle in HBM (kept from full_proximity, else uploaded)."""
        import torch
        if self._packed_dev is None:
            self._packed_dev = torch.from_numpy(np.ascontiguousarray(self.packed)).to(
                _lib.require_cuda())
        return self._packed_dev

    def to_dense(self) -> np.ndarray:
        dense = np.empty((self.n, self.n), dtype=np.float64)
        iu = np.triu_indices(self.n, k=1)
        dense[iu] = self.packed
        dense.T[iu] = self.packed
        np.fill_diagonal(dense, 1.0)
        return dense

    def nbytes(self) -> int:
        return self.packed.nbytes


def _device_budget(nbytes: int, what: str, n: int, B: int):
    """Refuse (BudgetError + planner dict) a device allocation that cannot fit:
    free device memory plus the blocks torch has cached but not handed out."""
    import torch
    free, _total = torch.cuda.mem_get_info()
    free += torch.cuda.memory_reserved() - torch.cuda.memory_allocated()
    if nbytes > free:
        raise BudgetError(f"{what} for n={n} needs {nbytes} bytes of device memory, "
                          f"{free} free; shard rows across GPUs or use the lowrank backend",
                          memory_plan(n, tree_count=B))


def _device_empty(numel: int, dtype, dev, what: str, n: int, B: int):
    """torch.empty on the device, an out-of-memory error mapped to BudgetError."""
    import torch
    try:
        return torch.empty(numel, dtype=dtype, device=dev)
    except torch.OutOfMemoryError as e:
        raise BudgetError(f"{what} for n={n}: device allocation of {numel} elements failed "
                          f"({e}); shard rows across GPUs or use the lowrank backend",
                          memory_plan(n, tree_count=B)) from e


def pair_counts_device(membership: LeafMembership, layout: int, row_lo: int = 0,
                       row_hi: int | None = None):
    """K3 on the device: returns the output tensor for rows [row_lo, row_hi)."""
    import torch
    d = membership.device()
    if d.is_shard:
        raise DataError("pair counts need every tree's codes (row-shard instead)")
    n, B = d.n, d.B
    row_hi = n if row_hi is None else row_hi
    if layout == _lib.BLOCK_I32:
        numel, dt = (row_hi - row_lo) * n, torch.int32
    else:
        numel = _row_start(n, row_hi) - _row_start(n, row_lo)
        dt = torch.float64 if layout == _lib.UPPER_F64 else torch.int32
    _device_budget(numel * (8 if dt == torch.float64 else 4), "pair counts", n, B)
    out = _device_empty(max(numel, 1), dt, d.codes_nb.device, "pair counts", n, B)
    if n >= 2 and row_hi > row_lo:
        choice = pair_kernel(d, decide=False)
        if choice == "auto" and layout == _lib.BLOCK_I32:
            choice = pair_kernel(d)  # the row-block layout is not gated (host choice)
        if choice == "auto":
            # both kernels launched; the device-side gate lets one of them run
            pos, (ids, idb), seg = d.positions(), d.walk_ids(), d.buckets()[1]
            gate = d.pair_gate()
            with region("pair_counts"):
                _lib.call("rfxc_pair_counts_leaf", _lib.ptr(pos), _lib.ptr(ids), idb,
                          _lib.ptr(d.codes_nb), _lib.ptr(seg), _lib.ptr(d.leaf_base), n, B,
                          row_lo, row_hi, layout, _lib.ptr(out), _lib.ptr(gate),
                          _lib.stream_handle())
                _lib.call("rfxc_pair_counts", _lib.ptr(d.codes_nb), n, B, row_lo, row_hi, layout,
                          _lib.ptr(out), _lib.ptr(gate), _lib.stream_handle())
        elif choice == "leaf":
            pos, (ids, idb), seg = d.positions(), d.walk_ids(), d.buckets()[1]
            with region("pair_counts"):
                _lib.call("rfxc_pair_counts_leaf", _lib.ptr(pos), _lib.ptr(ids), idb,
                          _lib.ptr(d.codes_nb), _lib.ptr(seg), _lib.ptr(d.leaf_base), n, B,
                          row_lo, row_hi, layout, _lib.ptr(out), None, _lib.stream_handle())
        else:
            with region("pair_counts"):
                _lib.call("rfxc_pair_counts", _lib.ptr(d.codes_nb), n, B, row_lo, row_hi, layout,
                          _lib.ptr(out), None, _lib.stream_handle())
    return out[:numel]


# The leaf-segmented kernel costs ~ n*B + (same-leaf pairs)/32 warp steps; the
# tile kernel n^2*B/2 compares whatever the leaves.  Measured crossover: the
# segmented kernel wins while same-leaf pairs are below this share of all
# (pair, tree) units (fully grown trees: well under 1 %).
LEAF_KERNEL_MAX_SHARE = 0.2


def pair_kernel(d, decide: bool = True) -> str:
    """'leaf' (K2-bucket walk, the reference's per-leaf formulation) or
    'tile' (compare tiles); RFX_PAIRS_KERNEL=leaf|tile forces one.  With
    decide=False the data-dependent case returns 'auto' (the device decides,
    no host round trip)."""
    forced = os.environ.get("RFX_PAIRS_KERNEL")
    if forced in ("leaf", "tile"):
        return forced
    if d.B > 4096 or d.n * d.Bl >= (1 << 32):  # shared per-tree tables, u32 perm indices
        return "tile"
    if not decide:
        return "auto"
    units = d.n * (d.n - 1) // 2 * d.Bl
    return "leaf" if d.same_leaf_pairs() <= LEAF_KERNEL_MAX_SHARE * units else "tile"


def full_proximity(membership: LeafMembership,
                   budget_bytes: int | None = DEFAULT_BUDGET) -> FullTriangle:
    """p(i, j) = (1/B) #{trees with node_b(i) = node_b(j)}, exact
    (proximity.py:188-201); the count/B division runs in the kernel
    epilogue as an IEEE f64 division."""
    n = membership.n
    est = 8 * _packed_len(n)
    if budget_bytes is not None and est > budget_bytes:
        raise BudgetError(
            f"full proximity for n={n} needs {est} bytes (packed), over the "
            f"{budget_bytes}-byte budget; consider the triblock or lowrank backend",
            memory_plan(n, tree_count=membership.tree_count))
    if n < 2:
        return FullTriangle(n=n, tree_count=membership.tree_count,
                            packed=np.empty(0, dtype=np.float64))
    out = pair_counts_device(membership, _lib.UPPER_F64)
    return FullTriangle(n=n, tree_count=membership.tree_count, packed=host_copy(out),
                        _packed_dev=out)


# ------------------------------------------------------------------ TriBlock
class PairMap(Mapping):
    """Read-only (i, j) -> value map over (i, j)-sorted arrays: the TriBlock
    dense tier without a Python dict insert per pair (proximity.py:315-316).
    Supports everything the reference does with the dict (get, [], len,
    iteration, items, values, keys)."""

    def __init__(self, n: int, i: np.ndarray, j: np.ndarray, v: np.ndarray):
        self.n = n
        self.i = np.asarray(i, dtype=np.int32)
        self.j = np.asarray(j, dtype=np.int32)
        self.v = np.asarray(v, dtype=np.float64)
        self._key = self.i.astype(np.int64) * n + self.j

    def _find(self, key):
        try:
            a, b = int(key[0]), int(key[1])
        except (TypeError, ValueError, IndexError):
            return -1
        k = a * self.n + b
        pos = int(np.searchsorted(self._key, k))
        return pos if pos < len(self._key) and self._key[pos] == k else -1

    def __getitem__(self, key):
        pos = self._find(key)
        if pos < 0:
            raise KeyError(key)
        return float(self.v[pos])

    def __contains__(self, key):
        return self._find(key) >= 0

    def __len__(self):
        return len(self._key)

    def __iter__(self):
        return zip(self.i.tolist(), self.j.tolist())

    def items(self):
        return zip(zip(self.i.tolist(), self.j.tolist()), self.v.tolist())

    def values(self):
        return self.v.tolist()


@dataclass
class TriBlock:
    """Value-tiered proximity storage (proximity.py:208-272)."""

    n: int
    tree_count: int
    tau: float
    dense: Mapping
    sparse_i: np.ndarray
    sparse_j: np.ndarray
    sparse_v: np.ndarray
    _sparse_key: np.ndarray = field(default=None, repr=False)

    def __post_init__(self):
        if self._sparse_key is None:
            self._sparse_key = self.sparse_i.astype(np.int64) * self.n + self.sparse_j

    def entry(self, i: int, j: int) -> float:
        i, j = _check_pair(self.n, i, j)
        if i == j:
            return 1.0
        v = self.dense.get((i, j))
        if v is not None:
            return float(v)
        key = i * self.n + j
        pos = np.searchsorted(self._sparse_key, key)
        if pos < len(self._sparse_key) and self._sparse_key[pos] == key:
            return float(self.sparse_v[pos])
        return 0.0

    @property
    def dense_count(self) -> int:
        return len(self.dense)

    @property
    def sparse_count(self) -> int:
        return len(self.sparse_v)

    @property
    def stored_pairs(self) -> int:
        return self.dense_count + self.sparse_count

    def compression_ratio(self) -> float:
        return _packed_len(self.n) / max(self.stored_pairs, 1)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n, self.n), dtype=np.float64)
        if isinstance(self.dense, PairMap):
            di, dj, dv = self.dense.i, self.dense.j, self.dense.v
        else:
            keys = list(self.dense)
            di = np.array([k[0] for k in keys], dtype=np.int64)
            dj = np.array([k[1] for k in keys], dtype=np.int64)
            dv = np.array([self.dense[k] for k in keys], dtype=np.float64)
        out[di, dj] = dv
        out[dj, di] = dv
        out[self.sparse_i, self.sparse_j] = self.sparse_v
        out[self.sparse_j, self.sparse_i] = self.sparse_v
        np.fill_diagonal(out, 1.0)
        return out

    def nbytes(self) -> int:
        return self.dense_count * 16 + self.sparse_count * 16


def _scan(x):
    import torch
    out = torch.empty_like(x)
    tot = torch.empty(1, dtype=torch.int64, device=x.device)
    _lib.call("rfxc_exclusive_scan_i64", _lib.ptr(x), x.numel(), _lib.ptr(out), _lib.ptr(tot),
              _lib.stream_handle())
    return out, tot


def triblock_proximity(membership: LeafMembership, tau: float = DEFAULT_TAU,
                       budget_bytes: int | None = DEFAULT_BUDGET) -> TriBlock:
    """Same values as full_proximity routed into tiers (proximity.py:275-327):
    int32 count tiles on the device, then a count / scan / emit compaction
    that writes both tiers already sorted by (i, j)."""
    import torch
    if not (ZERO_TIER < tau < 1.0):
        raise DataError(f"tau must lie in ({ZERO_TIER}, 1), got {tau}")
    n, B = membership.n, membership.tree_count
    est = int(8 * n * n * 0.5 * DEFAULT_RETENTION)
    if budget_bytes is not None and est > budget_bytes:
        raise BudgetError(
            f"triblock proximity for n={n} estimates {est} bytes, over the "
            f"{budget_bytes}-byte budget; consider the lowrank backend",
            memory_plan(n, tree_count=B))
    empty_i = np.empty(0, dtype=np.int32)
    if n < 2:
        return TriBlock(n, B, tau, PairMap(n, empty_i, empty_i, np.empty(0)), empty_i,
                        empty_i, np.empty(0))
    d = membership.device()
    dev = d.codes_nb.device
    # row blocks bounded to ~1 G int32 counters each
    hot, cold = [], []
    lo = 0
    while lo < n - 1:
        a, b = lo + 1, n  # largest hi with at most 2^30 counters (at least one row)
        while a < b:
            mid = (a + b + 1) // 2
            if _row_start(n, mid) - _row_start(n, lo) <= (1 << 30):
                a = mid
            else:
                b = mid - 1
        hi = a
        counts = pair_counts_device(membership, _lib.UPPER_I32, lo, hi)
        rows = hi - lo
        rc = torch.empty(2 * rows, dtype=torch.int64, device=dev)
        _lib.call("rfxc_triblock_count", _lib.ptr(counts), n, B, lo, hi, float(tau), _lib.ptr(rc),
                  _lib.stream_handle())
        oh, th = _scan(rc[:rows])
        oc, tc = _scan(rc[rows:])
        nh, nc = int(th.item()), int(tc.item())
        offs = torch.cat([oh, oc])
        hi_i = torch.empty(max(nh, 1), dtype=torch.int32, device=dev)
        hi_j = torch.empty(max(nh, 1), dtype=torch.int32, device=dev)
        hi_v = torch.empty(max(nh, 1), dtype=torch.float64, device=dev)
        co_i = torch.empty(max(nc, 1), dtype=torch.int32, device=dev)
        co_j = torch.empty(max(nc, 1), dtype=torch.int32, device=dev)
        co_v = torch.empty(max(nc, 1), dtype=torch.float64, device=dev)
        _lib.call("rfxc_triblock_emit", _lib.ptr(counts), n, B, lo, hi, float(tau),
                  _lib.ptr(offs), _lib.ptr(hi_i), _lib.ptr(hi_j), _lib.ptr(hi_v),
                  _lib.ptr(co_i), _lib.ptr(co_j), _lib.ptr(co_v), _lib.stream_handle())
        hot.append((hi_i[:nh].cpu().numpy(), hi_j[:nh].cpu().numpy(), hi_v[:nh].cpu().numpy()))
        cold.append((co_i[:nc].cpu().numpy(), co_j[:nc].cpu().numpy(), co_v[:nc].cpu().numpy()))
        del counts
        lo = hi
    cat = lambda parts, q: np.concatenate([p[q] for p in parts])
    dense = PairMap(n, cat(hot, 0), cat(hot, 1), cat(hot, 2))
    return TriBlock(n=n, tree_count=B, tau=tau, dense=dense, sparse_i=cat(cold, 0),
                    sparse_j=cat(cold, 1), sparse_v=cat(cold, 2))


# ------------------------------------------------------------------ low rank
@dataclass
class LowRankQuantized:
    """Symmetric factorisation P ~ Q Q^T with Q quantised (proximity.py:334-364).
    ``_dq_dev`` keeps the dequantised factor on the GPU for mds_lowrank."""

    n: int
    rank: int
    mode: str
    factor: QuantFactor
    pmax: float
    tree_count: int
    rank_degraded: bool = False
    _dq: np.ndarray = field(default=None, repr=False)
    _dq_dev: object = field(default=None, repr=False)
    # device results whose host copies are still in flight (event, builder):
    # ``factor`` / ``pmax`` resolve on first access, so the GPU path can run
    # on (mds_lowrank reads pmax from _pmax_dev) without a host round trip
    _pending: object = field(default=None, repr=False, compare=False)
    _pmax_dev: object = field(default=None, repr=False, compare=False)

    def __getattribute__(self, name):
        if name in ("factor", "pmax") and object.__getattribute__(self, "_pending") is not None:
            ev, build = object.__getattribute__(self, "_pending")
            ev.synchronize()
            f, pm = build()
            object.__setattr__(self, "factor", f)
            object.__setattr__(self, "pmax", pm)
            object.__setattr__(self, "_pending", None)
        return object.__getattribute__(self, name)

    def dequantized(self) -> np.ndarray:
        if self._dq is None:
            self._dq = self.factor.dequantize()
        return self._dq

    def device_codes(self):
        """(data, scales) of the quantised factor on the GPU."""
        import torch
        if getattr(self, "_codes_dev", None) is None:
            dev = _lib.require_cuda()
            data = torch.from_numpy(np.ascontiguousarray(self.factor.data)).to(dev)
            sc = None if self.factor.scales is None else torch.from_numpy(
                np.ascontiguousarray(self.factor.scales)).to(dev)
            self._codes_dev = (data, sc)
        return self._codes_dev

    def dequantized_device(self):
        """(n, r) f64 dequantised factor on the GPU."""
        if self._dq_dev is None:
            data, sc = self.device_codes()
            n, r = self.n, int(np.prod(self.factor.shape)) // max(self.n, 1)
            self._dq_dev = device_dequantize(data, sc, n, r, self.mode)
        return self._dq_dev

    def entry(self, i: int, j: int) -> float:
        i, j = _check_pair(self.n, i, j)
        if i == j:
            return 1.0
        Q = self.dequantized()
        return float(np.clip(Q[i] @ Q[j], 0.0, 1.0))

    def nbytes(self) -> int:
        return self.factor.payload_nbytes()


def _l2_bytes() -> int:
    import ctypes
    import torch
    sm, l2, smem = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
    _lib.call("rfxc_device_info", torch.cuda.current_device(), ctypes.byref(sm), ctypes.byref(l2),
              ctypes.byref(smem))
    return int(l2.value)


# fraction of L2 the sketch may fill with X, Y and two batches of leaf sums
SKETCH_L2_FRACTION = float(os.environ.get("RFX_SKETCH_L2_FRACTION", "0.9"))
SKETCH_FUSED_MAX_LD = 128


class _Sketch:
    """P X for the (local trees of the) membership, and the all-reduce of the
    partials when the membership is a tree shard.

    k <= 128: rfxc_sketch_pass (trees in batches whose leaf sums stay
    L2-resident; per batch a leaf-sum and a gather kernel, the next batch's
    leaf sums overlapping this batch's gather when two buffers fit); wider
    sketches use the two-kernel leaf_sums / leaf_gather path."""

    def __init__(self, d: DeviceMembership, k: int, group=None, budget: int | None = None):
        import ctypes
        import torch
        self.d = d
        self.k = k
        self.ld = (k + 3) // 4 * 4
        self.perm, self.seg = d.buckets()
        dev = d.codes_nb.device
        self.group = group
        # empty leaves are handled on the device (run-start search), so the
        # choice needs no host read of the bucketing's flag
        self.fused = self.ld <= SKETCH_FUSED_MAX_LD
        if self.fused:
            if budget is None:  # two batches of leaf sums next to X in L2 (Y streams)
                budget = int(SKETCH_L2_FRACTION * _l2_bytes()) - d.n * self.ld * 4
                budget = max(budget, 8 << 20)
            T, rows, nbuf, wb = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64()
            lc = np.ascontiguousarray(d.leaf_counts, dtype=np.int32)
            _lib.call("rfxc_sketch_plan", lc.ctypes.data_as(_lib.P), d.Bl, d.n, k, budget,
                      ctypes.byref(T), ctypes.byref(rows), ctypes.byref(nbuf), ctypes.byref(wb))
            self.T, self.s_rows, self.nbuf = int(T.value), int(rows.value), int(nbuf.value)
            self.work = torch.empty(int(wb.value), dtype=torch.uint8, device=dev)
            _lib.call("rfxc_sketch_prepare", _lib.ptr(self.seg), _lib.ptr(d.leaf_base), d.n, d.Bl,
                      k, self.T, self.s_rows, self.nbuf, _lib.ptr(self.work), _lib.stream_handle())
        else:
            self.S = torch.empty((max(d.total_leaves, 1), self.ld), dtype=torch.float32,
                                 device=dev)

    def apply(self, X32, kk: int, reduce: bool = True):
        """P X as (n, kk) f64; X32 is the (n, ld) f32 copy of X (zero beyond kk)."""
        import torch
        d = self.d
        Y = torch.empty((d.n, kk), dtype=torch.float64, device=X32.device)
        if self.fused:
            if kk != self.k:
                # fewer surviving columns: the padded operand keeps stride ld,
                # so sketch all ld columns and keep the first kk
                full = torch.empty((d.n, self.k), dtype=torch.float64, device=X32.device)
                self._pass(X32, full)
                Y.copy_(full[:, :kk])
            else:
                self._pass(X32, Y)
        else:
            with region("leaf_sums"):
                _lib.call("rfxc_leaf_sums", _lib.ptr(self.perm), _lib.ptr(self.seg), 0,
                          d.total_leaves, _lib.ptr(X32), kk, self.ld, _lib.ptr(self.S),
                          _lib.stream_handle())
            with region("leaf_gather"):
                _lib.call("rfxc_leaf_gather", _lib.ptr(d.codes_nb), d.n, d.Bl,
                          _lib.ptr(d.leaf_base), _lib.ptr(self.S), kk, self.ld, 1.0 / d.B, 0,
                          _lib.ptr(Y), _lib.stream_handle())
        if d.is_shard and reduce:
            import torch.distributed as dist
            dist.all_reduce(Y, op=dist.ReduceOp.SUM, group=self.group)
        return Y

    def _pass(self, X32, Y):
        d = self.d
        with region("sketch_pass"):
            _lib.call("rfxc_sketch_pass", _lib.ptr(self.perm), _lib.ptr(self.seg),
                      _lib.ptr(d.codes_nb), _lib.ptr(d.leaf_base), _lib.ptr(d.has_empty), d.n,
                      d.Bl, _lib.ptr(X32), self.k, self.ld, 1.0 / d.B, self.T, self.s_rows,
                      self.nbuf, _lib.ptr(Y), _lib.ptr(self.work), _lib.stream_handle())


def _gram(A, Bm):
    """A^T Bm (ka x kb) on the device (fixed-order skinny reduction)."""
    import torch
    n, ka = A.shape
    kb = Bm.shape[1]
    parts = torch.empty(_lib.load().rfxc_gram_parts(n) * ka * kb, dtype=torch.float64,
                        device=A.device)
    C = torch.empty((ka, kb), dtype=torch.float64, device=A.device)
    _lib.call("rfxc_gram", _lib.ptr(A), _lib.ptr(Bm), n, ka, kb, _lib.ptr(parts), _lib.ptr(C),
              _lib.stream_handle())
    return C


def _times(Y, M, ld32=0):
    """(Y @ M) on the device (M a device (ka, kb) tensor): f64, plus the padded
    f32 sketch operand when ld32 > 0."""
    import torch
    n, ka = Y.shape
    kb = M.shape[1]
    Z = torch.empty((n, kb), dtype=torch.float64, device=Y.device)
    Z32 = torch.empty((n, max(ld32, 4)), dtype=torch.float32, device=Y.device) if ld32 else None
    _lib.call("rfxc_matmul_small", _lib.ptr(Y), n, ka, _lib.ptr(M), kb, _lib.ptr(Z),
              _lib.ptr(Z32), Z32.shape[1] if ld32 else 0, _lib.stream_handle())
    return Z, Z32


def orthonormalize(Y, ld: int):
    """Orthonormal basis of range(Y) (the np.linalg.qr of proximity.py:395,
    :397), entirely on the device: shifted CholeskyQR3 (a shifted CholeskyQR
    step, then two plain ones; each = Gram, k x k Cholesky inverse, small
    matmul).  Returns (Q f64 (n, k), Q32 f32 (n, ld))."""
    with region("orthonormalize"):
        import torch
        n, k = Y.shape
        if k > LINALG_MAX_K:
            return _orthonormalize_host(Y, ld)
        shift = 11.0 * (n * k + k * (k + 1)) * np.finfo(np.float64).eps / 2
        Q = Y
        for step in range(3):
            Rinv = torch.empty((k, k), dtype=torch.float64, device=Y.device)
            _lib.call("rfxc_chol_inv", _lib.ptr(_gram(Q, Q)), k, shift if step == 0 else 0.0,
                      _lib.ptr(Rinv), _lib.stream_handle())
            Q, Q32 = _times(Q, Rinv, ld if step == 2 else 0)
        return Q, Q32


LINALG_MAX_K = 110  # one-CTA k x k kernels (csrc/linalg.cu)
RITZ_ON_DEVICE = os.environ.get("RFX_RITZ_ON_DEVICE", "0") == "1"


def _orthonormalize_host(Y, ld: int):
    """k > 110: the k x k steps on the host (eigen-map + one CholeskyQR step)."""
    import torch
    G = _gram(Y, Y).cpu().numpy()
    lam, V = np.linalg.eigh(0.5 * (G + G.T))
    top = lam.max() if lam.size else 0.0
    keep = lam > max(top, 0.0) * 1e-13
    if not keep.any():
        keep = np.zeros_like(keep)
        keep[-1] = True
        lam = np.maximum(lam, 1e-300)
    M1 = np.zeros((G.shape[0], G.shape[0]))
    sel = np.nonzero(keep)[0][::-1]  # strongest direction first
    M1[:, :len(sel)] = V[:, sel] / np.sqrt(lam[sel])[None, :]
    Q1, _ = _times(Y, torch.from_numpy(M1).to(Y.device))
    G2 = _gram(Q1, Q1).cpu().numpy()
    kk = len(sel)
    R = np.linalg.cholesky(0.5 * (G2[:kk, :kk] + G2[:kk, :kk].T)).T
    Rinv = np.zeros_like(M1)
    Rinv[:kk, :kk] = np.linalg.solve(R, np.eye(kk))
    return _times(Q1, torch.from_numpy(Rinv).to(Y.device), ld)


def _ritz_factor_map(T, k: int, r: int):
    """Wr (k x r) = W_r sqrt(clip(l_r, 0)) for the top-r eigenpairs of T."""
    import torch
    Wr = torch.empty((k, r), dtype=torch.float64, device=T.device)
    if k <= LINALG_MAX_K and RITZ_ON_DEVICE:
        _lib.call("rfxc_ritz_factor_map", _lib.ptr(T), k, r, _lib.ptr(Wr), _lib.stream_handle())
        return Wr
    # host LAPACK eigh of the k x k T (one small D2H; the one-CTA Jacobi
    # kernel is slower than this round trip at k = 40)
    Th = T.cpu().numpy()
    lam, W = np.linalg.eigh(0.5 * (Th + Th.T))
    order = np.argsort(lam)[::-1][:r]
    lam = np.clip(lam[order], 0.0, None)
    Wr.copy_(torch.from_numpy(W[:, order] * np.sqrt(lam)[None, :]))
    return Wr


# Limit of the device kernels (INTEGRATION.md "Limits"): the factor /
# quantisation and outlier kernels take r <= 256 columns, the MDS kernel
# r <= 192; lowrank_proximity refuses ranks above 192 up front so every factor
# it returns can go on through mds_lowrank and outlier_scores.
MAX_RANK = 192


def _total_leaves(membership: LeafMembership, group=None) -> int:
    """Leaves over the whole forest: a tree shard sums its own over ``group``
    (the ranks holding the other shards), exactly the group the sketch
    all-reduces over."""
    d = membership._dev
    local = int(membership.leaf_counts.sum())
    if d is None or not d.is_shard:
        return local
    from .distributed import all_reduce_int
    return all_reduce_int(local, group)


def lowrank_device(membership: LeafMembership, rank: int, mode: str = "i8", seed: int = 0,
                   group=None) -> "DeviceLowRank":
    """The device pipeline behind lowrank_proximity (results stay in HBM)."""
    import torch
    if mode not in MODES:
        raise DataError(f"unknown quantization mode {mode!r}")
    n = membership.n
    if rank < 1:
        raise DataError(f"rank must be >= 1, got {rank}")
    bound = min(n, _total_leaves(membership, group))
    if min(rank, bound) > MAX_RANK:
        raise DataError(f"rank {min(rank, bound)} above this build's limit {MAX_RANK} "
                        f"(the MDS kernel's; INTEGRATION.md 'Limits')")
    degraded = rank > bound
    if degraded:
        logger.warning("requested rank %d exceeds membership rank bound %d; "
                       "degrading to the exact bound", rank, bound)
    r = min(rank, bound)
    d = membership.device()
    dev = d.codes_nb.device
    k = min(n, r + _OVERSAMPLE)
    sk = _Sketch(d, k, group)
    ld = sk.ld
    omega = torch.empty((n, k), dtype=torch.float64, device=dev)
    _lib.call("rfxc_normals", seed, SEQ_FACTOR, n * k, _lib.ptr(omega), _lib.stream_handle())
    X32 = torch.empty((n, ld), dtype=torch.float32, device=dev)
    _lib.call("rfxc_pack_f32", _lib.ptr(omega), n, k, ld, _lib.ptr(X32), _lib.stream_handle())
    Q, Q32 = orthonormalize(sk.apply(X32, k), ld)
    for _ in range(_POWER_ITERS):
        Q, Q32 = orthonormalize(sk.apply(Q32, k), ld)
    Z = sk.apply(Q32, k)
    # Rayleigh-Ritz: T = Q^T (P Q), top-r eigenpairs -> Wr = W_r sqrt(l_r)
    with region("ritz"):
        Wr = _ritz_factor_map(_gram(Q, Z), k, r)
    with region("factor_quantize"):
        data, scales = factor_quantize(Q, Wr, mode)
    dq = device_dequantize(data, scales, n, r, mode)
    parts = torch.empty(_lib.load().rfxc_gram_parts(n) + 1, dtype=torch.float64, device=dev)
    pm = torch.empty(1, dtype=torch.float64, device=dev)
    with region("pmax"):
        _lib.call("rfxc_pmax", _lib.ptr(dq), n, r, seed, _lib.ptr(parts), _lib.ptr(pm),
                  _lib.stream_handle())
    return DeviceLowRank(n=n, rank=r, mode=mode, data=data, scales=scales, dq=dq,
                         pm=pm, tree_count=membership.tree_count, degraded=degraded)


@dataclass
class DeviceLowRank:
    """Device-resident result of the low-rank pipeline (factor codes, scales,
    dequantised factor, pmax) before any host copy."""

    n: int
    rank: int
    mode: str
    data: object
    scales: object
    dq: object
    pm: object  # (1,) f64 on the device
    tree_count: int
    degraded: bool

    @property
    def pmax(self) -> float:
        return float(self.pm.item())

    def to_host(self) -> LowRankQuantized:
        """The reference's LowRankQuantized; the factor codes, scales and pmax
        cross PCIe asynchronously (pinned buffers, stream-ordered) and are
        waited for on first access."""
        import torch
        pin = lambda t: torch.empty(t.shape, dtype=t.dtype, pin_memory=True)  # noqa: E731
        hd, hp = pin(self.data), pin(self.pm)
        hs = None if self.scales is None else pin(self.scales)
        hd.copy_(self.data, non_blocking=True)
        hp.copy_(self.pm, non_blocking=True)
        if hs is not None:
            hs.copy_(self.scales, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        mode, shape = self.mode, (self.n, self.rank)

        def build():
            d = hd.numpy()
            if mode in ("f32", "f16", "i8"):
                d = d.reshape(shape)
            s_ = None if hs is None else hs.numpy().astype(np.float64)
            return QuantFactor(mode, tuple(shape), d, s_), float(hp.numpy()[0])

        out = LowRankQuantized(n=self.n, rank=self.rank, mode=self.mode, factor=None, pmax=None,
                               tree_count=self.tree_count, rank_degraded=self.degraded,
                               _dq_dev=self.dq, _pending=(ev, build), _pmax_dev=self.pm)
        out._codes_dev = (self.data, self.scales)
        return out


def lowrank_proximity(membership: LeafMembership, rank: int, mode: str = "i8",
                      seed: int = 0, group=None) -> LowRankQuantized:
    """Randomised symmetric rank-r factorisation of P = M M^T followed by
    quantisation (proximity.py:367-420), with P applied implicitly on the
    GPU (K4) and never materialised.  ``group``: torch.distributed group of
    the tree shards when ``membership`` is a shard."""
    return lowrank_device(membership, rank, mode, seed, group).to_host()


# ------------------------------------------------------------- outlier scores
def outlier_scores(repr_, clamp_floor: float | None = None) -> np.ndarray:
    """Mean inverse-squared proximity of each sample to all others
    (proximity.py:432-485): proximities clamped below at ``clamp_floor``
    (default 1/B).  FullTriangle and LowRankQuantized run on the GPU
    (rfxc_outlier_packed / rfxc_outlier_lowrank, n^2 r on the FP64 tensor
    cores for the factor); a TriBlock's tiers are host arrays by contract, so
    its O(pairs) scatter stays the reference's host epilogue."""
    import torch
    n = repr_.n
    if n < 2:
        raise RfxError("outlier scores need n >= 2")
    floor = 1.0 / repr_.tree_count if clamp_floor is None else clamp_floor
    if floor <= 0:
        raise RfxError("clamp_floor must be positive")
    if isinstance(repr_, FullTriangle):
        packed = repr_.packed_device()
        work = torch.empty(int(_lib.load().rfxc_outlier_work_bytes(n)), dtype=torch.uint8,
                           device=packed.device)
        scores = torch.empty(n, dtype=torch.float64, device=packed.device)
        with region("outlier"):
            _lib.call("rfxc_outlier_packed", _lib.ptr(packed), n, float(floor), _lib.ptr(scores),
                      _lib.ptr(work), _lib.stream_handle())
        return scores.cpu().numpy()
    if isinstance(repr_, TriBlock):
        scores = np.zeros(n, dtype=np.float64)
        base = 1.0 / floor**2
        scores[:] = (n - 1) * base
        d = repr_.dense
        if repr_.dense_count:
            if isinstance(d, PairMap):
                di, dj, dv = d.i, d.j, d.v
            else:  # any Mapping {(i, j): v}, as proximity.py:455-466 reads it
                keys = list(d.keys())
                di = np.fromiter((k[0] for k in keys), dtype=np.int64, count=len(keys))
                dj = np.fromiter((k[1] for k in keys), dtype=np.int64, count=len(keys))
                dv = np.fromiter((d[k] for k in keys), dtype=np.float64, count=len(keys))
            adj = 1.0 / np.maximum(dv, floor) ** 2 - base
            np.add.at(scores, di, adj)
            np.add.at(scores, dj, adj)
        if repr_.sparse_count:
            adj = 1.0 / np.maximum(repr_.sparse_v, floor) ** 2 - base
            np.add.at(scores, repr_.sparse_i, adj)
            np.add.at(scores, repr_.sparse_j, adj)
        return scores / (n - 1)
    if isinstance(repr_, LowRankQuantized):
        dq = repr_.dequantized_device()
        r = int(dq.shape[1])
        scores = torch.empty(n, dtype=torch.float64, device=dq.device)
        with region("outlier"):
            _lib.call("rfxc_outlier_lowrank", _lib.ptr(dq), n, r, float(floor), _lib.ptr(scores),
                      _lib.stream_handle())
        return scores.cpu().numpy()
    raise RfxError(f"unknown proximity representation {type(repr_)!r}")


# ------------------------------------------------------------------ accessors
def entry(repr_, i: int, j: int) -> float:
    return repr_.entry(i, j)


# ------------------------------------------------------------------- planner
PLAN_MAXNODE, PLAN_FEATURES, PLAN_CLASSES = 1000, 50, 3
GiB = 2**30


def memory_plan(n: int, tree_count: int | None = None, rank: int | None = None,
                mode: str | None = None, backend: str | None = None,
                retention: float = DEFAULT_RETENTION, n_features: int = PLAN_FEATURES,
                maxnode: int = PLAN_MAXNODE, n_classes: int = PLAN_CLASSES) -> dict:
    """Closed-form byte counts and feasibility verdicts, same keys and
    arithmetic as the reference planner (proximity.py:500-595); carried by
    BudgetError."""
    if n < 1:
        raise DataError("memory_plan needs n >= 1")
    square = 8 * n * n
    tri = int(square * 0.5 * retention)

    def lr(rk, m):
        return {"two_factor": int(2 * n * rk * BYTES_PER_ELEMENT[m]),
                "single_factor": int(n * rk * BYTES_PER_ELEMENT[m])}

    table = {m: lr(32, m) for m in MODES}
    B = tree_count if tree_count is not None else 10_000
    model = {"training_data": n * n_features * 4, "tree_structures": 2 * maxnode * B * 4,
             "node_status": maxnode * B * 4, "split_values": maxnode * B * 4,
             "split_variables": maxnode * B * 4, "node_classes": maxnode * B * 4,
             "class_populations": n_classes * maxnode * B * 4,
             "oob_tracking": n * n_classes * 4}
    model["subtotal"] = sum(model.values())
    imp = {"overall": n_features * 4, "local_per_sample": n * 4,
           "local_matrix": n * n_features * 4, "importance_sd": n_features * 4}
    imp["subtotal"] = sum(imp.values())
    cand = {"full": square, "triblock": tri, "lowrank_i8_r32": table["i8"]["two_factor"],
            "lowrank_nf4_r32": table["nf4"]["two_factor"]}
    f32g = {k_: v <= 0.8 * 32 * GiB for k_, v in cand.items()}
    f12g = {k_: v <= 0.8 * 12 * GiB for k_, v in cand.items()}
    if n <= 5000:
        rec = "full or triblock"
    elif f32g["triblock"]:
        rec = "triblock"
    else:
        rec = "lowrank (i8 for speed, nf4 for minimum memory)"
    plan = {"samples": n, "trees": B, "full_headline_bytes": square,
            "full_packed_bytes": 8 * _packed_len(n), "triblock_bytes": tri,
            "triblock_retention": retention, "lowrank_r32_bytes": table, "model": model,
            "importance": imp, "feasible_32gb": f32g, "feasible_12gb": f12g,
            "recommended": rec}
    if rank is not None and mode is not None:
        req = lr(rank, mode)
        plan["requested"] = {"backend": backend or "lowrank", "rank": rank, "mode": mode,
                             "bytes": req, "compression_vs_full": square / max(req["two_factor"], 1)}
    elif backend in ("full", "triblock"):
        chosen = {"full": 8 * _packed_len(n), "triblock": tri}[backend]
        plan["requested"] = {"backend": backend, "bytes": {"stored": chosen},
                             "compression_vs_full": square / max(chosen, 1)}
    return plan
