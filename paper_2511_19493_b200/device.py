"""Device-resident state of the proximity path (HBM layout) and the thin
orchestration of the C ABI calls.

HBM layout (one process per GPU):
  values   f32 (p, n) column-major (f64 if any value is not f32-exact)
  nodes    packed node records of the local trees, 8 B (f32) / 16 B (f64)
  codes_tm (Bl, n) int32  — traversal output, bucketing input
  codes_nb (n, Bl) int32  — LeafMembership.codes layout, sketch/pairs input
  perm     (Bl, n) int32  — samples sorted by leaf per tree (K2)
  seg      (sum L + 1) int64 — start of every leaf's run in perm
  leaf_base (Bl + 1) int64 — global leaf id of each tree's leaf 0
Everything stays on the device between calls; host arrays are produced
only when a caller reads them.
"""

from __future__ import annotations

import warnings

import numpy as np

from . import _lib
from .errors import DataError
from .profiling import region


def _torch():
    import torch
    return torch


def relayout_siblings(status, split_var, threshold, cat_mask, left, right):
    """Renumber one tree breadth-first so that right == left + 1 for every
    internal node (the packed layout stores only the left child).  Trees
    grown by the trainer already satisfy this (_kernels.py:313-317); only
    hand-built trees take this path.  Terminal order (and therefore the
    dense leaf codes of forest.py:95-99) is preserved by carrying the
    original node id and remapping codes after packing."""
    nc = len(status)
    order = [0]
    newid = {0: 0}
    q = 0
    while q < len(order):
        old = order[q]
        q += 1
        if status[old] == 0:
            for ch in (left[old], right[old]):
                newid[int(ch)] = len(order)
                order.append(int(ch))
    order = np.asarray(order, dtype=np.int64)
    if len(order) != nc:
        raise DataError("tree has unreachable nodes")
    inv = np.empty(nc, dtype=np.int64)
    inv[order] = np.arange(nc)
    st = status[order]
    lf = np.where(st == 0, inv[np.maximum(left[order], 0)], -1).astype(np.int32)
    return (st, split_var[order], threshold[order], cat_mask[order], lf, order)


class DeviceForest:
    """Packed node records of trees [tree_lo, tree_hi) on the current GPU."""

    def __init__(self, forest, tree_lo: int = 0, tree_hi: int | None = None):
        torch = _torch()
        dev = _lib.require_cuda()
        trees = forest.trees
        tree_hi = len(trees) if tree_hi is None else tree_hi
        self.tree_lo, self.tree_hi = tree_lo, tree_hi
        self.p = int(forest.p)
        col_cat = np.ascontiguousarray(getattr(forest, "col_cat", trees[0].col_cat),
                                       dtype=np.uint8)
        st, sv, th, cm, lf, counts, code_maps = [], [], [], [], [], [], []
        for t in trees[tree_lo:tree_hi]:
            s = np.asarray(t.status, np.int8)
            l_ = np.asarray(t.left, np.int32)
            r_ = np.asarray(t.right, np.int32)
            internal = s == 0
            if np.all(r_[internal] == l_[internal] + 1):
                st.append(s); sv.append(np.asarray(t.split_var, np.int32))
                th.append(np.asarray(t.threshold, np.float64))
                cm.append(np.asarray(t.cat_mask, np.int64)); lf.append(l_)
                code_maps.append(None)
            else:
                s2, sv2, th2, cm2, lf2, order = relayout_siblings(
                    s, np.asarray(t.split_var, np.int32), np.asarray(t.threshold, np.float64),
                    np.asarray(t.cat_mask, np.int64), l_, r_)
                st.append(s2); sv.append(sv2); th.append(th2); cm.append(cm2); lf.append(lf2)
                # packed code (leaf ordinal in new order) -> reference code
                ref_code = np.cumsum(s == 1) - 1
                code_maps.append(ref_code[order[s2 == 1]].astype(np.int32))
            counts.append(len(s))
        self.relaid = any(m is not None for m in code_maps)
        leaf_code = None
        if self.relaid:  # explicit per-node codes in the reference's terminal order
            parts = []
            for s_, m in zip(st, code_maps):
                c = np.full(len(s_), -1, dtype=np.int32)
                c[s_ == 1] = m if m is not None else np.arange(int((s_ == 1).sum()))
                parts.append(c)
            leaf_code = np.concatenate(parts)
        self.node_counts = np.asarray(counts, dtype=np.int64)
        self.leaf_counts = np.asarray([int((a == 1).sum()) for a in st], dtype=np.int32)
        off = np.zeros(len(counts) + 1, dtype=np.int64)
        off[1:] = np.cumsum(self.node_counts)
        self.total_nodes = int(off[-1])
        up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        self._raw = dict(status=up(np.concatenate(st)), split_var=up(np.concatenate(sv)),
                         threshold=up(np.concatenate(th)), cat_mask=up(np.concatenate(cm)),
                         left=up(np.concatenate(lf)))
        self.leaf_code = up(leaf_code) if leaf_code is not None else None
        self.node_off = up(off)
        self.col_cat = up(col_cat)
        self._packed = {}
        fb = max(1, int(np.ceil(np.log2(max(self.p, 2)))))
        self.f32_ok = int(self.node_counts.max()) < (1 << (31 - fb))

    @property
    def ntree(self) -> int:
        return self.tree_hi - self.tree_lo

    def packed(self, layout: int):
        torch = _torch()
        if layout not in self._packed:
            nbytes = 8 if layout == _lib.NODES_F32 else 16
            nodes = torch.empty(self.total_nodes * nbytes, dtype=torch.uint8,
                                device=self.node_off.device)
            lc = torch.empty(self.ntree, dtype=torch.int32, device=self.node_off.device)
            r = self._raw
            _lib.call("rfxc_forest_pack", _lib.ptr(r["status"]), _lib.ptr(r["split_var"]),
                      _lib.ptr(r["threshold"]), _lib.ptr(r["cat_mask"]), _lib.ptr(r["left"]),
                      _lib.ptr(self.leaf_code), _lib.ptr(self.node_off), self.ntree, self.total_nodes,
                      _lib.ptr(self.col_cat), self.p, layout, _lib.ptr(nodes), _lib.ptr(lc),
                      _lib.stream_handle())
            self._packed[layout] = nodes
        return self._packed[layout]


class DeviceValues:
    """Dataset.values on the GPU: f32 when every value is f32-exact."""

    def __init__(self, values: np.ndarray):
        torch = _torch()
        dev = _lib.require_cuda()
        vals = np.asfortranarray(values, dtype=np.float64)
        self.n, self.p = vals.shape
        # F-order (n, p) is exactly (p, n) row-major
        with warnings.catch_warnings():  # read-only Dataset.values: torch only reads it
            warnings.simplefilter("ignore", UserWarning)
            self.f64 = torch.from_numpy(vals.T).to(dev)
        self.f32 = torch.empty((self.p, self.n), dtype=torch.float32, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("rfxc_values_to_f32", _lib.ptr(self.f64), self.n * self.p,
                  _lib.ptr(self.f32), _lib.ptr(flag), _lib.stream_handle())
        self.exact_f32 = int(flag.item()) == 0


class DeviceMembership:
    """Leaf codes of trees [tree_lo, tree_hi) of a B-tree forest, plus the
    lazily built per-tree leaf buckets."""

    def __init__(self, codes_nb, codes_tm, leaf_counts: np.ndarray, tree_lo: int, tree_hi: int,
                 B: int):
        torch = _torch()
        self.codes_nb = codes_nb
        self.codes_tm = codes_tm
        self.n = int(codes_nb.shape[0])
        self.tree_lo, self.tree_hi, self.B = tree_lo, tree_hi, B
        self.leaf_counts = np.ascontiguousarray(leaf_counts, dtype=np.int32)
        base = np.zeros(len(leaf_counts) + 1, dtype=np.int64)
        base[1:] = np.cumsum(self.leaf_counts)
        self.leaf_base_host = base
        self.leaf_base = torch.from_numpy(base).to(codes_nb.device)
        self.total_leaves = int(base[-1])
        self._perm = None
        self._seg = None

    @property
    def Bl(self) -> int:
        return self.tree_hi - self.tree_lo

    @property
    def is_shard(self) -> bool:
        return self.Bl != self.B

    def buckets(self):
        """K2 (once): perm (Bl, n) and seg (sum L + 1)."""
        torch = _torch()
        if self._perm is None:
            dev = self.codes_nb.device
            perm = torch.empty((self.Bl, self.n), dtype=torch.int32, device=dev)
            seg = torch.empty(self.total_leaves + 1, dtype=torch.int64, device=dev)
            maxl = int(self.leaf_counts.max())
            scratch = torch.empty(max(self.total_leaves, 1), dtype=torch.int32, device=dev)
            with region("bucket"):
                _lib.call("rfxc_bucket", _lib.ptr(self.codes_tm), self.n, self.Bl,
                          _lib.ptr(self.leaf_base), maxl, _lib.ptr(perm), _lib.ptr(seg),
                          _lib.ptr(scratch), _lib.stream_handle())
            self._perm, self._seg = perm, seg
        return self._perm, self._seg

    @classmethod
    def from_host(cls, codes: np.ndarray, leaf_counts: np.ndarray):
        torch = _torch()
        dev = _lib.require_cuda()
        codes = np.ascontiguousarray(codes, dtype=np.int32)
        lc = np.ascontiguousarray(leaf_counts, dtype=np.int32)
        n, B = codes.shape
        if lc.shape != (B,):
            raise DataError("leaf_counts length does not match the tree count")
        if n and (codes.min() < 0 or np.any(codes.max(axis=0) >= lc)):
            raise DataError("leaf code out of range for its tree's leaf_count")
        nb = torch.from_numpy(codes).to(dev)
        tm = torch.empty((B, n), dtype=torch.int32, device=dev)
        _lib.call("rfxc_transpose_i32", _lib.ptr(nb), n, B, _lib.ptr(tm), _lib.stream_handle())
        return cls(nb, tm, lc, 0, B, B)


def traverse(dforest: DeviceForest, dvalues: DeviceValues) -> DeviceMembership:
    """K1: codes of every sample in every local tree (tm and nb layouts)."""
    torch = _torch()
    use_f32 = dvalues.exact_f32 and dforest.f32_ok
    layout = _lib.NODES_F32 if use_f32 else _lib.NODES_F64
    vals = dvalues.f32 if use_f32 else dvalues.f64
    n, Bl = dvalues.n, dforest.ntree
    dev = vals.device
    tm = torch.empty((Bl, n), dtype=torch.int32, device=dev)
    nodes = dforest.packed(layout)
    with region("leaf_codes"):
        _lib.call("rfxc_leaf_codes", _lib.ptr(nodes), _lib.ptr(dforest.node_off), layout,
                  dvalues.p, 0, Bl, _lib.ptr(vals), n, _lib.ptr(tm), _lib.stream_handle())
    nb = torch.empty((n, Bl), dtype=torch.int32, device=dev)
    _lib.call("rfxc_transpose_i32", _lib.ptr(tm), Bl, n, _lib.ptr(nb), _lib.stream_handle())
    return nb, tm, layout
