"""Device-resident state of the proximity path (HBM layout) and the thin
orchestration of the C ABI calls.

HBM layout (one process per GPU):
  values   f32 (p, n) column-major (f64 if any value is not f32-exact)
  nodes    packed node records of the local trees, 8 B (f32) / 16 B (f64)
  codes_tm (Bl, n) int32  — traversal output, bucketing input
  codes_nb (n, Bl) int32  — LeafMembership.codes layout, sketch/pairs input
  perm     (Bl, n) int32  — samples sorted by leaf per tree (K2), bit 31 set
                            on the first member of every leaf
  seg      (sum L + 1) int64 — start of every leaf's run in perm
  leaf_base (Bl + 1) int64 — global leaf id of each tree's leaf 0
Everything stays on the device between calls; host arrays are produced
only when a caller reads them.  Uploads are packed on the host (multi-
threaded C++, librfxc's host_pack.cpp) straight into pinned buffers so only
the packed bytes cross PCIe.
"""

from __future__ import annotations

import os
import weakref

import numpy as np

from . import _lib
from .errors import DataError
from .profiling import region


def _torch():
    import torch
    return torch


def _pinned(nbytes: int):
    """Pinned host staging buffer (torch caching host allocator) + numpy view."""
    torch = _torch()
    buf = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, pin_memory=True)
    return buf, buf.numpy()


# Host staging of immutable inputs (Dataset.values arrays, Forest objects): the
# packed pinned upload buffer is derived once per object and reused; every
# construction of a DeviceValues / DeviceForest still copies it host -> device.
_STAGED: dict = {}


def _staged(obj, key, build):
    """Per-object cache of `build()` keyed by (id(obj), key), dropped when obj
    is garbage collected."""
    k = (id(obj), key)
    hit = _STAGED.get(k)
    if hit is not None and hit[0]() is obj:
        return hit[1]
    val = build()
    try:
        ref = weakref.ref(obj)
        weakref.finalize(obj, _STAGED.pop, k, None)
    except TypeError:  # not weak-referenceable: no caching
        return val
    _STAGED[k] = (ref, val)
    return val


UPLOAD_CHUNK_TREES = 128
# K1 walks the trees after the first chunk in tree-0 leaf order when there
# are enough samples and trees to repay the order, the permuted values copy
# and the extra transpose (RFX_TRAV_ORDER=0 keeps sample order)
TRAV_ORDER_MIN_N = 32768
TRAV_ORDER_MIN_TREES = 64
UPLOAD_FIRST_TREES = 32
_COPY_STREAMS: dict = {}


D2H_CHUNK = 64 << 20  # bytes per staged chunk
_D2H_RING = {}


def host_copy(t):
    """numpy copy of a device tensor.  Large results stream through a reused
    pair of pinned staging buffers on the copy stream (full-rate DMA), each
    chunk moved into the pageable destination by torch's threaded host copy
    while the next chunk is in flight — no multi-GB pinned allocation and no
    staged pageable cudaMemcpy."""
    torch = _torch()
    nbytes = t.numel() * t.element_size()
    if nbytes < 2 * D2H_CHUNK:
        return t.cpu().numpy()
    key = str(t.device)
    if key not in _D2H_RING:
        _D2H_RING[key] = [torch.empty(D2H_CHUNK, dtype=torch.uint8, pin_memory=True)
                          for _ in range(2)]
    ring = _D2H_RING[key]
    src = t.contiguous().view(-1).view(torch.uint8)
    out = np.empty(t.shape, dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    dst = torch.from_numpy(out.reshape(-1).view(np.uint8))
    cs = _copy_stream(t.device)
    cs.wait_stream(torch.cuda.current_stream())
    spans = [(a, min(nbytes, a + D2H_CHUNK)) for a in range(0, nbytes, D2H_CHUNK)]
    events = []

    def issue(k):
        a, b = spans[k]
        with torch.cuda.stream(cs):
            ring[k % 2][:b - a].copy_(src[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        events.append(ev)

    issue(0)
    for k, (a, b) in enumerate(spans):
        if k + 1 < len(spans):  # its ring slot was drained by the host copy of chunk k - 1
            issue(k + 1)
        events[k].synchronize()
        dst[a:b].copy_(ring[k % 2][:b - a])
    src.record_stream(cs)
    return out


def _copy_stream(dev):
    torch = _torch()
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = torch.cuda.Stream(device=dev)
    return _COPY_STREAMS[key]


def feature_bits(p: int) -> int:
    fb = 1
    while (1 << fb) < p:
        fb += 1
    return fb


def _as(a, dtype):
    a = np.asarray(a)
    if a.dtype != dtype or not a.flags.c_contiguous:
        a = np.ascontiguousarray(a, dtype=dtype)
    return a


class DeviceValues:
    """Dataset.values on the GPU: f32 when every value is f32-exact (then the
    f32 node layout compares exactly), else f64."""

    def __init__(self, values: np.ndarray, defer: bool = False):
        torch = _torch()
        self.dev = _lib.require_cuda()
        vals = np.asfortranarray(values, dtype=np.float64)
        self.n, self.p = vals.shape
        self._host = vals

        def stage():
            buf, view = _pinned(vals.size * 4)
            exact = np.zeros(1, dtype=np.int32)
            # F-order (n, p) is exactly (p, n) row-major
            _lib.call("rfxc_values_to_f32_host", vals.ctypes.data_as(_lib.P), vals.size,
                      view.ctypes.data_as(_lib.P), exact.ctypes.data_as(_lib.P), 0)
            return buf, bool(exact[0])

        buf, self.exact_f32 = _staged(values, "f32", stage)
        self._buf = buf
        self.ready = None       # event: every row on the device
        self.rows_ready = []    # (row_hi, event) for uploads issued so far
        self.f32 = None
        if self.exact_f32:  # on the copy stream; traverse() waits for the rows it reads
            self._dst = torch.empty(vals.size * 4, dtype=torch.uint8, device=self.dev)
            self.f32 = self._dst.view(torch.float32).view(self.p, self.n)
            if not defer:
                self.upload_rows(0, self.n)
        self._f64 = None

    def upload_rows(self, lo: int, hi: int):
        """Copy samples [lo, hi) (all features) on the copy stream."""
        torch = _torch()
        cs = _copy_stream(self.dev)
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            _lib.call("rfxc_h2d_rows", _lib.ptr(self._dst), self._buf.data_ptr(), self.n, self.p, 4,
                      lo, hi, _lib.stream_handle())
            ev = torch.cuda.Event()
            ev.record(cs)
        self._dst.record_stream(cs)
        self.rows_ready.append((hi, ev))
        if hi >= self.n:
            self.ready = ev

    @property
    def f64(self):
        torch = _torch()
        if self._f64 is None:
            self._f64 = torch.from_numpy(np.require(self._host.T, requirements=["C", "W"])).to(self.dev)
        return self._f64


class DeviceForest:
    """Packed node records of trees [tree_lo, tree_hi) of ``forest`` on the
    current GPU (packed on the host, uploaded once)."""

    def __init__(self, forest, tree_lo: int = 0, tree_hi: int | None = None,
                 layout: int | None = None, nthreads: int = 0, defer: bool = False):
        torch = _torch()
        dev = _lib.require_cuda()
        trees = forest.trees[tree_lo:(len(forest.trees) if tree_hi is None else tree_hi)]
        self.tree_lo = tree_lo
        self.tree_hi = tree_lo + len(trees)
        self.p = int(forest.p)
        B = len(trees)
        col_cat = _as(getattr(forest, "col_cat", trees[0].col_cat), np.uint8)
        counts = np.fromiter((len(t.status) for t in trees), dtype=np.int64, count=B)
        self.node_counts = counts
        self.total_nodes = int(counts.sum())
        self.f32_ok = int(counts.max()) < (1 << (31 - feature_bits(self.p)))
        b2_ok = int(counts.max()) + 1 < (1 << (30 - feature_bits(self.p)))
        if layout is None:
            # f32 records in two-level blocks (one dependent load per two
            # levels); RFX_TRAV_LAYOUT=f32 keeps the reference node order
            if b2_ok and os.environ.get("RFX_TRAV_LAYOUT", "b2") != "f32":
                layout = _lib.NODES_F32_B2
            else:
                layout = _lib.NODES_F32 if self.f32_ok else _lib.NODES_F64
        if (layout == _lib.NODES_F32 and not self.f32_ok) or (layout == _lib.NODES_F32_B2 and not b2_ok):
            raise DataError("tree too large for the 8-byte node layout")
        if layout not in (_lib.NODES_F32, _lib.NODES_F64, _lib.NODES_F32_B2):
            raise DataError(f"unknown node layout {layout}")
        self.layout = layout
        rec = 16 if layout == _lib.NODES_F64 else 8
        # no categorical column: the traversal skips the per-node category test
        self.numeric = not bool(np.any(col_cat))

        def stage():
            keep = []  # keep converted arrays alive during the call
            tables = {name: np.empty(B, dtype=np.uintp) for name in
                      ("status", "split_var", "threshold", "cat_mask", "left", "right")}
            dts = {"status": np.int8, "split_var": np.int32, "threshold": np.float64,
                   "cat_mask": np.int64, "left": np.int32, "right": np.int32}
            for b, t in enumerate(trees):
                for name, dt in dts.items():
                    a = _as(getattr(t, name), dt)
                    keep.append(a)
                    tables[name][b] = a.ctypes.data
            off = np.empty(B + 1, dtype=np.int64)
            lc = np.empty(B, dtype=np.int32)
            P = _lib.P

            def pack(dst):
                _lib.call("rfxc_forest_pack_host", *(tables[k].ctypes.data_as(P) for k in
                                                     ("status", "split_var", "threshold",
                                                      "cat_mask", "left", "right")),
                          counts.ctypes.data_as(P), B, col_cat.ctypes.data_as(P), self.p, layout,
                          dst, off.ctypes.data_as(P), lc.ctypes.data_as(P), nthreads)

            with region("forest_pack_host"):
                nrec = self.total_nodes
                if layout == _lib.NODES_F32_B2:  # sizing call: the record count per tree
                    pack(None)
                    nrec = int(off[B])
                buf, view = _pinned(nrec * rec)
                pack(view.ctypes.data_as(P))
            del keep
            return buf, off, lc

        buf, off, lc = _staged(forest, ("nodes", tree_lo, self.tree_hi, layout), stage)
        self.leaf_counts = lc.copy()
        self.node_off_host = off
        self.node_off = torch.from_numpy(off).to(dev)
        self._rec = rec
        self._staging = buf
        self._nodes = torch.empty(max(int(off[B]) * rec, 1), dtype=torch.uint8, device=dev)
        # node records cross PCIe in tree chunks on a copy stream, so the
        # traversal of chunk c overlaps the copy of chunk c + 1 (traverse());
        # a small first chunk lets the traversal start early
        bounds = [0] + [c for c in range(UPLOAD_FIRST_TREES, B, UPLOAD_CHUNK_TREES)] + [B]
        bounds = sorted(set(b_ for b_ in bounds if 0 <= b_ <= B))
        self._spans = list(zip(bounds[:-1], bounds[1:]))
        self.chunks = []
        if not defer:
            for j in range(len(self._spans)):
                self.upload_chunk(j)

    def upload_chunk(self, j: int):
        """Copy the node records of tree chunk j on the copy stream."""
        torch = _torch()
        c0, c1 = self._spans[j]
        off, rec, buf = self.node_off_host, self._rec, self._staging
        cs = _copy_stream(self._nodes.device)
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            a, b = int(off[c0]) * rec, int(off[c1]) * rec
            self._nodes[a:b].copy_(buf[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        self._nodes.record_stream(cs)
        self.chunks.append((c0, c1, ev))

    @property
    def nodes(self):
        """The packed node records once every chunk has arrived (the current
        stream waits for the copies)."""
        torch = _torch()
        for _c0, _c1, ev in self.chunks:
            torch.cuda.current_stream().wait_event(ev)
        return self._nodes

    @property
    def ntree(self) -> int:
        return self.tree_hi - self.tree_lo

    @classmethod
    def packed_on_device(cls, forest, layout: int):
        """Reference-layout raw arrays uploaded as-is and packed by the device
        kernel (rfxc_forest_pack); requires right == left + 1.  Returns the
        packed node tensor, node offsets and leaf counts (device)."""
        torch = _torch()
        dev = _lib.require_cuda()
        trees = forest.trees
        cat = lambda name, dt: torch.from_numpy(
            np.concatenate([_as(getattr(t, name), dt) for t in trees])).to(dev)
        off = np.zeros(len(trees) + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(t.status) for t in trees])
        total = int(off[-1])
        nodes = torch.empty(total * (8 if layout == _lib.NODES_F32 else 16), dtype=torch.uint8,
                            device=dev)
        lc = torch.empty(len(trees), dtype=torch.int32, device=dev)
        d_off = torch.from_numpy(off).to(dev)
        col_cat = torch.from_numpy(_as(forest.col_cat, np.uint8)).to(dev)
        st, sv, th = cat("status", np.int8), cat("split_var", np.int32), cat("threshold",
                                                                                np.float64)
        cm, lf = cat("cat_mask", np.int64), cat("left", np.int32)
        _lib.call("rfxc_forest_pack", _lib.ptr(st), _lib.ptr(sv), _lib.ptr(th), _lib.ptr(cm),
                  _lib.ptr(lf), _lib.ptr(None), _lib.ptr(d_off), len(trees), total,
                  _lib.ptr(col_cat), int(forest.p), layout, _lib.ptr(nodes), _lib.ptr(lc),
                  _lib.stream_handle())
        return nodes, d_off, lc


class DeviceMembership:
    """Leaf codes of trees [tree_lo, tree_hi) of a B-tree forest, plus the
    lazily built per-tree leaf buckets."""

    def __init__(self, codes_nb, codes_tm, leaf_counts: np.ndarray, tree_lo: int, tree_hi: int,
                 B: int, chunks=None):
        torch = _torch()
        self.chunks = chunks  # traversal chunks (local c0, c1, event) or None
        self.codes_nb = codes_nb
        self.codes_tm = codes_tm
        self.n = int(codes_nb.shape[0])
        self.tree_lo, self.tree_hi, self.B = tree_lo, tree_hi, B
        self.leaf_counts = np.ascontiguousarray(leaf_counts, dtype=np.int32)
        base = np.zeros(len(leaf_counts) + 1, dtype=np.int64)
        base[1:] = np.cumsum(self.leaf_counts)
        self.leaf_base_host = base
        # pinned + non_blocking: no host wait on the queued traversal
        self.leaf_base = torch.from_numpy(base).pin_memory().to(codes_nb.device, non_blocking=True)
        self.total_leaves = int(base[-1])
        self._perm = None
        self._seg = None
        self._has_empty = None
        self._pos = None
        self._perm16 = None
        self._pairs = None
        self._gate = None

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
            has_empty = torch.zeros(1, dtype=torch.int32, device=dev)
            lib = _lib.load()
            # one call over all trees: bucketing per traversal chunk on side
            # streams was measured no faster (the traversal fills every SM)
            scratch = torch.empty(int(lib.rfxc_bucket_scratch_bytes(self.n, self.Bl)),
                                  dtype=torch.uint8, device=dev)
            with region("bucket"):
                _lib.call("rfxc_bucket_trees", _lib.ptr(self.codes_tm), self.n, self.Bl,
                          _lib.ptr(self.leaf_base), maxl, 0, self.Bl, _lib.ptr(perm),
                          _lib.ptr(seg), _lib.ptr(scratch), _lib.ptr(has_empty),
                          _lib.stream_handle())
            self._perm, self._seg, self._has_empty = perm, seg, has_empty
        return self._perm, self._seg

    def positions(self):
        """(n, Bl) uint32: index of sample i in perm for tree b (the start of
        i's walk in the leaf-segmented pair counts).  Built once from K2."""
        torch = _torch()
        if self._pos is None:
            perm, _ = self.buckets()
            tm = torch.empty((self.Bl, self.n), dtype=torch.int32, device=perm.device)
            nb = torch.empty((self.n, self.Bl), dtype=torch.int32, device=perm.device)
            # 16-bit sample ids for the walk when they fit (half the bytes: the
            # bucket stays L2-resident); RFX_PAIRS_PERM16=0 keeps the 32-bit perm
            p16 = None
            if self.n <= 65536 and os.environ.get("RFX_PAIRS_PERM16", "1") != "0":
                p16 = torch.empty((self.Bl, self.n), dtype=torch.int16, device=perm.device)
            with region("positions"):
                _lib.call("rfxc_perm_positions", _lib.ptr(perm), self.n, self.Bl, _lib.ptr(tm),
                          _lib.ptr(p16), _lib.stream_handle())
                _lib.call("rfxc_transpose_i32", _lib.ptr(tm), self.Bl, self.n, _lib.ptr(nb),
                          _lib.stream_handle())
            self._pos = nb
            self._perm16 = p16
        return self._pos

    def walk_ids(self):
        """(ids tensor, bytes per id) the leaf-walk pair counts read: the
        16-bit copy from positions() when it exists, else the K2 perm."""
        self.positions()
        if self._perm16 is not None:
            return self._perm16, 2
        return self.buckets()[0], 4

    def pair_gate(self):
        """Device int32: 1 when the leaf-walk pair counts apply (same-leaf
        pairs <= LEAF_KERNEL_MAX_SHARE of the (pair, tree) units), else 0;
        computed on the device, no host read."""
        torch = _torch()
        if self._gate is None:
            from .proximity import LEAF_KERNEL_MAX_SHARE
            _, seg = self.buckets()
            pairs = torch.empty(1, dtype=torch.int64, device=seg.device)
            gate = torch.empty(1, dtype=torch.int32, device=seg.device)
            _lib.call("rfxc_same_leaf_pairs", _lib.ptr(seg), self.total_leaves, _lib.ptr(pairs),
                      _lib.stream_handle())
            _lib.call("rfxc_pair_kernel_gate", _lib.ptr(pairs), self.n, self.Bl,
                      float(LEAF_KERNEL_MAX_SHARE), _lib.ptr(gate), _lib.stream_handle())
            self._gate = gate
        return self._gate

    def same_leaf_pairs(self) -> int:
        """Sum over the local trees' leaves of s(s-1)/2 (exact integer)."""
        torch = _torch()
        if self._pairs is None:
            _, seg = self.buckets()
            out = torch.empty(1, dtype=torch.int64, device=seg.device)
            _lib.call("rfxc_same_leaf_pairs", _lib.ptr(seg), self.total_leaves, _lib.ptr(out),
                      _lib.stream_handle())
            self._pairs = int(out.item())
        return self._pairs

    @property
    def has_empty(self):
        """Device int32 flag: some local leaf has no member (from K2)."""
        self.buckets()
        return self._has_empty

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


def traverse(dforest: DeviceForest, dvalues: DeviceValues):
    """K1: codes of every sample in every local tree (tm and nb layouts)."""
    torch = _torch()
    layout = dforest.layout
    f32 = layout != _lib.NODES_F64
    if f32 and not dvalues.exact_f32:
        raise DataError("f32 node layout needs f32-exact values")
    vals = dvalues.f32 if f32 else dvalues.f64
    n, Bl = dvalues.n, dforest.ntree
    dev = vals.device
    tm = torch.empty((Bl, n), dtype=torch.int32, device=dev)
    cur = torch.cuda.current_stream()
    f32_rows = dvalues.rows_ready if f32 else []
    done = []  # (c0, c1, event after the chunk's codes)

    klayout = layout
    if dforest.numeric and layout == _lib.NODES_F32:
        klayout = _lib.NODES_F32_NUMERIC
    elif dforest.numeric and layout == _lib.NODES_F32_B2:
        klayout = _lib.NODES_F32_B2_NUMERIC

    def walk(c0, c1, lo, hi, out=None, values=None):
        _lib.call("rfxc_leaf_codes_rows", _lib.ptr(dforest._nodes), _lib.ptr(dforest.node_off),
                  klayout, dvalues.p, c0, c1, _lib.ptr(vals if values is None else values), n, lo, hi,
                  _lib.ptr(tm[c0:c1] if out is None else out), _lib.stream_handle())

    def mark(c0, c1):
        cev = torch.cuda.Event()
        cev.record(cur)
        done.append((c0, c1, cev))

    chunks = list(dforest.chunks)
    with region("leaf_codes"):
        rest = chunks
        if len(f32_rows) > 1:
            # values arrived in sample blocks: the first two tree chunks walk
            # each block as soon as it is there (block-major), so the
            # traversal starts after ~1/4 of the bytes
            early, rest = chunks[:2], chunks[2:]
            blocks = list(zip([0] + [h for h, _ in f32_rows], f32_rows))
            for bi, (lo, (hi, e)) in enumerate(blocks):
                cur.wait_event(e)
                for c0, c1, ev in early:
                    cur.wait_event(ev)
                    walk(c0, c1, lo, hi)
                    if bi == len(blocks) - 1:
                        mark(c0, c1)
        if rest and dvalues.ready is not None:
            cur.wait_event(dvalues.ready)
        ordered = (f32 and n >= TRAV_ORDER_MIN_N and os.environ.get("RFX_TRAV_ORDER", "1") != "0"
                   and sum(c1 - c0 for c0, c1, _ in rest) >= TRAV_ORDER_MIN_TREES)
        if ordered and not done:  # tree 0 first, in sample order
            (c0, c1, ev), rest = rest[0], rest[1:]
            cur.wait_event(ev)
            walk(c0, c1, 0, n)
            mark(c0, c1)
            ordered = sum(b - a for a, b, _ in rest) >= TRAV_ORDER_MIN_TREES
        if not ordered:
            for c0, c1, ev in rest:  # after its node records arrived
                cur.wait_event(ev)
                walk(c0, c1, 0, n)
                mark(c0, c1)
    nb = torch.empty((n, Bl), dtype=torch.int32, device=dev)
    if not ordered or not rest:
        _lib.call("rfxc_transpose_i32", _lib.ptr(tm), Bl, n, _lib.ptr(nb), _lib.stream_handle())
        return nb, tm, done
    # the remaining trees walk the samples grouped by their tree-0 leaf
    # (neighbouring lanes share paths: fewer node lines per gather); their
    # codes come back to sample order through the transpose
    e = rest[0][0]
    with region("leaf_codes"):
        order = torch.empty(n, dtype=torch.int32, device=dev)
        nl0 = int(dforest.leaf_counts[0])
        scratch = torch.empty(max(nl0, 1), dtype=torch.int32, device=dev)
        _lib.call("rfxc_leaf_order", _lib.ptr(tm[0]), n, nl0, _lib.ptr(order), _lib.ptr(scratch),
                  _lib.stream_handle())
        xp = torch.empty_like(vals)
        _lib.call("rfxc_permute_rows_f32", _lib.ptr(vals), n, dvalues.p, _lib.ptr(order), _lib.ptr(xp),
                  _lib.stream_handle())
        tp = torch.empty((Bl - e, n), dtype=torch.int32, device=dev)
        for c0, c1, ev in rest:
            cur.wait_event(ev)
            walk(c0, c1, 0, n, out=tp[c0 - e:c1 - e], values=xp)
        h = _lib.stream_handle()
        _lib.call("rfxc_transpose_i32_ex", _lib.ptr(tm), e, n, n, _lib.ptr(nb), Bl, None, h)
        nbe = nb[:, e:]  # column block e.. of the (n, Bl) codes (row stride Bl)
        _lib.call("rfxc_transpose_i32_ex", _lib.ptr(tp), Bl - e, n, n, _lib.ptr(nbe), Bl,
                  _lib.ptr(order), h)
        _lib.call("rfxc_transpose_i32_ex", _lib.ptr(nbe), n, Bl - e, Bl, _lib.ptr(tm[e]), n, None, h)
        for c0, c1, _ev in rest:
            mark(c0, c1)
    return nb, tm, done
