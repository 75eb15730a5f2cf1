"""Forest types, the RFX1 file format, and the input producer.

The proximity path's input is "the forest grown by the reference's CPU
trainer with the same seed".  ``Tree`` / ``Forest`` / ``TrainConfig``
mirror forest.py:42-130 field for field (the proximity functions accept the
reference's own objects too: only the node arrays are read).  ``train``
restates ``rfx.train`` (forest.py:262-302) in C++ (csrc/host/rfx_train.cpp),
byte-identical in RFX1 form, so the GPU box — where the reference does not
exist — can regenerate the exact input forest from the seed.  Training is
not on the hot path and is never timed.
"""

from __future__ import annotations

import ctypes
import io
import os
import struct
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .dataset import Dataset, column_arrays
from .errors import DataError, RfxError

_MAGIC = b"RFX1"
_VERSION = 1


@dataclass
class TrainConfig:
    ntree: int = 500
    mtry: int | None = None
    iseed: int = 1
    min_node_size: int = 1
    max_nodes: int | None = None
    casewise: bool = False

    def resolved(self, n: int, p: int) -> "TrainConfig":
        """forest.py:53-64."""
        if self.ntree < 1:
            raise DataError(f"ntree must be >= 1, got {self.ntree}")
        if self.min_node_size < 1:
            raise DataError(f"min_node_size must be >= 1, got {self.min_node_size}")
        mtry = self.mtry if self.mtry is not None else max(1, int(np.sqrt(p)))
        if not 1 <= mtry <= p:
            raise DataError(f"mtry must be in [1, {p}], got {mtry}")
        max_nodes = self.max_nodes if self.max_nodes is not None else 2 * n + 1
        if max_nodes < 1:
            raise DataError("max_nodes must be >= 1")
        return replace(self, mtry=mtry, max_nodes=max_nodes)


@dataclass
class Tree:
    status: np.ndarray
    split_var: np.ndarray
    threshold: np.ndarray
    cat_mask: np.ndarray
    left: np.ndarray
    right: np.ndarray
    node_class: np.ndarray
    class_pops: np.ndarray
    node_raw: np.ndarray
    node_weight: np.ndarray
    col_cat: np.ndarray

    @property
    def node_count(self) -> int:
        return len(self.status)

    @property
    def leaf_count(self) -> int:
        return int((self.status == 1).sum())

    def leaf_codes(self) -> np.ndarray:
        codes = np.cumsum(self.status == 1).astype(np.int32) - 1
        codes[self.status == 0] = -1
        return codes


@dataclass
class BootstrapRecord:
    counts: np.ndarray  # (B, n) int32

    @property
    def oob_mask(self) -> np.ndarray:
        return self.counts == 0


@dataclass
class Forest:
    trees: tuple
    bootstrap: BootstrapRecord
    config: TrainConfig
    n: int
    p: int
    class_count: int
    col_cat: np.ndarray
    col_levels: np.ndarray
    oob_votes: np.ndarray

    @property
    def ntree(self) -> int:
        return len(self.trees)


# ------------------------------------------------------------------ trainer
_train_lib = None


def _tlib():
    global _train_lib
    if _train_lib is None:
        if not os.path.exists(_lib.TRAIN_LIB_PATH):
            raise RfxError(f"{_lib.TRAIN_LIB_PATH} missing: run build()")
        L = ctypes.CDLL(_lib.TRAIN_LIB_PATH)
        P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.rfxt_train.restype = P
        L.rfxt_train.argtypes = [P, I64, I32, P, I32, P, P, I32, I32, I32, I64, I32, I64, I32]
        L.rfxt_last_error.restype = ctypes.c_char_p
        L.rfxt_node_counts.argtypes = [P, P]
        L.rfxt_copy.argtypes = [P] * 13
        L.rfxt_free.argtypes = [P]
        _train_lib = L
    return _train_lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def train(dataset: Dataset, config: TrainConfig, nthreads: int = 0,
          trees: tuple | None = None) -> Forest:
    """Grow the forest exactly as rfx.train does (forest.py:262-302).

    ``trees=(lo, hi)`` grows only that tree range of the ``config.ntree``
    forest (tree t is seeded by iseed + t, so a shard's trees are identical to
    the whole forest's); the returned Forest then holds hi - lo trees and its
    OOB votes cover those trees only."""
    cfg = config.resolved(dataset.n, dataset.p)
    col_cat, col_levels = column_arrays(dataset.columns)
    n, p, C = dataset.n, dataset.p, dataset.class_count
    lo, hi = (0, cfg.ntree) if trees is None else (int(trees[0]), int(trees[1]))
    if not 0 <= lo < hi <= cfg.ntree:
        raise DataError(f"tree range {trees} outside [0, {cfg.ntree})")
    B = hi - lo
    vals = np.asfortranarray(dataset.values, dtype=np.float64)
    labels = np.ascontiguousarray(dataset.labels, dtype=np.int32)
    L = _tlib()
    h = L.rfxt_train(_p(vals), n, p, _p(labels), C, _p(col_cat), _p(col_levels), lo, B,
                     cfg.mtry, cfg.iseed, cfg.min_node_size, cfg.max_nodes, nthreads)
    if not h:
        raise RfxError(L.rfxt_last_error().decode())
    try:
        counts = np.empty(B, dtype=np.int64)
        L.rfxt_node_counts(h, _p(counts))
        tot = int(counts.sum())
        status = np.empty(tot, np.int8)
        split_var = np.empty(tot, np.int32)
        threshold = np.empty(tot, np.float64)
        cat_mask = np.empty(tot, np.int64)
        left = np.empty(tot, np.int32)
        right = np.empty(tot, np.int32)
        node_class = np.empty(tot, np.int32)
        class_pops = np.empty(tot * C, np.int64)
        node_raw = np.empty(tot, np.int32)
        node_weight = np.empty(tot, np.int64)
        inbag = np.empty((B, n), np.int32)
        votes = np.empty((n, C), np.int64)
        L.rfxt_copy(h, _p(status), _p(split_var), _p(threshold), _p(cat_mask), _p(left),
                    _p(right), _p(node_class), _p(class_pops), _p(node_raw),
                    _p(node_weight), _p(inbag), _p(votes))
    finally:
        L.rfxt_free(h)
    off = np.concatenate([[0], np.cumsum(counts)])
    shard = None if (lo, hi) == (0, cfg.ntree) else (lo, hi, cfg.ntree)
    trees = []
    for b in range(B):
        s, e = int(off[b]), int(off[b + 1])
        trees.append(Tree(status[s:e].copy(), split_var[s:e].copy(), threshold[s:e].copy(),
                          cat_mask[s:e].copy(), left[s:e].copy(), right[s:e].copy(),
                          node_class[s:e].copy(), class_pops[s * C:e * C].reshape(e - s, C),
                          node_raw[s:e].copy(), node_weight[s:e].copy(), col_cat))
    f = Forest(trees=tuple(trees), bootstrap=BootstrapRecord(inbag), config=cfg, n=n,
               p=p, class_count=C, col_cat=col_cat, col_levels=col_levels, oob_votes=votes)
    f.tree_range = shard  # (lo, hi, B_total) for a shard-grown forest, else None
    return f


# --------------------------------------------------------------- RFX1 format
def _w(buf, arr, dtype):
    buf.write(np.ascontiguousarray(arr, dtype=dtype).tobytes())


def forest_to_bytes(forest) -> bytes:
    """Versioned little-endian layout of forest.py:373-398."""
    cfg = forest.config
    buf = io.BytesIO()
    buf.write(_MAGIC)
    buf.write(struct.pack("<I", _VERSION))
    buf.write(struct.pack("<qIIIIB3x", cfg.iseed, cfg.ntree, cfg.mtry, cfg.min_node_size,
                          cfg.max_nodes, 1 if cfg.casewise else 0))
    buf.write(struct.pack("<III", forest.n, forest.p, forest.class_count))
    _w(buf, forest.col_cat, "<u1")
    _w(buf, forest.col_levels, "<i4")
    for t in forest.trees:
        buf.write(struct.pack("<I", t.node_count))
        for arr, dt in ((t.status, "<i1"), (t.split_var, "<i4"), (t.threshold, "<f8"),
                        (t.cat_mask, "<u4"), (t.left, "<i4"), (t.right, "<i4"),
                        (t.node_class, "<i4"), (t.class_pops, "<i8"), (t.node_raw, "<i4"),
                        (t.node_weight, "<i8")):
            _w(buf, arr, dt)
    _w(buf, forest.bootstrap.counts, "<i4")
    _w(buf, forest.oob_votes, "<i8")
    return buf.getvalue()


def forest_from_bytes(data: bytes) -> Forest:
    """forest.py:420-457."""
    if data[:4] != _MAGIC:
        raise DataError(f"not a forest file (magic {data[:4]!r})")
    pos = 4
    (version,) = struct.unpack_from("<I", data, pos)
    pos += 4
    if version != _VERSION:
        raise DataError(f"unsupported forest format version {version}")
    iseed, ntree, mtry, mns, max_nodes, casewise = struct.unpack_from("<qIIIIB3x", data, pos)
    pos += struct.calcsize("<qIIIIB3x")
    n, p, C = struct.unpack_from("<III", data, pos)
    pos += 12

    def take(dt, count):
        nonlocal pos
        d = np.dtype(dt)
        a = np.frombuffer(data, dtype=d, count=count, offset=pos).copy()
        pos += d.itemsize * count
        return a

    col_cat = take("<u1", p).astype(np.uint8)
    col_levels = take("<i4", p).astype(np.int32)
    cfg = TrainConfig(ntree=ntree, mtry=mtry, iseed=iseed, min_node_size=mns,
                      max_nodes=max_nodes, casewise=bool(casewise))
    trees = []
    for _ in range(ntree):
        (nc,) = struct.unpack_from("<I", data, pos)
        pos += 4
        trees.append(Tree(take("<i1", nc).astype(np.int8), take("<i4", nc).astype(np.int32),
                          take("<f8", nc), take("<u4", nc).astype(np.int64),
                          take("<i4", nc).astype(np.int32), take("<i4", nc).astype(np.int32),
                          take("<i4", nc).astype(np.int32), take("<i8", nc * C).reshape(nc, C),
                          take("<i4", nc).astype(np.int32), take("<i8", nc), col_cat))
    counts = take("<i4", ntree * n).reshape(ntree, n).astype(np.int32)
    votes = take("<i8", n * C).reshape(n, C)
    if pos != len(data):
        raise DataError("trailing bytes in forest file")
    return Forest(trees=tuple(trees), bootstrap=BootstrapRecord(counts), config=cfg, n=n,
                  p=p, class_count=C, col_cat=col_cat, col_levels=col_levels, oob_votes=votes)


def save_forest(forest, path) -> None:
    with open(path, "wb") as fh:
        fh.write(forest_to_bytes(forest))


def load_forest(path) -> Forest:
    with open(path, "rb") as fh:
        return forest_from_bytes(fh.read())
