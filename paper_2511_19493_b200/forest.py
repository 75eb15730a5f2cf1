"""Forest types and the RFX1 file format.

The proximity path's input is "the forest grown by the reference's CPU
trainer with the same seed".  ``Tree`` / ``Forest`` / ``TrainConfig``
mirror forest.py:42-130 field for field (the proximity functions accept the
reference's own objects too: only the node arrays are read).  Growing the
forest is out of scope for the product: the reference trainer restated in
C++ (byte-identical RFX1) lives with the test infrastructure in
``oracle/trainer.py`` and is used by the tests and bench.py to produce the
input on the GPU box, where the reference does not exist.
"""

from __future__ import annotations

import io
import struct
from dataclasses import dataclass, replace

import numpy as np

from .errors import DataError

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
