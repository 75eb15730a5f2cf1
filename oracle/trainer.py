"""Input producer — TEST / BENCH INFRASTRUCTURE, not the product.

The proximity path's input is "the forest grown by the reference's CPU
trainer with the same seed" (BASELINE.json north_star).  The reference
trainer (``rfx.train``, forest.py:262-302, Numba kernels _kernels.py:28-330)
is out of scope for the GPU build and absent on the GPU
box, so ``rfx_train.cpp`` restates it in C++ — byte-identical RFX1 output,
pinned by tests/test_train.py against SHA-256s the reference produced
(tests/golden/fixtures.json, scale.json).  The tests, ``smoke()`` and
bench.py call ``train`` to regenerate the exact input forest from the seed;
training is never inside a timed region.  The product package never imports
this module.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from paper_2511_19493_b200.dataset import Dataset, column_arrays
from paper_2511_19493_b200.errors import DataError, RfxError
from paper_2511_19493_b200.forest import BootstrapRecord, Forest, TrainConfig, Tree

_HERE = os.path.dirname(os.path.abspath(__file__))
TRAIN_LIB_PATH = os.path.join(_HERE, "_build", "librfx_train.so")

_train_lib = None


def _tlib():
    global _train_lib
    if _train_lib is None:
        if not os.path.exists(TRAIN_LIB_PATH):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        L = ctypes.CDLL(TRAIN_LIB_PATH)
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
