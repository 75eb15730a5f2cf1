"""Install the B200 proximity path into the reference ``rfx`` package.

``install(rfx)`` replaces the bodies of the reference's hot-path functions
 with thin adapters around this package, keeping their
signatures, defaults, return dataclasses (the reference's own classes, which
downstream code type-checks: ``mds.mds_full`` ``mds.py:100-101``,
``proximity.outlier_scores`` ``proximity.py:447-484``,
``proximity.save_proximity`` ``proximity.py:729-736``) and exception types:

  rfx.proximity.leaf_membership     proximity.py:100-116
  rfx.proximity.full_proximity      proximity.py:188-201
  rfx.proximity.triblock_proximity  proximity.py:275-327
  rfx.proximity.lowrank_proximity   proximity.py:367-420
  rfx.proximity.outlier_scores      proximity.py:432-485
  rfx.mds.gram_matvec               mds.py:161-181
  rfx.mds.mds_lowrank               mds.py:184-268

Device state survives between calls: the reference ``LeafMembership``
returned by ``leaf_membership`` is remembered (by identity) together with the
device membership it came from, so ``full_proximity(leaf_membership(f, d))``
does not re-upload the (n, B) codes.  ``uninstall()`` restores the originals.
"""

from __future__ import annotations

import functools
import weakref

import numpy as np

from . import errors as _errors
from . import mds as _mds
from . import proximity as _prox
from .quantize import QuantFactor as _QuantFactor

PATCHED = {
    "proximity": ("leaf_membership", "full_proximity", "triblock_proximity",
                  "lowrank_proximity", "outlier_scores"),
    "mds": ("gram_matvec", "mds_lowrank"),
}

_saved: dict = {}
_device_of: "weakref.WeakKeyDictionary | dict" = {}


def _translate(rfx):
    """Re-raise this package's exceptions as the reference's own types."""
    def deco(fn):
        @functools.wraps(fn)
        def wrapper(*a, **kw):
            try:
                return fn(*a, **kw)
            except _errors.BudgetError as e:
                raise rfx.errors.BudgetError(str(e), e.plan) from e
            except _errors.DataError as e:
                raise rfx.errors.DataError(str(e)) from e
            except _errors.RfxError as e:
                raise rfx.errors.RfxError(str(e)) from e
        return wrapper
    return deco


def _ours_membership(m):
    """This package's LeafMembership for a reference one (device copy reused
    when ``m`` came out of the patched leaf_membership)."""
    if isinstance(m, _prox.LeafMembership):
        return m
    mine = _device_of.get(id(m))
    if mine is not None and mine[0]() is m:
        return mine[1]
    return _prox.LeafMembership(codes=np.asarray(m.codes), leaf_counts=np.asarray(m.leaf_counts))


def _ours_lowrank(lr):
    if isinstance(lr, _prox.LowRankQuantized):
        return lr
    qf = lr.factor
    return _prox.LowRankQuantized(
        n=lr.n, rank=lr.rank, mode=lr.mode,
        factor=_QuantFactor(qf.mode, tuple(qf.shape), qf.data, qf.scales),
        pmax=lr.pmax, tree_count=lr.tree_count, rank_degraded=lr.rank_degraded)


def install(rfx=None):
    """Patch the reference package (imported ``rfx`` module, or import it)."""
    if rfx is None:
        import rfx  # noqa: F811
    import rfx.mds
    import rfx.proximity
    RP, RM = rfx.proximity, rfx.mds
    tr = _translate(rfx)

    @tr
    def leaf_membership(forest, dataset):
        mine = _prox.leaf_membership(forest, dataset)
        # the reference dataclass needs host codes; read them once, keep the
        # device membership for the next backend call
        ref = RP.LeafMembership(codes=mine.codes, leaf_counts=mine.leaf_counts)
        _device_of[id(ref)] = (weakref.ref(ref), mine)
        return ref

    @tr
    def full_proximity(membership, budget_bytes=_prox.DEFAULT_BUDGET):
        out = _prox.full_proximity(_ours_membership(membership), budget_bytes)
        return RP.FullTriangle(n=out.n, tree_count=out.tree_count, packed=out.packed)

    @tr
    def triblock_proximity(membership, tau=_prox.DEFAULT_TAU, budget_bytes=_prox.DEFAULT_BUDGET):
        out = _prox.triblock_proximity(_ours_membership(membership), tau, budget_bytes)
        return RP.TriBlock(n=out.n, tree_count=out.tree_count, tau=out.tau, dense=out.dense,
                           sparse_i=out.sparse_i, sparse_j=out.sparse_j, sparse_v=out.sparse_v)

    @tr
    def lowrank_proximity(membership, rank, mode="i8", seed=0):
        out = _prox.lowrank_proximity(_ours_membership(membership), rank, mode, seed)
        qf = out.factor
        factor = rfx.quantize.QuantFactor(qf.mode, tuple(qf.shape), qf.data, qf.scales)
        return RP.LowRankQuantized(n=out.n, rank=out.rank, mode=out.mode, factor=factor,
                                   pmax=out.pmax, tree_count=out.tree_count,
                                   rank_degraded=out.rank_degraded)

    @tr
    def outlier_scores(repr_, clamp_floor=None):
        if isinstance(repr_, RP.FullTriangle):
            mine = _prox.FullTriangle(n=repr_.n, tree_count=repr_.tree_count, packed=repr_.packed)
        elif isinstance(repr_, RP.TriBlock):
            mine = _prox.TriBlock(n=repr_.n, tree_count=repr_.tree_count, tau=repr_.tau,
                                  dense=repr_.dense, sparse_i=repr_.sparse_i,
                                  sparse_j=repr_.sparse_j, sparse_v=repr_.sparse_v)
        elif isinstance(repr_, RP.LowRankQuantized):
            mine = _ours_lowrank(repr_)
        else:
            mine = repr_
        return _prox.outlier_scores(mine, clamp_floor)

    @tr
    def gram_matvec(lowrank, v):
        return _mds.gram_matvec(_ours_lowrank(lowrank), v)

    @tr
    def mds_lowrank(lowrank, config=None):
        cfg = None if config is None else _mds.PowerIterConfig(
            max_iterations=config.max_iterations, tol=config.tol, k=config.k, seed=config.seed)
        e = _mds.mds_lowrank(_ours_lowrank(lowrank), cfg)
        return RM.MdsEmbedding(coordinates=e.coordinates, eigenvalues=e.eigenvalues,
                               iterations=e.iterations, residuals=e.residuals,
                               converged=e.converged)

    new = {"proximity": {"leaf_membership": leaf_membership, "full_proximity": full_proximity,
                         "triblock_proximity": triblock_proximity,
                         "lowrank_proximity": lowrank_proximity,
                         "outlier_scores": outlier_scores},
           "mds": {"gram_matvec": gram_matvec, "mds_lowrank": mds_lowrank}}
    for modname, names in PATCHED.items():
        mod = getattr(rfx, modname)
        for name in names:
            _saved.setdefault((mod.__name__, name), getattr(mod, name))
            setattr(mod, name, new[modname][name])
    return rfx


def uninstall(rfx=None):
    """Restore the reference functions patched by ``install``."""
    if rfx is None:
        import rfx  # noqa: F811
    for modname, names in PATCHED.items():
        mod = getattr(rfx, modname)
        for name in names:
            orig = _saved.pop((mod.__name__, name), None)
            if orig is not None:
                setattr(mod, name, orig)
    _device_of.clear()
