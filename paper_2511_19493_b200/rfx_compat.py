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

Device state survives between calls without any global registry: the
patched ``leaf_membership`` returns an instance of a subclass of the
reference's ``LeafMembership`` that holds this package's device membership
and materialises ``codes`` (the (n, B) int32 host array) only when something
reads it, so ``full_proximity(leaf_membership(f, d))`` neither copies the
codes to the host nor re-uploads them; likewise ``lowrank_proximity`` returns
a reference ``LowRankQuantized`` subclass carrying the device factor, which
``mds_lowrank`` / ``gram_matvec`` / ``outlier_scores`` use as long as the
object's factor and pmax are the ones it was built with.  The device state
lives exactly as long as the returned object.  ``uninstall()`` restores the
originals.
"""

from __future__ import annotations

import functools

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
_classes: dict = {}  # reference module id -> device-backed LeafMembership subclass


def _device_classes(rfx):
    """Subclass of the reference LeafMembership that carries this package's
    device membership (isinstance checks downstream keep working)."""
    key = id(rfx.proximity)
    if key in _classes:
        return _classes[key]
    RP = rfx.proximity

    class DeviceLeafMembership(RP.LeafMembership):
        """rfx.proximity.LeafMembership whose codes stay in HBM until read."""

        def __init__(self, mine):  # noqa: D107 - bypasses the dataclass __init__
            self._mine = mine
            self._host_codes = None
            self.leaf_counts = mine.leaf_counts

        @property
        def codes(self):
            if self._host_codes is None:
                self._host_codes = self._mine.codes
            return self._host_codes

        @codes.setter
        def codes(self, value):  # reassigned by a caller: the device copy is stale
            self._host_codes = np.asarray(value)
            self._mine = None

        @property
        def n(self):
            return self._mine.n if self._mine is not None else self.codes.shape[0]

        @property
        def tree_count(self):
            return self._mine.tree_count if self._mine is not None else self.codes.shape[1]

    _classes[key] = DeviceLeafMembership
    return _classes[key]


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
    """This package's LeafMembership for a reference one: the device copy when
    ``m`` came out of the patched leaf_membership (and its codes were not
    reassigned), else an upload of ``m.codes``."""
    if isinstance(m, _prox.LeafMembership):
        return m
    mine = getattr(m, "_mine", None)  # None again once a caller reassigned m.codes
    if mine is not None:
        return mine
    return _prox.LeafMembership(codes=np.asarray(m.codes), leaf_counts=np.asarray(m.leaf_counts))


def _ours_lowrank(lr):
    if isinstance(lr, _prox.LowRankQuantized):
        return lr
    mine = getattr(lr, "_mine", None)
    if mine is not None and lr.factor is lr._mine_factor and lr.pmax == mine.pmax:
        return mine  # factor and pmax untouched since the device produced them
    qf = lr.factor
    return _prox.LowRankQuantized(
        n=lr.n, rank=lr.rank, mode=lr.mode,
        factor=_QuantFactor(qf.mode, tuple(qf.shape), qf.data, qf.scales),
        pmax=lr.pmax, tree_count=lr.tree_count, rank_degraded=lr.rank_degraded)


def import_reference():
    """Import the reference ``rfx`` package: already importable, else the
    copy installed into ``baseline/_ref`` (travels to the GPU box), else
    ``/root/reference/pkg/src`` (the build container)."""
    import importlib
    import os
    import sys
    try:
        return importlib.import_module("rfx")
    except ImportError:
        pass
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (os.path.join(root, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "rfx")):
            sys.path.insert(0, p)
            return importlib.import_module("rfx")
    raise _errors.RfxError("the reference package rfx is not importable (baseline/_ref)")


def install(rfx=None):
    """Patch the reference package (imported ``rfx`` module, or import it)."""
    if rfx is None:
        rfx = import_reference()
    import importlib
    RP = importlib.import_module(rfx.__name__ + ".proximity")
    RM = importlib.import_module(rfx.__name__ + ".mds")
    tr = _translate(rfx)

    DevMembership = _device_classes(rfx)

    @tr
    def leaf_membership(forest, dataset):
        return DevMembership(_prox.leaf_membership(forest, dataset))

    @tr
    def full_proximity(membership, budget_bytes=_prox.DEFAULT_BUDGET):
        out = _prox.full_proximity(_ours_membership(membership), budget_bytes)
        ref = RP.FullTriangle(n=out.n, tree_count=out.tree_count, packed=out.packed)
        ref._mine = out  # the HBM triangle rides along (outlier_scores reuses it)
        return ref

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
        ref = RP.LowRankQuantized(n=out.n, rank=out.rank, mode=out.mode, factor=factor,
                                  pmax=out.pmax, tree_count=out.tree_count,
                                  rank_degraded=out.rank_degraded)
        ref._mine, ref._mine_factor = out, factor  # the device factor rides along
        return ref

    @tr
    def outlier_scores(repr_, clamp_floor=None):
        if isinstance(repr_, RP.FullTriangle):
            mine = getattr(repr_, "_mine", None)
            if mine is None or repr_.packed is not mine.packed:
                mine = _prox.FullTriangle(n=repr_.n, tree_count=repr_.tree_count,
                                          packed=repr_.packed)
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
        rfx = import_reference()
    for modname, names in PATCHED.items():
        mod = getattr(rfx, modname)
        for name in names:
            orig = _saved.pop((mod.__name__, name), None)
            if orig is not None:
                setattr(mod, name, orig)
