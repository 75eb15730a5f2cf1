"""Classical MDS from proximity representations — drop-in for mds.py.

``mds_lowrank`` / ``gram_matvec`` run the factor-route power iteration on
the GPU (csrc/mds.cu: one persistent cooperative kernel for all k
eigenpairs, mds.py:184-268).  ``mds_full`` is the reference's dense route
for n <= 5000 (mds.py:93-137): host LAPACK eigh of the double-centred
Gram matrix, exactly as the reference computes it (the Wine config).
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DataError, RfxError
from .profiling import region
from .proximity import FullTriangle, LowRankQuantized, TriBlock

logger = logging.getLogger(__name__)

DEFAULT_ORACLE_BOUND = 5000   # mds.py:33
MAX_COMPONENTS = 8            # mds.py:41


@dataclass
class PowerIterConfig:
    max_iterations: int = 300
    tol: float = 1e-8
    k: int = 3
    seed: int = 0

    def __post_init__(self):
        if self.tol <= 0:
            raise DataError("tol must be positive")
        if not 1 <= self.k <= MAX_COMPONENTS:
            raise DataError(f"k must be in [1, {MAX_COMPONENTS}]")


@dataclass
class MdsEmbedding:
    coordinates: np.ndarray
    eigenvalues: np.ndarray
    iterations: np.ndarray
    residuals: np.ndarray
    converged: np.ndarray

    @property
    def n(self) -> int:
        return self.coordinates.shape[0]

    @property
    def k(self) -> int:
        return self.coordinates.shape[1]


def _sign_fix(vec: np.ndarray) -> np.ndarray:
    idx = int(np.argmax(np.abs(vec)))
    return -vec if vec[idx] < 0 else vec


def mds_full(prox, k: int = 3, oracle_bound: int = DEFAULT_ORACLE_BOUND) -> MdsEmbedding:
    """Dense-eigendecomposition MDS of a FullTriangle or TriBlock
    (mds.py:93-137); reference semantics, host LAPACK."""
    if not isinstance(prox, (FullTriangle, TriBlock)):
        raise DataError("mds_full expects a FullTriangle or TriBlock")
    n = prox.n
    if not 1 <= k <= MAX_COMPONENTS:
        raise DataError(f"k must be in [1, {MAX_COMPONENTS}]")
    if n > oracle_bound:
        raise DataError(f"n={n} exceeds the dense-route bound {oracle_bound}; "
                        "use the lowrank backend")
    P = prox.to_dense()
    D2 = (float(P.max()) - P) ** 2
    G = -0.5 * (D2 - D2.mean(axis=1, keepdims=True) - D2.mean(axis=0, keepdims=True)
                + D2.mean())
    lam, vecs = np.linalg.eigh(G)
    order = np.argsort(lam)[::-1]
    lam, vecs = lam[order], vecs[:, order]
    kp = int(min(k, (lam > 0).sum()))
    if kp < k:
        logger.warning("only %d positive eigenvalues available; returning %d coordinate "
                       "columns instead of %d", kp, kp, k)
    coords = np.empty((n, kp))
    res = np.empty(kp)
    for c in range(kp):
        v = _sign_fix(vecs[:, c])
        coords[:, c] = np.sqrt(lam[c]) * v
        res[c] = np.linalg.norm(G @ v - lam[c] * v) / abs(lam[c])
    return MdsEmbedding(coords, lam[:kp].copy(), np.zeros(kp, dtype=np.int64), res,
                        np.ones(kp, dtype=bool))


MAX_RANK = 192  # rfxc_mds_power / rfxc_gram_matvec (csrc/mds.cu MAXRT)


def _work(n: int, r: int, k: int, dev):
    import torch
    nbytes = int(_lib.load().rfxc_mds_work_bytes(n, r, k))
    return torch.empty(nbytes, dtype=torch.uint8, device=dev)


def gram_matvec(lowrank: LowRankQuantized, v: np.ndarray, _cache: dict | None = None) -> np.ndarray:
    """G v = -1/2 H D2 H v from the factors, on the GPU (mds.py:161-181)."""
    import torch
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (lowrank.n,):
        raise DataError(f"vector length {v.shape} does not match n={lowrank.n}")
    if int(lowrank.rank) > MAX_RANK:
        raise DataError(f"gram_matvec: rank {lowrank.rank} above this build's limit {MAX_RANK}")
    dq = lowrank.dequantized_device()
    n, r = dq.shape
    dv = torch.from_numpy(np.ascontiguousarray(v)).to(dq.device)
    w = torch.empty(n, dtype=torch.float64, device=dq.device)
    _lib.call("rfxc_gram_matvec", _lib.ptr(dq), n, r, float(lowrank.pmax), _lib.ptr(dv),
              _lib.ptr(w), _lib.ptr(_work(n, r, 1, dq.device)), _lib.stream_handle())
    return w.cpu().numpy()


def mds_lowrank_device(lowrank: LowRankQuantized, config: PowerIterConfig | None = None):
    """Run the persistent power-iteration kernel; returns device tensors
    (coords (n, k), info (k, 4), k_used (1,))."""
    import torch
    cfg = config or PowerIterConfig()
    r = int(lowrank.rank)
    if r > MAX_RANK:  # before any upload or launch (INTEGRATION.md "Limits")
        raise DataError(f"mds_lowrank: rank {r} above this build's limit {MAX_RANK}")
    dq = lowrank.dq if hasattr(lowrank, "dq") else lowrank.dequantized_device()
    n, r = dq.shape
    dev = dq.device
    codes = scales = None
    if lowrank.mode == "i8":  # int8 factor: shared-memory-resident slices at large n
        if hasattr(lowrank, "data"):
            codes, scales = lowrank.data, lowrank.scales
        else:
            codes, scales = lowrank.device_codes()
    coords = torch.empty((n, cfg.k), dtype=torch.float64, device=dev)
    info = torch.empty((cfg.k, 4), dtype=torch.float64, device=dev)
    kused = torch.empty(1, dtype=torch.int32, device=dev)
    work = _work(n, r, cfg.k, dev)
    # pmax straight from the device when the factorisation left it there
    pm_dev = getattr(lowrank, "pm", None)
    if pm_dev is None:
        pm_dev = getattr(lowrank, "_pmax_dev", None)
    pmax = 0.0 if pm_dev is not None else float(lowrank.pmax)
    with region("mds_power"):
        _lib.call("rfxc_mds_power", _lib.ptr(dq), _lib.ptr(codes), _lib.ptr(scales), n, r,
                  pmax, _lib.ptr(pm_dev), cfg.k, cfg.max_iterations, float(cfg.tol), cfg.seed,
                  _lib.ptr(coords), _lib.ptr(info), _lib.ptr(kused), _lib.ptr(work),
                  _lib.stream_handle())
    return coords, info, kused


def mds_lowrank(lowrank: LowRankQuantized, config: PowerIterConfig | None = None) -> MdsEmbedding:
    """Power iteration with implicit deflation on the factor-space Gram
    operator (mds.py:184-268), one cooperative kernel on the GPU."""
    cfg = config or PowerIterConfig()
    coords, info, kused = mds_lowrank_device(lowrank, cfg)
    ku = int(kused.item())
    inf = info.cpu().numpy()[:ku]
    for c in range(ku):
        if inf[c, 3] == 0.0:
            logger.warning("power iteration for eigenpair %d stopped at the %d-iteration cap "
                           "(relative residual %.3g)", c, cfg.max_iterations, inf[c, 2])
    if ku < cfg.k:
        logger.warning("eigenpair %d is non-positive; returning %d coordinate columns", ku, ku)
    return MdsEmbedding(coordinates=np.ascontiguousarray(coords.cpu().numpy()[:, :ku]),
                        eigenvalues=inf[:, 0].copy(),
                        iterations=inf[:, 1].astype(np.int64),
                        residuals=inf[:, 2].copy(),
                        converged=inf[:, 3] != 0.0)


def mds_correlation(a: MdsEmbedding, b: MdsEmbedding) -> float:
    """Pearson correlation of pairwise-distance vectors (mds.py:271-280)."""
    from scipy.spatial.distance import pdist
    if a.n != b.n:
        raise DataError(f"embeddings disagree on n: {a.n} vs {b.n}")
    da, db = pdist(a.coordinates), pdist(b.coordinates)
    if da.std() == 0 or db.std() == 0:
        raise RfxError("zero-variance distance vector; correlation undefined")
    return float(np.corrcoef(da, db)[0, 1])
