"""K8/K9 parity: factor-space MDS on the GPU vs the reference.

Tolerances (stated): eigenvalues rtol 1e-5; coordinates after sign fix /
Procrustes relative residual 1e-5; mds_correlation >= 0.99999;
a single gram_matvec within 1e-9 relative."""

import numpy as np
import pytest
from scipy.linalg import orthogonal_procrustes

from conftest import golden
from paper_2511_19493_b200 import mds as M
from paper_2511_19493_b200 import proximity as P
from paper_2511_19493_b200.quantize import QuantFactor

pytestmark = pytest.mark.gpu


def ref_lowrank(g, n):
    qf = QuantFactor("i8", g["lr_data"].shape, g["lr_data"], g["lr_scales"])
    return P.LowRankQuantized(n=n, rank=g["lr_data"].shape[1], mode="i8", factor=qf,
                              pmax=float(g["lr_pmax"]), tree_count=50)


def procrustes_rel(A, B):
    R, _ = orthogonal_procrustes(A, B)
    return np.linalg.norm(A @ R - B) / np.linalg.norm(B)


def test_gram_matvec_matches_reference():
    g = golden("wine50.npz")
    lr = ref_lowrank(g, 178)
    w = M.gram_matvec(lr, g["gmv_v"])
    assert np.linalg.norm(w - g["gmv_w"]) / np.linalg.norm(g["gmv_w"]) < 1e-9


def test_gram_matvec_properties():
    g = golden("wine50.npz")
    lr = ref_lowrank(g, 178)
    assert np.abs(M.gram_matvec(lr, np.ones(178))).max() < 1e-9
    v = np.random.default_rng(0).normal(size=178)
    np.testing.assert_allclose(M.gram_matvec(lr, 2.5 * v), 2.5 * M.gram_matvec(lr, v),
                               atol=1e-9)
    from paper_2511_19493_b200.errors import DataError
    with pytest.raises(DataError):
        M.gram_matvec(lr, np.ones(179))


def test_mds_lowrank_matches_reference():
    g = golden("wine50.npz")
    emb = M.mds_lowrank(ref_lowrank(g, 178), M.PowerIterConfig(seed=0))
    assert emb.k == len(g["mds_eig"])
    np.testing.assert_allclose(emb.eigenvalues, g["mds_eig"], rtol=1e-8)
    np.testing.assert_allclose(emb.coordinates, g["mds_coords"], atol=1e-6)
    assert np.array_equal(emb.converged, g["mds_conv"])
    assert np.all(np.abs(emb.iterations - g["mds_iter"]) <= 1)


def test_end_to_end_synth2k_vs_reference(synth2k):
    ds, forest = synth2k
    g = golden("synth2k.npz")
    lr = P.lowrank_proximity(P.leaf_membership(forest, ds), rank=32, mode="i8", seed=0)
    emb = M.mds_lowrank(lr, M.PowerIterConfig(seed=0))
    np.testing.assert_allclose(emb.eigenvalues, g["mds_eig"], rtol=1e-5)
    assert procrustes_rel(emb.coordinates, g["mds_coords"]) <= 1e-5
    ref = M.MdsEmbedding(g["mds_coords"], g["mds_eig"], g["mds_iter"], g["mds_eig"] * 0,
                         np.ones(len(g["mds_eig"]), bool))
    assert M.mds_correlation(emb, ref) >= 0.99999


def test_power_iteration_matches_dense(wine50, wine_ds):
    mem = P.leaf_membership(wine50, wine_ds)
    full = P.full_proximity(mem)
    rep = P.lowrank_proximity(mem, rank=178, mode="f32", seed=0)
    emb_lr = M.mds_lowrank(rep, M.PowerIterConfig(seed=3))
    emb_full = M.mds_full(full)
    assert emb_lr.k == emb_full.k == 3
    np.testing.assert_allclose(emb_lr.eigenvalues, emb_full.eigenvalues, rtol=1e-4)
    assert procrustes_rel(emb_lr.coordinates, emb_full.coordinates) <= 1e-4
    assert np.all(emb_lr.residuals <= 1e-6) and np.all(emb_lr.converged)


def test_mds_full_matches_reference(wine50, wine_ds):
    g = golden("wine50.npz")
    emb = M.mds_full(P.full_proximity(P.leaf_membership(wine50, wine_ds)))
    np.testing.assert_allclose(emb.eigenvalues, g["mdsfull_eig"], rtol=1e-12)
    np.testing.assert_allclose(emb.coordinates, g["mdsfull_coords"], atol=1e-10)


def test_rank1_membership_collapses():
    mem = P.LeafMembership(np.zeros((12, 4), np.int32), np.ones(4, np.int32))
    emb = M.mds_lowrank(P.lowrank_proximity(mem, rank=3, mode="f32"), M.PowerIterConfig())
    assert emb.k <= 1
    if emb.k == 1:
        assert emb.eigenvalues[0] < 1e-6


def test_nonconvergence_recorded_not_fatal():
    g = golden("wine50.npz")
    emb = M.mds_lowrank(ref_lowrank(g, 178), M.PowerIterConfig(max_iterations=2, tol=1e-15))
    assert emb.k >= 1 and not emb.converged.all() and np.isfinite(emb.residuals).all()
    assert np.all(emb.iterations == 2)


def test_deterministic():
    g = golden("wine50.npz")
    a = M.mds_lowrank(ref_lowrank(g, 178), M.PowerIterConfig(seed=9))
    b = M.mds_lowrank(ref_lowrank(g, 178), M.PowerIterConfig(seed=9))
    assert np.array_equal(a.coordinates, b.coordinates)


def test_int8_resident_slices_large_n(orc):
    """n = 150k, r = 32: the f64 factor slice no longer fits shared memory,
    so every CTA keeps int8 codes x scales (QS_I8 layout); five power
    iterations of three components against the oracle restatement."""
    rng = np.random.default_rng(11)
    n, r = 150_000, 32
    data = rng.integers(-127, 128, size=(n, r)).astype(np.int8)
    scales = rng.uniform(0.5e-3, 2e-3, r)
    Q = data.astype(np.float64) * scales[None, :]
    pmax = float(np.einsum("ij,ij->i", Q, Q).max())
    lr = P.LowRankQuantized(n=n, rank=r, mode="i8", factor=QuantFactor("i8", (n, r), data, scales),
                            pmax=pmax, tree_count=100)
    emb = M.mds_lowrank(lr, M.PowerIterConfig(seed=0, max_iterations=5, tol=1e-30, k=3))
    coords, eig, its, *_ = orc.mds_lowrank(Q, pmax, max_iterations=5, tol=1e-30, k=3, seed=0)
    assert np.all(emb.iterations == its)
    np.testing.assert_allclose(emb.eigenvalues, eig, rtol=1e-9)
    np.testing.assert_allclose(emb.coordinates, coords, rtol=1e-6, atol=1e-9 * np.abs(coords).max())
