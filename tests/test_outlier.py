"""SURVEY §8(f) epilogues: outlier_scores (proximity.py:432-485, rank 1)
and the OOB votes recomputed from the leaf codes (rank 4, last test).

CPU: the oracle restatement against the reference's own scores
(tests/golden/outlier_wine50.npz, tests/golden/make_outlier_golden.py).
GPU: the device FullTriangle / low-rank kernels and the TriBlock epilogue
against the same goldens (rtol 1e-12 for the exact triangle; the factor's
q_i . q_j are f64 DMMA sums in another order than BLAS, rtol 1e-10), and
against the oracle at n = 2000 with floors that bite."""

import numpy as np
import pytest

from conftest import cuda_ok, golden


def test_oracle_matches_reference_scores():
    from oracle import oracle as orc
    g, o = golden("wine50.npz"), golden("outlier_wine50.npz")
    n = g["codes"].shape[0]
    np.testing.assert_allclose(orc.outlier_packed(g["packed"], n, 1 / 50), o["full"], rtol=1e-13)
    np.testing.assert_allclose(orc.outlier_packed(g["packed"], n, 0.05), o["full_floor"], rtol=1e-13)
    Q = g["lr_data"].astype(np.float64) * g["lr_scales"][None, :]
    np.testing.assert_allclose(orc.outlier_lowrank(Q, 1 / 50), o["lowrank"], rtol=1e-13)
    np.testing.assert_allclose(orc.outlier_lowrank(Q, 0.1), o["lowrank_floor"], rtol=1e-13)


def test_errors_match_reference():
    from paper_2511_19493_b200 import proximity as P
    from paper_2511_19493_b200.errors import RfxError
    with pytest.raises(RfxError, match="n >= 2"):
        P.outlier_scores(P.FullTriangle(n=1, tree_count=5, packed=np.empty(0)))
    with pytest.raises(RfxError, match="positive"):
        P.outlier_scores(P.FullTriangle(n=3, tree_count=5, packed=np.ones(3)), clamp_floor=0.0)
    with pytest.raises(RfxError, match="unknown"):
        P.outlier_scores(type("X", (), {"n": 4, "tree_count": 2})())




@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")
def test_wine_matches_reference_scores(built):
    from paper_2511_19493_b200 import proximity as P
    from paper_2511_19493_b200.quantize import QuantFactor
    g, o = golden("wine50.npz"), golden("outlier_wine50.npz")
    n = g["codes"].shape[0]
    full = P.FullTriangle(n=n, tree_count=50, packed=g["packed"])
    np.testing.assert_allclose(P.outlier_scores(full), o["full"], rtol=1e-12)
    np.testing.assert_allclose(P.outlier_scores(full, clamp_floor=0.05), o["full_floor"], rtol=1e-12)
    tb = P.TriBlock(n=n, tree_count=50, tau=0.05,
                    dense=P.PairMap(n, g["tb_dense_i"], g["tb_dense_j"], g["tb_dense_v"]),
                    sparse_i=g["tb_sparse_i"], sparse_j=g["tb_sparse_j"], sparse_v=g["tb_sparse_v"])
    np.testing.assert_allclose(P.outlier_scores(tb), o["triblock"], rtol=1e-12)
    lr = P.LowRankQuantized(n=n, rank=16, mode="i8",
                            factor=QuantFactor("i8", (n, 16), g["lr_data"], g["lr_scales"]),
                            pmax=float(g["lr_pmax"]), tree_count=50)
    np.testing.assert_allclose(P.outlier_scores(lr), o["lowrank"], rtol=1e-10)
    np.testing.assert_allclose(P.outlier_scores(lr, clamp_floor=0.1), o["lowrank_floor"], rtol=1e-10)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")
@pytest.mark.parametrize("n,r", [(2, 1), (130, 3), (2000, 32), (3001, 40), (500, 110), (701, 150), (333, 256)])
def test_lowrank_kernel_vs_oracle(built, n, r):
    from paper_2511_19493_b200 import proximity as P
    from paper_2511_19493_b200.quantize import QuantFactor
    from oracle import oracle as orc
    rng = np.random.default_rng(n + r)
    Q = rng.normal(size=(n, r)) * (0.6 / np.sqrt(r))
    lr = P.LowRankQuantized(n=n, rank=r, mode="f32",
                            factor=QuantFactor("f32", (n, r), Q.astype(np.float32), None),
                            pmax=1.0, tree_count=40)
    Qd = Q.astype(np.float32).astype(np.float64)
    for floor in (None, 0.2):
        want = orc.outlier_lowrank(Qd, 1 / 40 if floor is None else floor)
        np.testing.assert_allclose(P.outlier_scores(lr, clamp_floor=floor), want, rtol=1e-10)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")
def test_full_triangle_device_copy_vs_oracle(synth2k):
    from paper_2511_19493_b200 import proximity as P
    from oracle import oracle as orc
    ds, forest = synth2k
    full = P.full_proximity(P.leaf_membership(forest, ds))
    assert full._packed_dev is not None  # the K3 output stays in HBM for the epilogue
    for floor in (None, 0.1):
        want = orc.outlier_packed(full.packed, full.n, 1 / 40 if floor is None else floor)
        np.testing.assert_allclose(P.outlier_scores(full, clamp_floor=floor), want, rtol=1e-12)


@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")
def test_oob_votes_equal_the_trainers(wine50, wine_ds, synth2k):
    """OOB votes from the device leaf codes equal the
    votes the trainer accumulated (forest.oob_votes, byte-identical to the
    reference's RFX1 record, tests/test_train.py)."""
    from paper_2511_19493_b200 import proximity as P
    for forest, ds in ((wine50, wine_ds), synth2k[::-1]):
        got = P.oob_votes(forest, ds)
        assert got.dtype == np.int64 and np.array_equal(got, forest.oob_votes)
