"""BASELINE configs[3] at full size: synthetic 100k x 100, 500 trees (the
bench workload).

Pinned to the REFERENCE run at this size (tests/golden/scale.json["100k"] and
lowrank_100k.npz, from make_golden.py --scale --only 100k): the regrown
forest's RFX1 SHA-256, the (n, B) leaf codes' SHA-256, and the reference's
rank-32 INT8 factor, pmax and 3-D MDS embedding at the stated tolerances
(relative Frobenius 1e-4, pmax 1e-4, eigenvalues rtol 1e-5, Procrustes 1e-5).

Size-independent properties of the sketch and the factor on top:

* P 1 (a sketch pass of the all-ones column) equals (1/B) sum_b s_{b,l_b(i)}
  from the leaf sizes — exact integers in f32, rtol 1e-12;
* P is symmetric: x^T (P y) = y^T (P x) for random x, y (f32 operands, 1e-6);
* a tree-batch sample of the sketch (first 32 trees) matches the CPU oracle's
  per-tree restatement;
* the INT8 factor Q reproduces the top of P: for the unit-norm vector u = Q_1 /
  |Q_1|, u^T P u (one more sketch pass) equals |Q^T u|^2 within 1e-3 relative
  (the rank-32 truncation plus quantisation)."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


@pytest.fixture(scope="module")
def inputs100k(built):
    import os

    from oracle.trainer import train
    from paper_2511_19493_b200.dataset import from_arrays, make_synthetic
    from paper_2511_19493_b200.forest import TrainConfig
    X, y = make_synthetic(100_000, 100, seed=0)
    ds = from_arrays(X, y)
    return ds, train(ds, TrainConfig(ntree=500, iseed=1), nthreads=os.cpu_count() or 1)


@pytest.fixture(scope="module")
def mem100k(inputs100k):
    from paper_2511_19493_b200 import proximity as P
    ds, forest = inputs100k
    return P.leaf_membership(forest, ds)


def sketch(mem, X):
    import torch
    from paper_2511_19493_b200 import proximity as P
    n, k = X.shape
    sk = P._Sketch(mem.device(), k)
    X32 = torch.zeros((n, sk.ld), dtype=torch.float32, device="cuda")
    X32[:, :k] = torch.from_numpy(X.astype(np.float32)).cuda()
    return sk.apply(X32, k).cpu().numpy()


def test_sketch_of_ones_is_mean_leaf_size(mem100k):
    codes, lc = mem100k.codes, mem100k.leaf_counts
    n, B = codes.shape
    want = np.zeros(n)
    for b in range(B):
        sizes = np.bincount(codes[:, b], minlength=lc[b])
        want += sizes[codes[:, b]]
    want /= B
    got = sketch(mem100k, np.ones((n, 1)))[:, 0]
    np.testing.assert_allclose(got, want, rtol=1e-12)


def test_sketch_symmetric(mem100k):
    rng = np.random.default_rng(3)
    n = mem100k.n
    X = rng.normal(size=(n, 2)).astype(np.float32).astype(np.float64)
    Y = sketch(mem100k, X)
    a, b = X[:, 0] @ Y[:, 1], X[:, 1] @ Y[:, 0]
    assert abs(a - b) <= 1e-6 * max(abs(a), abs(b))


def test_sketch_tree_batch_vs_oracle(orc, mem100k):
    from paper_2511_19493_b200 import proximity as P
    codes = np.ascontiguousarray(mem100k.codes[:, :32])
    lc = np.ascontiguousarray(mem100k.leaf_counts[:32])
    rng = np.random.default_rng(5)
    X = rng.normal(size=(codes.shape[0], 40)).astype(np.float32).astype(np.float64)
    want = np.empty_like(X)
    orc.lib().orc_sketch_pass(orc._p(codes), codes.shape[0], 32, orc._p(lc), orc._p(X), 40,
                              orc._p(want), 8)
    got = sketch(P.LeafMembership(codes, lc), X)
    assert np.abs(got - want).max() <= 2e-6 * np.abs(want).max()


def test_factor_captures_the_top_of_P(mem100k):
    from paper_2511_19493_b200 import proximity as P
    lr = P.lowrank_proximity(mem100k, rank=32, mode="i8", seed=0)
    Q = lr.dequantized()
    u = Q[:, 0] / np.linalg.norm(Q[:, 0])
    uPu = float(u @ sketch(mem100k, u[:, None])[:, 0])
    uQQu = float(np.sum((Q.T @ u) ** 2))
    assert abs(uPu - uQQu) <= 1e-3 * uPu, (uPu, uQQu)
    assert 0.0 < lr.pmax <= 1.0 + 1e-6


def test_forest_and_codes_are_the_references(inputs100k, mem100k):
    import hashlib
    import json
    import os

    from conftest import GOLDEN
    from paper_2511_19493_b200.forest import forest_to_bytes
    rec = json.load(open(os.path.join(GOLDEN, "scale.json")))["100k"]
    ds, forest = inputs100k
    assert hashlib.sha256(forest_to_bytes(forest)).hexdigest() == rec["rfx1_sha"]
    assert hashlib.sha256(mem100k.codes.tobytes()).hexdigest() == rec["codes_sha"]
    assert int(mem100k.leaf_counts.sum()) == rec["total_leaves"]


def test_factor_and_mds_vs_reference(mem100k):
    from conftest import golden
    from paper_2511_19493_b200 import mds as M
    from paper_2511_19493_b200 import proximity as P
    from test_gpu_lowrank import frob_rel
    from test_gpu_mds import procrustes_rel
    g = golden("lowrank_100k.npz")
    lr = P.lowrank_proximity(mem100k, rank=32, mode="i8", seed=0)
    ref = g["data"].astype(np.float64) * g["scales"][None, :]
    assert frob_rel(lr.dequantized(), ref) <= 1e-4
    assert abs(lr.pmax - float(g["pmax"])) / float(g["pmax"]) <= 1e-4
    emb = M.mds_lowrank(lr, M.PowerIterConfig(seed=0))
    np.testing.assert_allclose(emb.eigenvalues, g["mds_eig"], rtol=1e-5)
    assert procrustes_rel(emb.coordinates, g["mds_coords"]) <= 1e-5
    assert np.all(np.abs(np.asarray(emb.iterations) - g["mds_iter"]) <= 2)
