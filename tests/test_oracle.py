"""The CPU oracle (oracle/) is pinned against golden vectors produced by the
reference itself (tests/golden/make_golden.py)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden


def test_pcg32_known_answers(orc):
    kats = json.load(open(os.path.join(GOLDEN, "pcg32.json")))
    for k in kats:
        g = orc.Pcg32(k["seed"], k["seq"])
        assert [g.next_u32() for _ in range(8)] == k["u32"]
        assert [g.bounded(b) for b in (1, 2, 3, 1000, 178, 100000, 2**31 + 11)] == k["bounded"]
        want = np.array([float.fromhex(x) for x in k["normals"]])
        got = orc.Pcg32(k["seed"], k["seq"]).normals(9)
        np.testing.assert_allclose(got, want, rtol=2e-15, atol=0)


def test_wine_membership_and_counts(orc, wine50, wine_ds):
    g = golden("wine50.npz")
    codes, lc = orc.leaf_membership(wine50.trees, wine50.col_cat, wine_ds.values)
    assert np.array_equal(codes, g["codes"])
    assert np.array_equal(lc, g["leaf_counts"])
    counts = orc.pair_counts(codes, lc)
    assert np.array_equal(counts, g["pair_counts"])
    packed = orc.full_packed(codes, lc)
    assert np.array_equal(packed, g["packed"])  # bit-exact IEEE division


def test_wine_triblock(orc):
    g = golden("wine50.npz")
    di, dj, dv, si, sj, sv = orc.triblock(g["codes"], g["leaf_counts"], 0.05)
    assert np.array_equal(di, g["tb_dense_i"]) and np.array_equal(dj, g["tb_dense_j"])
    assert np.array_equal(dv, g["tb_dense_v"])
    assert np.array_equal(si, g["tb_sparse_i"]) and np.array_equal(sj, g["tb_sparse_j"])
    assert np.array_equal(sv, g["tb_sparse_v"])


def test_wine_lowrank_and_mds(orc):
    g = golden("wine50.npz")
    res = orc.lowrank(g["codes"], g["leaf_counts"], 16, "i8", seed=5)
    # same algorithm and third-party calls; only libm ulps of Omega differ
    dq_ref = g["lr_data"].astype(np.float64) * g["lr_scales"][None, :]
    Pr, Pg = dq_ref @ dq_ref.T, res["dq"] @ res["dq"].T
    assert np.linalg.norm(Pg - Pr) / np.linalg.norm(Pr) < 1e-9
    assert abs(res["pmax"] - float(g["lr_pmax"])) < 1e-9
    coords, eig, its, res_, conv = orc.mds_lowrank(dq_ref, float(g["lr_pmax"]), seed=0)
    np.testing.assert_allclose(eig, g["mds_eig"], rtol=1e-10)
    np.testing.assert_allclose(coords, g["mds_coords"], atol=1e-8)
    assert np.array_equal(its, g["mds_iter"])
    w = orc.gram_matvec(dq_ref, float(g["lr_pmax"]), g["gmv_v"])
    np.testing.assert_allclose(w, g["gmv_w"], rtol=1e-10, atol=1e-12)


def test_wine_mds_full(orc):
    g = golden("wine50.npz")
    P = orc.packed_to_dense(g["packed"], g["codes"].shape[0])
    coords, eig = orc.mds_full(P)
    np.testing.assert_allclose(eig, g["mdsfull_eig"], rtol=1e-10)
    np.testing.assert_allclose(np.abs(coords), np.abs(g["mdsfull_coords"]), atol=1e-9)


def test_synth2k_membership_counts_lowrank(orc, synth2k, fixtures):
    import hashlib
    ds, forest = synth2k
    g = golden("synth2k.npz")
    codes, lc = orc.leaf_membership(forest.trees, forest.col_cat, ds.values)
    assert np.array_equal(codes, g["codes"])
    c = orc.pair_counts(codes, lc)
    assert hashlib.sha256(c.astype(np.int32).tobytes()).hexdigest() == \
        fixtures["synth2k"]["counts_i32_sha"]
    res = orc.lowrank(codes, lc, 32, "i8", seed=0)
    dq_ref = g["lr_data"].astype(np.float64) * g["lr_scales"][None, :]
    Pr, Pg = dq_ref @ dq_ref.T, res["dq"] @ res["dq"].T
    assert np.linalg.norm(Pg - Pr) / np.linalg.norm(Pr) < 1e-9


def test_mixed_and_handbuilt_traversal(orc, mixed):
    ds, forest = mixed
    g = golden("mixed.npz")
    codes, _ = orc.leaf_membership(forest.trees, forest.col_cat, ds.values)
    assert np.array_equal(codes, g["codes"])
    h = golden("handbuilt.npz")

    class T:
        pass
    t = T()
    t.status, t.split_var, t.threshold = h["status"], h["split_var"], h["threshold"]
    t.cat_mask, t.left, t.right = np.zeros(7, np.int64), h["left"], h["right"]
    codes, _ = orc.leaf_membership([t], np.zeros(2, np.uint8), h["points"])
    assert np.array_equal(codes[:, 0], h["codes"])


def test_sketch_pass_matches_scipy(orc):
    g = golden("synth2k.npz")
    codes, lc = g["codes"], g["leaf_counts"]
    X = np.random.default_rng(0).normal(size=(codes.shape[0], 7))
    M = orc.onehot(codes, lc)
    want = M @ (M.T.tocsr() @ X)
    Y = np.empty_like(X)
    import ctypes
    orc.lib().orc_sketch_pass(orc._p(np.ascontiguousarray(codes)), codes.shape[0],
                              codes.shape[1], orc._p(np.ascontiguousarray(lc)),
                              orc._p(np.ascontiguousarray(X)), 7, orc._p(Y), 4)
    np.testing.assert_allclose(Y, want, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("mode", ["i8", "nf4", "f16", "f32"])
def test_quantize_matches_reference_semantics(orc, mode):
    rng = np.random.default_rng(11)
    x = rng.normal(size=(37, 5)) * rng.uniform(0.1, 3, size=5)
    x[:, 2] = 0.0
    data, scales = orc.quantize(x, mode)
    back = orc.dequantize(data, scales, mode, x.shape)
    if mode == "i8":
        assert np.all(np.abs(x - back) <= np.abs(x).max(axis=0) / 127 + 1e-15)
    if mode == "nf4":
        assert data.nbytes * 2 == x.size + (-x.size) % 64
