"""K4-K7 parity: implicit sketch + QLORA quantisation + pmax.

Tolerances (stated): relative Frobenius error of the
reconstructed proximity ||Q_g Q_g^T - Q_r Q_r^T||_F / ||Q_r Q_r^T||_F <= 1e-4
against the reference's factor (same seed, same Omega stream), pmax relative
difference <= 1e-4.  Quantisation of a given factor is bit-exact."""

import numpy as np
import pytest

from conftest import golden
from paper_2511_19493_b200 import proximity as P
from paper_2511_19493_b200 import quantize as Qz

pytestmark = pytest.mark.gpu

FROB_TOL = 1e-4
PMAX_TOL = 1e-4


def frob_rel(A, R):
    """||A A^T - R R^T||_F / ||R R^T||_F through r x r products (never n x n)."""
    aa = np.linalg.norm(A.T @ A) ** 2
    rr = np.linalg.norm(R.T @ R) ** 2
    ar = np.linalg.norm(A.T @ R) ** 2
    return np.sqrt(max(aa + rr - 2 * ar, 0.0)) / np.sqrt(rr)


def dq_of(data, scales):
    return data.astype(np.float64) * scales[None, :]


def test_wine_i8_matches_reference(wine50, wine_ds):
    g = golden("wine50.npz")
    mem = P.leaf_membership(wine50, wine_ds)
    lr = P.lowrank_proximity(mem, rank=16, mode="i8", seed=5)
    assert lr.rank == 16 and lr.factor.data.dtype == np.int8 and lr.factor.data.shape == (178, 16)
    ref = dq_of(g["lr_data"], g["lr_scales"])
    got = lr.dequantized()
    assert frob_rel(got, ref) <= FROB_TOL
    # direct check on the full (small) matrix too
    assert np.abs(got @ got.T - ref @ ref.T).max() <= 1e-3
    assert abs(lr.pmax - float(g["lr_pmax"])) / float(g["lr_pmax"]) <= PMAX_TOL


def test_synth2k_i8_matches_reference(synth2k):
    g = golden("synth2k.npz")
    ds, forest = synth2k
    lr = P.lowrank_proximity(P.leaf_membership(forest, ds), rank=32, mode="i8", seed=0)
    assert frob_rel(lr.dequantized(), dq_of(g["lr_data"], g["lr_scales"])) <= FROB_TOL
    assert abs(lr.pmax - float(g["lr_pmax"])) / float(g["lr_pmax"]) <= PMAX_TOL


def test_against_oracle_pipeline(orc, synth2k):
    ds, forest = synth2k
    g = golden("synth2k.npz")
    res = orc.lowrank(g["codes"], g["leaf_counts"], 20, "f32", seed=3)
    lr = P.lowrank_proximity(P.leaf_membership(forest, ds), rank=20, mode="f32", seed=3)
    assert frob_rel(lr.dequantized(), res["dq"]) <= FROB_TOL


def test_deterministic_bytes(synth2k):
    ds, forest = synth2k
    mem = P.leaf_membership(forest, ds)
    a = P.lowrank_proximity(mem, rank=16, mode="i8", seed=5)
    b = P.lowrank_proximity(mem, rank=16, mode="i8", seed=5)
    assert np.array_equal(a.factor.data, b.factor.data)
    assert np.array_equal(a.factor.scales, b.factor.scales) and a.pmax == b.pmax


def test_rank_degrades_with_notice():
    codes = np.zeros((10, 2), np.int32)
    codes[5:, :] = 1
    rep = P.lowrank_proximity(P.LeafMembership(codes, np.array([2, 2], np.int32)), rank=50,
                              mode="f32")
    assert rep.rank_degraded and rep.rank <= 4
    Q = rep.dequantized()
    want = np.where(codes[:, 0][:, None] == codes[:, 0][None, :], 1.0, 0.0)
    assert np.abs(Q @ Q.T - want).max() < 1e-5


def test_fullrank_f32_matches_full():
    rng = np.random.default_rng(6)
    codes = rng.integers(0, 8, size=(50, 10)).astype(np.int32)
    mem = P.LeafMembership(codes, np.full(10, 8, np.int32))
    full = P.full_proximity(mem)
    rep = P.lowrank_proximity(mem, rank=min(50, mem.total_leaves), mode="f32")
    for i in range(0, 50, 3):
        for j in range(50):
            assert abs(rep.entry(i, j) - full.entry(i, j)) <= 1e-4


def test_mode_bytes(synth2k):
    ds, forest = synth2k
    mem = P.leaf_membership(forest, ds)
    i8 = P.lowrank_proximity(mem, rank=32, mode="i8")
    nf4 = P.lowrank_proximity(mem, rank=32, mode="nf4")
    f16 = P.lowrank_proximity(mem, rank=32, mode="f16")
    assert nf4.factor.data.nbytes * 2 == i8.factor.data.nbytes
    assert f16.factor.data.dtype == np.float16
    assert frob_rel(nf4.dequantized(), i8.dequantized()) < 0.2


@pytest.mark.parametrize("mode", ["i8", "f16", "f32", "nf4"])
def test_quantize_bit_exact_vs_oracle(orc, mode):
    rng = np.random.default_rng(21)
    x = rng.normal(size=(301, 7)) * rng.uniform(0.01, 5, size=7)
    x[:, 3] = 0.0
    x[5, 1] = 0.5 * np.abs(x[:, 1]).max() / 127 * 127  # exercise rounding ties region
    qf = Qz.quantize(x, mode)
    data, scales = orc.quantize(x, mode)
    assert np.array_equal(qf.data.reshape(data.shape), data)
    if scales is not None:
        assert np.array_equal(qf.scales, scales)
    np.testing.assert_array_equal(qf.dequantize(), orc.dequantize(data, scales, mode, x.shape))


def test_quantize_1d_block(orc):
    x = np.linspace(-3, 2, 77)
    qf = Qz.quantize(x, "i8")
    data, scales = orc.quantize(x, "i8")
    assert qf.data.shape == (77,) and np.array_equal(qf.data, data.reshape(-1))


def test_tree_shard_sum_equals_whole(synth2k):
    """Sketch partials of tree shards add up to the whole-forest sketch (the
    all-reduce of the multi-GPU path is a plain sum; gloo test in
    test_distributed.py)."""
    import torch
    ds, forest = synth2k
    k = 12
    X32 = torch.randn((ds.n, k), dtype=torch.float32, device="cuda")
    Yw = P._Sketch(P.leaf_membership(forest, ds).device(), k).apply(X32, k)
    Ys = sum(P._Sketch(P.leaf_membership(forest, ds, trees=t).device(), k)
             .apply(X32, k, reduce=False) for t in [(0, 13), (13, 31), (31, 40)])
    # per-batch f32 partial sums (rfxc_sketch_pass): shard boundaries change
    # the batching, so agreement is to f32 rounding of the batch partials
    assert torch.allclose(Ys, Yw, rtol=1e-6, atol=1e-6 * float(Yw.abs().max()))
