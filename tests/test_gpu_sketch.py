"""K4 fused sketch pass (rfxc_sketch_pass) against the CPU oracle's per-tree
restatement of M @ (Mt @ X) (proximity.py:389-398): tree batching, leaves cut
by item boundaries (pieces combined by the last arriver), empty leaves,
determinism, and agreement with the two-kernel path."""

import numpy as np
import pytest

from conftest import cuda_ok, golden

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

from paper_2511_19493_b200 import proximity as P  # noqa: E402


def oracle_sketch(orc, codes, lc, X):
    n, B = codes.shape
    Y = np.empty((n, X.shape[1]))
    orc.lib().orc_sketch_pass(orc._p(np.ascontiguousarray(codes, dtype=np.int32)), n, B,
                              orc._p(np.ascontiguousarray(lc, dtype=np.int32)),
                              orc._p(np.ascontiguousarray(X)), X.shape[1], orc._p(Y), 4)
    return Y


def device_sketch(codes, lc, X, budget=None, fused=True):
    import torch
    mem = P.LeafMembership(codes, lc)
    n, k = X.shape
    sk = P._Sketch(mem.device(), k, budget=budget)
    if not fused:
        sk.fused = False
        sk.S = torch.empty((max(mem.device().total_leaves, 1), sk.ld), dtype=torch.float32,
                           device="cuda")
    X32 = torch.zeros((n, sk.ld), dtype=torch.float32, device="cuda")
    X32[:, :k] = torch.from_numpy(X.astype(np.float32)).cuda()
    return sk, sk.apply(X32, k).cpu().numpy()


def check(orc, codes, lc, k, budget=None, rtol=2e-6):
    rng = np.random.default_rng(k)
    X = rng.normal(size=(codes.shape[0], k)).astype(np.float32).astype(np.float64)
    want = oracle_sketch(orc, codes, lc, X)
    sk, got = device_sketch(codes, lc, X, budget)
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= rtol * scale, (np.abs(got - want).max(), scale)
    return sk, got


@pytest.mark.parametrize("k", [3, 12, 40, 108])
def test_synth2k_matches_oracle(orc, k):
    g = golden("synth2k.npz")
    sk, _ = check(orc, g["codes"], g["leaf_counts"], k)
    assert sk.fused


@pytest.mark.parametrize("budget", [1, 20_000, 200_000])
def test_tree_batches(orc, budget):
    """Tiny budgets force batches of 1..a few trees (many epochs)."""
    g = golden("synth2k.npz")
    sk, _ = check(orc, g["codes"], g["leaf_counts"], 40, budget=budget)
    assert sk.T < g["codes"].shape[1]


def test_big_leaves_span_many_items(orc):
    """Single-leaf and two-leaf trees: every leaf is cut into pieces across
    256-position items and recombined."""
    rng = np.random.default_rng(3)
    n = 3000
    codes = np.stack([np.zeros(n), rng.integers(0, 2, n), rng.permutation(np.arange(n) % 700),
                      (np.arange(n) >= 2999).astype(int)], axis=1).astype(np.int32)
    lc = np.array([1, 2, 700, 2], np.int32)
    sk, _ = check(orc, codes, lc, 40, budget=1)
    assert sk.fused
    check(orc, codes, lc, 40)


def test_empty_leaves(orc):
    """leaf_counts beyond max(code)+1 and gaps in the codes (membership built
    without a forest, tests/test_proximity.py:74-100)."""
    rng = np.random.default_rng(5)
    n, B = 1500, 9
    codes = (rng.integers(0, 40, size=(n, B)) * 3).astype(np.int32)  # only multiples of 3
    lc = np.full(B, 130, np.int32)
    sk, _ = check(orc, codes, lc, 12)
    assert sk.fused  # leaf ids from a run-start search when a leaf is empty
    check(orc, codes, lc, 40, budget=1)  # small batches, pieces across items
    _, a = device_sketch(codes, lc, np.random.default_rng(1).normal(size=(n, 12)))
    _, b = device_sketch(codes, lc, np.random.default_rng(1).normal(size=(n, 12)), fused=False)
    np.testing.assert_allclose(a, b, rtol=1e-6, atol=1e-7 * np.abs(b).max())


def test_deterministic_and_close_to_two_kernel_path(orc):
    g = golden("synth2k.npz")
    codes, lc = g["codes"], g["leaf_counts"]
    X = np.random.default_rng(9).normal(size=(codes.shape[0], 40)).astype(np.float32)
    X = X.astype(np.float64)
    _, a = device_sketch(codes, lc, X)
    _, b = device_sketch(codes, lc, X)
    assert np.array_equal(a, b)
    _, c = device_sketch(codes, lc, X, fused=False)
    np.testing.assert_allclose(a, c, rtol=1e-6, atol=1e-7 * np.abs(c).max())
