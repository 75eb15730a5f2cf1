"""BASELINE configs[1] at full size: synthetic 10k x 50, 4 classes, 500
trees — dense + TriBlock upper-triangle proximity (triblock_proximity,
proximity.py:275-327).  Checked against the bit-exact int32 triangle (itself
checked against the CPU oracle on row blocks here): with the default tau every
non-zero pair lands in the dense tier (1/B > tau), with tau =
0.05 the tiers split by value; tiers are disjoint, (i, j)-sorted and hold
exactly count / B for every count > 0."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


@pytest.fixture(scope="module")
def tri10k(built):
    import os

    from paper_2511_19493_b200 import _lib
    from paper_2511_19493_b200 import proximity as P
    from paper_2511_19493_b200.dataset import from_arrays, make_synthetic
    from oracle.trainer import train
    from paper_2511_19493_b200.forest import TrainConfig
    X, y = make_synthetic(10_000, 50, seed=0)
    ds = from_arrays(X, y)
    forest = train(ds, TrainConfig(ntree=500, iseed=1), nthreads=os.cpu_count() or 1)
    mem = P.leaf_membership(forest, ds)
    counts = P.pair_counts_device(mem, _lib.UPPER_I32).cpu().numpy()
    return mem, counts


def _expected(mem, counts, tau):
    n, B = mem.n, mem.tree_count
    iu = np.triu_indices(n, k=1)
    v = counts / float(B)
    keep = v > 1e-6
    hot = keep & (v >= tau)
    cold = keep & (v < tau)
    return (iu[0][hot], iu[1][hot], v[hot]), (iu[0][cold], iu[1][cold], v[cold])


def test_counts_row_blocks_vs_oracle(orc, tri10k):
    from paper_2511_19493_b200 import proximity as P
    mem, counts = tri10k
    n = mem.n
    for lo, hi in ((0, 64), (n - 200, n - 100)):
        blk = orc.block_counts(mem.codes, mem.leaf_counts, lo, hi)
        a, b = P._row_start(n, lo), P._row_start(n, hi)
        assert np.array_equal(counts[a:b], np.concatenate([blk[i - lo, i + 1:] for i in range(lo, hi)]))


@pytest.mark.parametrize("tau", [1e-4, 0.05])
def test_triblock_tiers(tri10k, tau):
    from paper_2511_19493_b200 import proximity as P
    mem, counts = tri10k
    tb = P.triblock_proximity(mem, tau=tau)
    (hi_i, hi_j, hi_v), (co_i, co_j, co_v) = _expected(mem, counts, tau)
    d = tb.dense
    assert np.array_equal(d.i, hi_i) and np.array_equal(d.j, hi_j) and np.array_equal(d.v, hi_v)
    assert np.array_equal(tb.sparse_i, co_i) and np.array_equal(tb.sparse_j, co_j)
    assert np.array_equal(tb.sparse_v, co_v)
    if tau == 1e-4:
        assert tb.sparse_count == 0 and tb.dense_count == int((counts > 0).sum())
    else:
        assert tb.sparse_count > 0 and tb.dense_count > 0
    # spot entries through the reference accessor
    i, j = int(hi_i[len(hi_i) // 2]), int(hi_j[len(hi_j) // 2])
    assert tb.entry(i, j) == tb.entry(j, i) == hi_v[len(hi_v) // 2]
