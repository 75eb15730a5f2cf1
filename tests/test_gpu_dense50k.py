"""BASELINE configs[2] at full size: synthetic 50k x 100, 500 trees, exact
dense proximity on one B200.  Bit-exact against the CPU oracle
(accumulate_pair_counts_block, _kernels.py:452-480) on row blocks at both
ends of the triangle, and through size-independent properties over the whole
1.25e9-entry triangle: the total equals sum_b sum_l s_l (s_l - 1) / 2 from the
leaf sizes, and the f64 packed triangle is exactly count / B."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


@pytest.fixture(scope="module")
def dense50k(built):
    import os

    from paper_2511_19493_b200 import proximity as P
    from paper_2511_19493_b200.dataset import from_arrays, make_synthetic
    from paper_2511_19493_b200.forest import TrainConfig, train
    X, y = make_synthetic(50_000, 100, seed=0)
    ds = from_arrays(X, y)
    forest = train(ds, TrainConfig(ntree=500, iseed=1), nthreads=os.cpu_count() or 1)
    mem = P.leaf_membership(forest, ds)
    return ds, forest, mem


def test_codes_bit_exact_on_a_tree_sample(orc, dense50k):
    ds, forest, mem = dense50k
    sel = [0, 137, 499]
    codes, lc = orc.leaf_membership([forest.trees[b] for b in sel], forest.col_cat, ds.values)
    got = mem.codes[:, sel]
    assert np.array_equal(got, codes)
    assert np.array_equal(mem.leaf_counts[sel], lc)


def test_counts_bit_exact_and_total(orc, dense50k):
    import torch

    from paper_2511_19493_b200 import _lib
    from paper_2511_19493_b200 import proximity as P
    ds, forest, mem = dense50k
    n, B = mem.n, mem.tree_count
    codes = mem.codes
    # whole triangle as int32 on the device: total = sum of same-leaf pairs
    up = P.pair_counts_device(mem, _lib.UPPER_I32)
    total = int(up.sum(dtype=torch.int64).item())
    want = 0
    for b in range(B):
        s = np.bincount(codes[:, b], minlength=int(mem.leaf_counts[b])).astype(np.int64)
        want += int((s * (s - 1) // 2).sum())
    assert total == want
    # bit-exact row blocks at both ends against the oracle
    for lo, hi in ((0, 48), (n - 300, n - 256)):
        blk = P.pair_counts_device(mem, _lib.BLOCK_I32, lo, hi).view(hi - lo, n).cpu().numpy()
        assert np.array_equal(blk, orc.block_counts(codes, mem.leaf_counts, lo, hi))
        a, b = P._row_start(n, lo), P._row_start(n, hi)
        packed = up[a:b].cpu().numpy()
        rows = [blk[i - lo, i + 1:] for i in range(lo, hi)]
        assert np.array_equal(packed, np.concatenate(rows))
    del up
    # packed f64 = count / B as one IEEE division (proximity.py:200)
    f = P.pair_counts_device(mem, _lib.UPPER_F64, 0, 48).cpu().numpy()
    blk = orc.block_counts(codes, mem.leaf_counts, 0, 48)
    want = np.concatenate([blk[i, i + 1:] for i in range(48)]) / float(B)
    assert np.array_equal(f, want)
