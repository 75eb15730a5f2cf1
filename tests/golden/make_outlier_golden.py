"""Golden outlier scores from the reference (run in the build container,
where /root/reference is importable): outlier_scores (proximity.py:432-485)
of the Wine B=50 (iseed 17) FullTriangle, TriBlock (tau 0.05) and i8 rank-16
(seed 5) factor — the same objects wine50.npz holds.  Output:
outlier_wine50.npz."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import rfx  # noqa: E402
from rfx import proximity as rprox  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    from sklearn.datasets import load_wine
    w = load_wine()
    ds = rfx.from_arrays(w.data, w.target)
    f = rfx.train(ds, rfx.TrainConfig(ntree=50, iseed=17))
    mem = rprox.leaf_membership(f, ds)
    full = rprox.full_proximity(mem)
    tb = rprox.triblock_proximity(mem, tau=0.05)
    lr = rprox.lowrank_proximity(mem, rank=16, mode="i8", seed=5)
    g = np.load(os.path.join(HERE, "wine50.npz"))
    assert np.array_equal(full.packed, g["packed"]) and np.array_equal(lr.factor.data, g["lr_data"])
    np.savez_compressed(os.path.join(HERE, "outlier_wine50.npz"),
                        full=rprox.outlier_scores(full),
                        full_floor=rprox.outlier_scores(full, clamp_floor=0.05),
                        triblock=rprox.outlier_scores(tb),
                        lowrank=rprox.outlier_scores(lr),
                        lowrank_floor=rprox.outlier_scores(lr, clamp_floor=0.1))


if __name__ == "__main__":
    main()
