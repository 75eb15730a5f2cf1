"""Small end-to-end run of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): synthetic 2000 x 20, 40 trees —
traversal, bucketing, both pair-count kernels (all layouts), TriBlock,
the implicit sketch (fused pass + wide two-kernel path), CholeskyQR,
quantisation (all modes), pmax, MDS (int8-resident and f64 slices),
outlier scores and OOB votes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.trainer import train  # noqa: E402
from paper_2511_19493_b200 import _lib, mds as M, proximity as P  # noqa: E402
from paper_2511_19493_b200.dataset import from_arrays, make_synthetic  # noqa: E402
from paper_2511_19493_b200.forest import TrainConfig  # noqa: E402

X, y = make_synthetic(2000, 20, seed=1)
ds = from_arrays(X, y)
forest = train(ds, TrainConfig(ntree=40, iseed=1))
mem = P.leaf_membership(forest, ds)
for kern in ("leaf", "tile"):
    os.environ["RFX_PAIRS_KERNEL"] = kern
    for layout in (_lib.UPPER_I32, _lib.UPPER_F64):
        P.pair_counts_device(mem, layout)
    P.pair_counts_device(mem, _lib.BLOCK_I32, 100, 300)
full = P.full_proximity(mem)
tb = P.triblock_proximity(mem, tau=0.05)
for mode in ("i8", "f32", "f16", "nf4"):
    lr = P.lowrank_proximity(mem, rank=16, mode=mode, seed=3)
lr = P.lowrank_proximity(mem, rank=32, mode="i8", seed=0)
emb = M.mds_lowrank(lr, M.PowerIterConfig(seed=0, max_iterations=20))
os.environ["RFXC_MDS_F64"] = "1"
emb2 = M.mds_lowrank(lr, M.PowerIterConfig(seed=0, max_iterations=20))
wide = P.lowrank_proximity(mem, rank=130, mode="f32", seed=0)  # k > 128: two-kernel sketch
P.outlier_scores(full)
P.outlier_scores(lr)
P.oob_votes(forest, ds, mem)
torch.cuda.synchronize()
print("sanitize probe done", emb.eigenvalues, emb2.eigenvalues)
