"""Run traversal, bucketing and one sketch pass on a 100k x 100 synthetic
forest subset (default 64 trees) — a short command for ncu captures of the
K1/K2/K4 kernels with the same per-tree shapes as the bench workload."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2511_19493_b200.dataset import from_arrays, make_synthetic
from oracle.trainer import train
from paper_2511_19493_b200.forest import TrainConfig
from paper_2511_19493_b200.device import DeviceForest, DeviceMembership, DeviceValues, traverse
from paper_2511_19493_b200 import proximity as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
N = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
X, y = make_synthetic(N, 100, seed=0)
ds = from_arrays(X, y)
t0 = time.time()
forest = train(ds, TrainConfig(ntree=500, iseed=1), trees=(0, B))
print(f"trained {B} trees in {time.time()-t0:.1f}s", flush=True)
dv = DeviceValues(ds.values)
df = DeviceForest(forest, 0, B)
for rep in range(2):
    nb, tm, chunks = traverse(df, dv)
    dm = DeviceMembership(nb, tm, df.leaf_counts, 0, B, B, chunks)
    sk = P._Sketch(dm, 40)
    if rep == 0:
        lc = dm.leaf_counts
        print("has_empty", int(dm.has_empty.item()), "T", getattr(sk, "T", None), "nbuf", getattr(sk, "nbuf", None), "s_rows",
              getattr(sk, "s_rows", None), "leaves/tree", lc.mean(), lc.max(), flush=True)
    X32 = torch.randn((ds.n, sk.ld), dtype=torch.float32, device="cuda")
    sk.apply(X32, 40)
torch.cuda.synchronize()
print("done", flush=True)
