"""Time K1 traversal (rfxc_leaf_codes) on the bench-shaped forest subset."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2511_19493_b200.dataset import from_arrays, make_synthetic
from oracle.trainer import train
from paper_2511_19493_b200.forest import TrainConfig
from paper_2511_19493_b200.device import DeviceForest, DeviceValues, traverse, DeviceMembership
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
N = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
X, y = make_synthetic(N, 100, seed=0)
ds = from_arrays(X, y)
forest = train(ds, TrainConfig(ntree=500, iseed=1), trees=(0, B))
dv = DeviceValues(ds.values)
df = DeviceForest(forest, 0, B)
for _ in range(3):
    nb, tm, chunks = traverse(df, dv)
    DeviceMembership(nb, tm, df.leaf_counts, 0, B, B, chunks).buckets()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ev[0].record()
for _ in range(5):
    nb, tm, chunks = traverse(df, dv)
ev[1].record()
for _ in range(5):
    DeviceMembership(nb, tm, df.leaf_counts, 0, B, B, chunks).buckets()
ev[2].record()
torch.cuda.synchronize()
print(f"traverse {ev[0].elapsed_time(ev[1]) / 5:.3f} ms  bucket {ev[1].elapsed_time(ev[2]) / 5:.3f} ms  "
      f"(n={N}, trees={B})", flush=True)
