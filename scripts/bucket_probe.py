"""Time K2 bucketing (rfxc_bucket_trees) alone on the bench forest (100k x 100,
500 trees) and print a checksum of perm / seg (variants must agree)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import torch  # noqa: E402

from paper_2511_19493_b200.device import DeviceForest, DeviceMembership, DeviceValues, traverse  # noqa: E402

cfg = bench.CONFIGS["100k"]
ds, forest = bench.make_inputs(cfg, (0, cfg["B"]), os.cpu_count() or 1)
dv, df = DeviceValues(ds.values), DeviceForest(forest, 0, forest.ntree)
nb, tm, ch = traverse(df, dv)
B = cfg["B"]
for _ in range(3):
    DeviceMembership(nb, tm, df.leaf_counts, 0, B, B).buckets()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    dm = DeviceMembership(nb, tm, df.leaf_counts, 0, B, B)
    perm, seg = dm.buckets()
b.record()
torch.cuda.synchronize()
h = hashlib.sha256(perm.cpu().numpy().tobytes() + seg.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"bucket {a.elapsed_time(b) / 5:.3f} ms  sha {h}", flush=True)
