"""K1 with the samples in three orders (as given; sorted by their tree-0 leaf;
sorted tiles strided so co-resident CTAs sit far apart), each timed 3x5
calls alternately in one process:
    python scripts/trav_order_probe.py TREES N P NTREE_TOTAL"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.trainer import train  # noqa: E402
from paper_2511_19493_b200.dataset import from_arrays, make_synthetic  # noqa: E402
from paper_2511_19493_b200.device import DeviceForest, DeviceValues, traverse  # noqa: E402
from paper_2511_19493_b200.forest import TrainConfig  # noqa: E402

B, N, P, BT = (int(a) for a in sys.argv[1:5])
X, y = make_synthetic(N, P, seed=0)
ds = from_arrays(X, y)
forest = train(ds, TrainConfig(ntree=BT, iseed=1), trees=(0, B))
df = DeviceForest(forest, 0, B)
dv = DeviceValues(ds.values)
nb, tm, _ = traverse(df, dv)
order = np.argsort(tm[0].cpu().numpy(), kind="stable")
tiles = (N + 127) // 128
stride = max(1, tiles // 296) | 1
while np.gcd(stride, tiles) != 1:
    stride += 2
strided = np.concatenate([order[t * 128:(t + 1) * 128] for t in (np.arange(tiles) * stride) % tiles])
vals = {"given": dv}
for name, o in (("sorted", order), ("strided", strided)):
    vals[name] = DeviceValues(from_arrays(np.ascontiguousarray(X[o]), y[o]).values)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
res = {k: [] for k in vals}
for rep in range(3):
    for name, v in vals.items():
        for _ in range(2):
            traverse(df, v)
        torch.cuda.synchronize()
        ev[0].record()
        for _ in range(5):
            traverse(df, v)
        ev[1].record()
        torch.cuda.synchronize()
        res[name].append(ev[0].elapsed_time(ev[1]) / 5)
print(f"n={N} p={P} trees={B}: " + "  ".join(f"{k} {min(t):.3f}-{max(t):.3f} ms" for k, t in res.items()),
      flush=True)
