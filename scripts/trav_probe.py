"""Time K1 traversal (rfxc_leaf_codes) on a bench-shaped forest subset:
    python scripts/trav_probe.py TREES N P [NTREE_TOTAL]
prints the traversal time per call and the SHA-256 of the codes (so tree-top
staging variants, RFXC_TRAV_TOP=63/127/255, can be checked for equality)."""
import hashlib
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from oracle.trainer import train  # noqa: E402
from paper_2511_19493_b200.dataset import from_arrays, make_synthetic  # noqa: E402
from paper_2511_19493_b200.device import DeviceForest, DeviceValues, traverse  # noqa: E402
from paper_2511_19493_b200.forest import TrainConfig  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
N = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
P = int(sys.argv[3]) if len(sys.argv) > 3 else 100
BT = int(sys.argv[4]) if len(sys.argv) > 4 else 500
X, y = make_synthetic(N, P, seed=0)
ds = from_arrays(X, y)
forest = train(ds, TrainConfig(ntree=BT, iseed=1), trees=(0, B))
dv = DeviceValues(ds.values)
df = DeviceForest(forest, 0, B)
for _ in range(3):
    nb, tm, chunks = traverse(df, dv)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(5):
    nb, tm, chunks = traverse(df, dv)
ev[1].record()
torch.cuda.synchronize()
sha = hashlib.sha256(tm.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"traverse {ev[0].elapsed_time(ev[1]) / 5:.3f} ms  (n={N}, p={P}, trees={B}) codes {sha}",
      flush=True)

if len(sys.argv) > 5 and sys.argv[5] in ("sorted", "strided"):
    # the same traversal with the samples reordered by their leaf in tree 0
    # (neighbouring lanes then share most of their paths)
    import numpy as np
    from paper_2511_19493_b200.dataset import from_arrays as fa
    order = np.argsort(tm[0].cpu().numpy(), kind="stable")
    if sys.argv[5] == "strided":
        # 128-sample tiles stay coherent, but consecutive tiles (the CTAs
        # resident together) come from far-apart parts of the sorted order
        tiles = (N + 127) // 128
        stride = max(1, tiles // 296) | 1
        while np.gcd(stride, tiles) != 1:
            stride += 2
        pt = (np.arange(tiles) * stride) % tiles
        parts = [order[t * 128:(t + 1) * 128] for t in pt]
        order = np.concatenate(parts)
    ds2 = fa(np.ascontiguousarray(X[order]), y[order])
    dv2 = DeviceValues(ds2.values)
    for _ in range(3):
        traverse(df, dv2)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(5):
        nb2, tm2, _c = traverse(df, dv2)
    ev[1].record()
    torch.cuda.synchronize()
    same = bool((tm2.cpu().numpy() == tm.cpu().numpy()[:, order]).all())
    print(f"{sys.argv[5]} by tree-0 leaf: traverse {ev[0].elapsed_time(ev[1]) / 5:.3f} ms, codes permuted "
          f"equal: {same}", flush=True)
