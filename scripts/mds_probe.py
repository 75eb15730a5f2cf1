"""Time the MDS kernel alone on a random INT8 factor (n, r) — for ncu and
per-iteration cost."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2511_19493_b200 import mds as M, proximity as P
from paper_2511_19493_b200.quantize import QuantFactor
n, r = int(sys.argv[1]), int(sys.argv[2])
its = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [5, 25]
rng = np.random.default_rng(0)
data = rng.integers(-127, 128, size=(n, r)).astype(np.int8)
lr = P.LowRankQuantized(n=n, rank=r, mode="i8",
                        factor=QuantFactor("i8", (n, r), data, rng.uniform(1e-3, 2e-3, r)),
                        pmax=1.0, tree_count=10)
for it in its:
    cfg = M.PowerIterConfig(seed=0, max_iterations=it, tol=1e-30, k=1)
    M.mds_lowrank(lr, cfg)
    torch.cuda.synchronize()
    ts = []
    for rep in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        e = M.mds_lowrank(lr, cfg)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"n={n} r={r} iterations={it}: median {ts[3]:.3f} ms (min {ts[0]:.3f})", flush=True)
