"""Time outlier_scores on a random (n, r) factor and a packed triangle."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2511_19493_b200 import proximity as P
from paper_2511_19493_b200.quantize import QuantFactor
n, r = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(0)
Q = (rng.normal(size=(n, r)) * 0.15).astype(np.float32)
lr = P.LowRankQuantized(n=n, rank=r, mode="f32", factor=QuantFactor("f32", (n, r), Q, None),
                        pmax=1.0, tree_count=500)
P.outlier_scores(lr)
torch.cuda.synchronize(); a = time.perf_counter(); P.outlier_scores(lr); torch.cuda.synchronize()
print(f"lowrank outlier n={n} r={r}: {1e3 * (time.perf_counter() - a):.2f} ms", flush=True)
m = 20000
packed = rng.random(m * (m - 1) // 2)
full = P.FullTriangle(n=m, tree_count=500, packed=packed)
P.outlier_scores(full)
torch.cuda.synchronize(); a = time.perf_counter(); P.outlier_scores(full); torch.cuda.synchronize()
print(f"packed outlier n={m}: {1e3 * (time.perf_counter() - a):.2f} ms", flush=True)
