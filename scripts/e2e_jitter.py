"""Per-step wall time of the end-to-end public-API step (bench workload), 30
steps, with Python's garbage collector on and frozen:
    python scripts/e2e_jitter.py"""
import gc
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, make_inputs  # noqa: E402
from paper_2511_19493_b200 import mds as M  # noqa: E402
from paper_2511_19493_b200 import proximity as P  # noqa: E402

cfg = CONFIGS["100k"]
ds, forest = make_inputs(cfg, (0, cfg["B"]), os.cpu_count())
mcfg = M.PowerIterConfig(seed=0)


def step():
    lr = P.lowrank_proximity(P.leaf_membership(forest, ds), cfg["rank"], cfg["mode"], seed=0)
    emb = M.mds_lowrank(lr, mcfg)
    assert lr.factor.data.shape[0] == cfg["n"] and emb.coordinates.shape[0] == cfg["n"]


for mode in ("gc on", "gc frozen", "gc on"):
    if mode == "gc frozen":
        gc.collect()
        gc.freeze()
        gc.disable()
    else:
        gc.enable()
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    ts = np.array(ts)
    print(f"{mode:10s} median {np.median(ts):.2f} mean {ts.mean():.2f} max {ts.max():.2f} ms; "
          f">18 ms: {int((ts > 18).sum())}", flush=True)
