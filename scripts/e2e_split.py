"""Where the end-to-end step's time goes (steady state, bench workload): CUDA
events on the compute stream at each public-API boundary of the e2e loop,
host timestamps beside them.
    python scripts/e2e_split.py [CONFIG]"""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, make_inputs  # noqa: E402
from paper_2511_19493_b200 import mds as M  # noqa: E402
from paper_2511_19493_b200 import proximity as P  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "100k"]
ds, forest = make_inputs(cfg, (0, cfg["B"]), os.cpu_count())
mcfg = M.PowerIterConfig(seed=0)


def step(rec):
    rec("start")
    mem = P.leaf_membership(forest, ds)
    rec("leaf_membership")
    lr = P.lowrank_proximity(mem, cfg["rank"], cfg["mode"], seed=0)
    rec("lowrank")
    emb = M.mds_lowrank(lr, mcfg)
    rec("mds")
    assert lr.factor.data.shape[0] == cfg["n"] and emb.coordinates.shape[0] == cfg["n"]
    rec("results on host")


for _ in range(3):
    step(lambda name: None)
torch.cuda.synchronize()
rows = []
for _ in range(8):
    marks = []

    def rec(name):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        marks.append((name, ev, time.perf_counter()))
    step(rec)
    torch.cuda.synchronize()
    rows.append(marks)
names = [m[0] for m in rows[0]]
dev = np.array([[r[i][1].elapsed_time(r[i + 1][1]) for i in range(len(r) - 1)] for r in rows])
host = np.array([[1e3 * (r[i + 1][2] - r[i][2]) for i in range(len(r) - 1)] for r in rows])
gap = np.array([rows[j + 1][0][1].elapsed_time(rows[j + 1][0][1]) for j in range(len(rows) - 1)])
for i in range(len(names) - 1):
    print(f"{names[i]:>16s} -> {names[i + 1]:<16s} device {np.median(dev[:, i]):7.3f} ms   host {np.median(host[:, i]):7.3f} ms")
print(f"{'step':>36s} device {np.median(dev.sum(1)):7.3f} ms   host {np.median(host.sum(1)):7.3f} ms")
