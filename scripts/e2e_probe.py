"""Break down the end-to-end public-API call of the bench workload."""
import os, sys, time
sys.path.insert(0, ".")
import torch
from bench import CONFIGS, make_inputs
from paper_2511_19493_b200 import proximity as P, mds as M
from paper_2511_19493_b200.device import DeviceForest, DeviceValues
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "100k"]
ds, forest = make_inputs(cfg, (0, cfg["B"]), os.cpu_count())
def t(label, fn):
    torch.cuda.synchronize(); a = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    print(f"{label:28s} {1e3 * (time.perf_counter() - a):8.2f} ms", flush=True); return r
for rep in range(3):
    print("rep", rep)
    dv = t("DeviceValues", lambda: DeviceValues(ds.values))
    df = t("DeviceForest (pack+H2D)", lambda: DeviceForest(forest, 0, forest.ntree))
    mem = t("leaf_membership (all)", lambda: P.leaf_membership(forest, ds))
    lr = t("lowrank_proximity", lambda: P.lowrank_proximity(mem, cfg["rank"], cfg["mode"], seed=0))
    emb = t("mds_lowrank", lambda: M.mds_lowrank(lr, M.PowerIterConfig(seed=0)))
