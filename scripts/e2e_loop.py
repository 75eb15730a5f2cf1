"""The bench's end-to-end loop (public API, host inputs), per-step wall and
CUDA-event times, no synchronisation inside a step."""
import os, sys, time
sys.path.insert(0, ".")
import torch
from bench import CONFIGS, make_inputs
from paper_2511_19493_b200 import proximity as P, mds as M
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "100k"]
ds, forest = make_inputs(cfg, (0, cfg["B"]), os.cpu_count())
mcfg = M.PowerIterConfig(seed=0)
for step in range(6):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a = time.perf_counter(); e0.record()
    mem = P.leaf_membership(forest, ds)
    b = time.perf_counter()
    lr = P.lowrank_proximity(mem, cfg["rank"], cfg["mode"], seed=0)
    c = time.perf_counter()
    emb = M.mds_lowrank(lr, mcfg)
    e1.record(); torch.cuda.synchronize(); d = time.perf_counter()
    print(f"step {step}: events {e0.elapsed_time(e1):7.2f} ms  host: membership {1e3*(b-a):6.2f} "
          f"lowrank {1e3*(c-b):6.2f} mds {1e3*(d-c):6.2f}", flush=True)
