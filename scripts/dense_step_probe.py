"""Where the dense (configs[2]) step's wall time goes on the host: per call
host durations (no extra syncs) next to the device time of the step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (sets PYTORCH_CUDA_ALLOC_CONF before torch initialises CUDA)
import torch  # noqa: E402
from paper_2511_19493_b200 import _lib  # noqa: E402
from paper_2511_19493_b200.device import DeviceForest, DeviceMembership, DeviceValues, traverse  # noqa: E402
from paper_2511_19493_b200.proximity import LeafMembership, pair_counts_device  # noqa: E402

cfg = bench.CONFIGS["50k-dense"]
ds, forest = bench.make_inputs(cfg, (0, cfg["B"]), os.cpu_count() or 1)
dv = DeviceValues(ds.values)
df = DeviceForest(forest, 0, forest.ntree)
B = cfg["B"]
for rep in range(int(os.environ.get("REPS", "6"))):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t = [time.perf_counter()]
    nb, tm, chunks = traverse(df, dv)
    t.append(time.perf_counter())
    dm = DeviceMembership(nb, tm, df.leaf_counts, 0, B, B, chunks)
    mem = LeafMembership(leaf_counts=df.leaf_counts, _dev=dm)
    t.append(time.perf_counter())
    out = pair_counts_device(mem, _lib.UPPER_F64)
    t.append(time.perf_counter())
    e1.record()
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(f"device {e0.elapsed_time(e1):.2f} ms | host traverse {d[0]:.2f} membership {d[1]:.2f} "
          f"pair_counts {d[2]:.2f} wait {d[3]:.2f}", flush=True)
    del out
