"""When each traversal chunk finishes in the end-to-end call (uploads issued
as leaf_membership issues them) vs with every input already on the device.
    python scripts/trav_e2e_probe.py [CONFIG]"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, make_inputs  # noqa: E402
from paper_2511_19493_b200 import proximity as P  # noqa: E402
from paper_2511_19493_b200.device import DeviceForest, DeviceValues, traverse  # noqa: E402

_Event = torch.cuda.Event
torch.cuda.Event = lambda *a, **k: _Event(enable_timing=True)  # the chunk marks get timestamps
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "100k"]
ds, forest = make_inputs(cfg, (0, cfg["B"]), os.cpu_count())


def run(resident):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    if resident:
        dv, df = DeviceValues(ds.values), DeviceForest(forest)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        nb, tm, done = traverse(df, dv)
    else:
        mem = P.leaf_membership(forest, ds)
        done = mem._dev.chunks
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    torch.cuda.synchronize()
    ev = []
    for c0, c1, e in done:
        e.synchronize()
        ev.append((c0, c1, e0.elapsed_time(e)))
    return ev, e0.elapsed_time(e1)


for resident in (False, True):
    for _ in range(2):
        run(resident)
    res = [run(resident) for _ in range(5)]
    ends = np.median([[t for *_, t in r[0]] for r in res], axis=0)
    tot = np.median([r[1] for r in res])
    print(("resident " if resident else "e2e      ") +
          " ".join(f"[{c0},{c1}) {t:.2f}" for (c0, c1, _), t in zip(res[0][0], ends)) + f"  total {tot:.2f} ms",
          flush=True)
