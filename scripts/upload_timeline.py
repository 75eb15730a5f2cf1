"""Timeline of leaf_membership's PCIe uploads and traversal launches (CUDA
events on the copy and compute streams), to see when the first traversal
starts relative to the uploads."""
import os, sys
sys.path.insert(0, ".")
import torch
from bench import CONFIGS, make_inputs
from paper_2511_19493_b200 import proximity as P, device as D
cfg = CONFIGS["100k"]
ds, forest = make_inputs(cfg, (0, cfg["B"]), os.cpu_count())
for rep in range(3):
    P.leaf_membership(forest, ds)
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
cs = D._copy_stream(torch.device("cuda", 0))
marks = []
orig_call = D._lib.call
def call(name, *a):
    orig_call(name, *a)
    ev = torch.cuda.Event(enable_timing=True)
    ev.record(torch.cuda.current_stream())
    marks.append((name, a[5] if name == "rfxc_h2d_rows" else (a[4], a[5], a[8], a[9]) if name == "rfxc_leaf_codes_rows" else "", ev))
D._lib.call = call
P._lib.call = call
mem = P.leaf_membership(forest, ds)
end = torch.cuda.Event(enable_timing=True); end.record(); torch.cuda.synchronize()
for name, arg, ev in marks:
    print(f"{t0.elapsed_time(ev):8.3f} ms  {name} {arg}")
print(f"{t0.elapsed_time(end):8.3f} ms  end")
