"""Time rfxc_normals for the bench's Omega (n = 100k, k = 40)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2511_19493_b200 import _lib  # noqa: E402
count = 100_000 * 40
out = torch.empty(count, dtype=torch.float64, device="cuda")
for _ in range(3):
    _lib.call("rfxc_normals", 0, 3, count, _lib.ptr(out), _lib.stream_handle())
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(20):
    _lib.call("rfxc_normals", 0, 3, count, _lib.ptr(out), _lib.stream_handle())
ev[1].record()
torch.cuda.synchronize()
print(f"normals {count}: {ev[0].elapsed_time(ev[1]) / 20 * 1e3:.1f} us  checksum {float(out.sum()):.12e}", flush=True)
