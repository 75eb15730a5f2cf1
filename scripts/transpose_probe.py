"""Time rfxc_transpose_i32 on the (B, n) -> (n, B) codes shape."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2511_19493_b200 import _lib  # noqa: E402
B, n = 500, 100_000
a = torch.randint(0, 1000, (B, n), dtype=torch.int32, device="cuda")
b = torch.empty((n, B), dtype=torch.int32, device="cuda")
for _ in range(3):
    _lib.call("rfxc_transpose_i32", _lib.ptr(a), B, n, _lib.ptr(b), _lib.stream_handle())
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(20):
    _lib.call("rfxc_transpose_i32", _lib.ptr(a), B, n, _lib.ptr(b), _lib.stream_handle())
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / 20
assert torch.equal(b, a.t())
print(f"transpose (B={B}, n={n}) int32: {ms * 1e3:.1f} us, {2 * B * n * 4 / ms / 1e6:.0f} GB/s", flush=True)
