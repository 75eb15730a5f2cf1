import sys
sys.path.insert(0, ".")
import torch
from paper_2511_19493_b200 import _lib
k = 40
G = torch.randn(k, k, dtype=torch.float64, device="cuda")
G = G @ G.T + 40 * torch.eye(k, dtype=torch.float64, device="cuda")
R = torch.empty_like(G)
for _ in range(5):
    _lib.call("rfxc_chol_inv", _lib.ptr(G), k, 1e-10, _lib.ptr(R), _lib.stream_handle())
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(100):
    _lib.call("rfxc_chol_inv", _lib.ptr(G), k, 1e-10, _lib.ptr(R), _lib.stream_handle())
b.record(); torch.cuda.synchronize()
print("chol_inv back-to-back avg us", a.elapsed_time(b) * 10)
