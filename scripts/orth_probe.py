"""Time orthonormalize (shifted CholeskyQR3) and its kernels on an n x k
Gaussian matrix (for ncu -k regex:gram|chol|matmul)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2511_19493_b200 import proximity as P
n, k = int(sys.argv[1]), int(sys.argv[2])
Y = torch.randn((n, k), dtype=torch.float64, device="cuda")
for _ in range(3):
    P.orthonormalize(Y, (k + 3) // 4 * 4)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    P.orthonormalize(Y, (k + 3) // 4 * 4)
b.record()
torch.cuda.synchronize()
print(f"orthonormalize n={n} k={k}: {a.elapsed_time(b) / 10:.3f} ms", flush=True)
