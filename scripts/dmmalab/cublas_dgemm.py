"""cuBLAS DGEMM (torch.matmul f64) at 8192^3 — the ncu target for reading
its kernel configuration (grid, block, registers, shared memory) against
the DMMA DGEMM (dev tool)."""
import torch

n = 8192
a = torch.rand(n, n, dtype=torch.float64, device="cuda")
b = torch.rand(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    c = a @ b
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
c = a @ b
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e)
print({"n": n, "ms": ms, "TFLOPs": 2 * n ** 3 / ms / 1e9})
