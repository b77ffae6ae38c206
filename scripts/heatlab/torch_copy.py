"""torch copy_ bandwidth at the driver's size (1 Gi bf16) and at heat_3d's
(400^3 f64), best-of and mean over back-to-back launches (CUDA events)."""
import json

import torch

for name, numel, dt in (("bf16_1Gi", 1 << 30, torch.bfloat16), ("f64_400c", 400 ** 3, torch.float64)):
    a = torch.rand(numel, device="cuda").to(dt)
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    ts = []
    for r in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        src, dst = (a, b) if r % 2 == 0 else (b, a)
        e0.record()
        dst.copy_(src)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    nb = 2 * a.numel() * a.element_size()
    print(json.dumps({"copy": name, "best_GBps": nb / min(ts) / 1e6, "mean_GBps": nb / (sum(ts) / len(ts)) / 1e6}))
