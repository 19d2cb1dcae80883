"""Small driver for ncu: a few fused filter-step launches at the bench shape.

    python scripts/profile_filter.py [n] [k] [launches]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2200
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
g = torch.Generator(device=dev)
g.manual_seed(0)
H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
Y1 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
Y0 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
for _ in range(reps):
    eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, Y0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, Y0)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"n={n} k={k}: {ms:.3f} ms, {8.0 * n * n * k / ms / 1e9:.2f} TFLOP/s")
