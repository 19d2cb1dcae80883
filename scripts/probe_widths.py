"""Per-step time of filter calls (planner's pick, H declared as in a solve) over block
widths at n = 20000: the shard-width speed table of scripts/scaling_model.py.

    python scripts/probe_widths.py > gpurun_out/widths.json
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
widths = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else \
    [8, 16, 26, 32, 48, 64, 96, 128, 160, 210, 275, 400, 550, 800, 1100, 1650, 2200]
dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
g = torch.Generator(device=dev)
g.manual_seed(0)
H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
eng.declare_operator(H)
DEG = 4
out = []
for k in widths:
    Y0 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g) * 1e-3
    Y = torch.empty_like(Y0)
    W = torch.empty_like(Y0)
    Y.copy_(Y0)
    eng.filter(H, Y, W, DEG, -1.0, 1.0, -2.0)
    torch.cuda.synchronize()
    reps = max(2, min(6, int(6e12 / (8.0 * n * n * k * DEG))))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        Y.copy_(Y0)
        eng.filter(H, Y, W, DEG, -1.0, 1.0, -2.0)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / (reps * DEG)
    out.append({"n": n, "k": k, "cfg": -1, "ms": ms, "tflops": 8.0 * n * n * k / ms / 1e9})
    print(json.dumps(out[-1]), file=sys.stderr, flush=True)
eng.declare_operator(None)
print(json.dumps(out, indent=1))
