"""ncu driver: filter calls (chfsi_filter, 3M sum planes when on) at one shape with H
declared, as inside a solve.

    python scripts/profile_filter_call.py [n] [k] [degree] [forced cfg] [forced split]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2200
deg = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if len(sys.argv) > 4:
    from paper_1305_5120_b200 import _native  # noqa: E402
    assert _native.load().chfsi_gemm_override(int(sys.argv[4]),
                                              int(sys.argv[5]) if len(sys.argv) > 5 else 0) == 0
dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
g = torch.Generator(device=dev)
g.manual_seed(0)
H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
Y = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g) * 1e-3
W = torch.empty_like(Y)
eng.declare_operator(H)
for _ in range(2):
    eng.filter(H, Y, W, deg, -1.0, 1.0, -2.0)
torch.cuda.synchronize()
print("ok", n, k, deg)
