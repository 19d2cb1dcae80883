import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D
eng = D.Engine.get(torch.device("cuda", 0)); dev = eng.device
for n, k in ((1000, 21), (1000, 120), (2000, 60)):
    H = torch.randn((n, n), dtype=torch.complex128, device=dev)
    Y = torch.randn((k, n), dtype=torch.complex128, device=dev); W = torch.empty_like(Y)
    for _ in range(3): eng.filter(H, Y, W, 15, 0.5, 3.0, -3.0)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(200): eng.filter(H, Y, W, 15, 0.5, 3.0, -3.0)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 200
    print(f"n={n} k={k}: {dt*1e6:8.1f} us per filter call (15 steps)", flush=True)
