"""HBM-bound GEMV of the Lanczos bound (core.py:202-256) at c4 size: y = H v with
n = 20000 (6.4 GB of H per product). Prints the CUDA-event time per GEMV and the
achieved bandwidth against the measured copy peak, and the time of a full 10-step
lanczos_bound (10 GEMVs + reorthogonalisation + host syncs). Run under ncu for the
kernel's own DRAM bytes: profiles/r02/gemv_*.csv."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
g = torch.Generator(device=dev)
g.manual_seed(0)
H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
x = torch.randn((1, n), dtype=torch.complex128, device=dev, generator=g)
y = torch.empty_like(x)
for _ in range(3):
    eng.zgemm("N", "N", n, 1, n, 1.0, H, x, 0.0, y)
torch.cuda.synchronize()
stream = torch.cuda.current_stream(dev)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(stream)
for _ in range(reps):
    eng.zgemm("N", "N", n, 1, n, 1.0, H, x, 0.0, y)
b.record(stream)
torch.cuda.synchronize()
t = a.elapsed_time(b) * 1e-3 / reps
algo_bytes = 16.0 * n * n + 32.0 * n  # H once, x read, y written
v0 = np.random.default_rng(1).standard_normal(n) + 0j
v0 /= np.linalg.norm(v0)
vb = D.to_device(v0, dev)
eng.lanczos_bound(H, vb, 10)
torch.cuda.synchronize()
la, lb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
la.record(stream)
eng.lanczos_bound(H, vb, 10)
lb.record(stream)
torch.cuda.synchronize()
print(json.dumps({"n": n, "gemv_ms": t * 1e3, "gemv_gbs": algo_bytes / t / 1e9,
                  "algorithmic_bytes": algo_bytes, "peak_gbs_measured_copy": 6555.0,
                  "frac": algo_bytes / t / 1e9 / 6555.0,
                  "lanczos10_ms": la.elapsed_time(lb)}))
