"""Time the k x k Hermitian eigensolve of Rayleigh-Ritz on the GPU: the library's
chfsi_heevd (cuSOLVER zheevd) against torch.linalg.eigh, over the block widths of the
BASELINE configs.

    python scripts/heevd_probe.py
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D  # noqa: E402

dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
for k in (24, 60, 120, 240, 550, 1100, 2200):
    a = torch.randn((k, k), dtype=torch.complex128, device=dev)
    a = a + a.conj().T
    reps = 20 if k <= 600 else 5
    for name, fn in (("chfsi_heevd", lambda: eng.heevd(a.clone())),
                     ("torch.eigh", lambda: torch.linalg.eigh(a))):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        print(f"k={k:5d} {name:12s} {(time.perf_counter() - t) / reps * 1e3:8.3f} ms", flush=True)
