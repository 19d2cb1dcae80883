"""Time the replicated k x k steps of one sharded outer iteration on the GPU: the
Cholesky + triangular inverse of a CholQR pass (chfsi_cholesky_inverse) and the
Rayleigh-Ritz eigensolve (hermitize + zheevd). Input of scripts/scaling_model.py.

    python scripts/kxk_probe.py > gpurun_out/kxk.json
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D  # noqa: E402

dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
out = {}
for k in (26, 64, 120, 210, 275, 550, 1100, 1650, 2200):
    x = torch.randn((k, 4 * k), dtype=torch.complex128, device=dev)
    g0 = torch.empty((k, k), dtype=torch.complex128, device=dev)
    eng.zgemm("C", "N", k, k, 4 * k, 1.0, x, x, 0.0, g0)  # SPD Gram
    li = torch.empty_like(g0)
    row = {}
    for name, fn in (("chol_inv_s", lambda: eng.cholesky_inverse(g0.clone(), li)),
                     ("eig_s", lambda: eng.heevd(eng.hermitize(g0.clone())))):
        fn()
        torch.cuda.synchronize()
        reps = 10 if k <= 600 else 3
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        row[name] = (time.perf_counter() - t) / reps
    out[str(k)] = row
    print(k, row, file=sys.stderr, flush=True)
print(json.dumps(out))
