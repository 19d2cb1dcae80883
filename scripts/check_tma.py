import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1305_5120_b200 import _native, device as D
eng = D.Engine.get(torch.device("cuda", 0)); lib = _native.load()
rng = np.random.default_rng(0)
worst = 0
for cfg in (7, 8, 9):
    for split in (1, 3):
        for (m, n, k) in [(64, 32, 8), (100, 37, 53), (1000, 120, 1000), (513, 70, 2000), (8, 8, 8), (3, 5, 7)]:
            lib.chfsi_gemm_override(cfg, split)
            A = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
            B = rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
            C = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
            dA, dB, dC = D.to_device(A, eng.device), D.to_device(B, eng.device), D.to_device(C, eng.device)
            eng.zgemm("N", "N", m, n, k, 0.5 + 0.25j, dA, dB, -0.5, dC)
            ref = (0.5 + 0.25j) * (A @ B) - 0.5 * C
            err = np.linalg.norm(D.to_host(dC) - ref) / np.linalg.norm(ref)
            worst = max(worst, err)
            if err > 1e-13: print("BAD", cfg, split, m, n, k, err, flush=True)
            # filter epilogue
            if m == k:
                Y1 = D.to_device(B, eng.device); Y0 = D.to_device(C, eng.device); out = D.zeros(m, n, eng.device)
                eng.filter_step(dA, Y1, 0.5, -0.25, Y0, 0.125, out)
                ref = 0.5 * (A @ B) - 0.25 * B + 0.125 * C
                err = np.linalg.norm(D.to_host(out) - ref) / np.linalg.norm(ref)
                worst = max(worst, err)
                if err > 1e-13: print("BADF", cfg, split, m, n, err, flush=True)
lib.chfsi_gemm_override(-1, 0)
print("worst", worst)
