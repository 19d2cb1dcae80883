import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1305_5120_b200 import _native, device as D
eng = D.Engine.get(torch.device("cuda", 0)); lib = _native.load(); dev = eng.device
for n in (4096, 20000):
    g = torch.Generator(device=dev); g.manual_seed(1)
    A = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)   # block: row j = column j
    for k in (6, 26, 64):
        Y = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
        C = torch.zeros((k, n), dtype=torch.complex128, device=dev)
        eng.zgemm("N", "N", n, k, n, 1.0, A, Y, 0.0, C)
        ref = (A.T @ Y.T).T    # H = A^T (row-major), H @ Ycols
        cfg, spl = ctypes.c_int(), ctypes.c_int()
        lib.chfsi_gemm_plan(eng.h, 0, 0, 0, n, k, n, ctypes.byref(cfg), ctypes.byref(spl))
        err = (torch.linalg.norm(C - ref) / torch.linalg.norm(ref)).item()
        print(n, k, "plan", cfg.value, spl.value, "relerr", err, flush=True)
        for c in (1, 7, 8):
            for s in (1, 4):
                lib.chfsi_gemm_override(c, s)
                C.zero_(); eng.zgemm("N", "N", n, k, n, 1.0, A, Y, 0.0, C)
                e = (torch.linalg.norm(C - ref) / torch.linalg.norm(ref)).item()
                if e > 1e-12: print("   BAD cfg", c, "split", s, e, flush=True)
        lib.chfsi_gemm_override(-1, 0)
