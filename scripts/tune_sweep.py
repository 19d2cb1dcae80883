"""Measure the fused filter step (op N x N, EPI_FILTER) for every tile config x split-K
factor over the solve sizes of BASELINE configs 0-4; the data the GEMM cost model in
csrc/zgemm.cu is fitted to (scripts/fit_cost_model.py).

    python scripts/tune_sweep.py > gpurun_out/sweep.log   # writes gpurun_out/sweep.json
    SWEEP_MODE=gemm python scripts/tune_sweep.py          # solver GEMM shapes -> sweep_gemm.json

The gemm mode times the other products of one outer iteration: Gram Q^H Q (op C N,
M = N = k, K = n), Z = Q W (N N, K = k), the locked projections L^H F (C N, K = n) and
F - L C (N N, K = nl).
"""
import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import _native, device as D  # noqa: E402

SIZES = {
    1000: [8, 24, 60, 120],
    2000: [16, 48, 120, 240],
    5000: [26, 60, 150, 300, 550],
    10000: [26, 70, 140, 300, 600, 1100],
    20000: [26, 64, 140, 210, 275, 560, 1100, 2200],
}
SPLITS = [1, 2, 3, 4, 6, 8, 12, 16]
NCFG = 11

dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
lib = _native.load()
g = torch.Generator(device=dev)
g.manual_seed(0)
out = []
t_start = time.time()
only = [int(x) for x in os.environ.get("SWEEP_N", "").split(",") if x]


def gemm_sweep():
    shapes = []  # (opa, opb, M, N, K)
    for n in (1000, 5000, 20000):
        for k in (24, 120, 240, 550, 1100, 2200):
            if k > n // 2:
                continue
            shapes.append(("C", "N", k, k, n))    # Gram
            shapes.append(("N", "N", n, k, k))    # Q W
        for nl, k in ((n // 10, 40), (n // 10, 220), (n // 20, n // 10 + n // 100)):
            shapes.append(("C", "N", nl, k, n))   # L^H F
            shapes.append(("N", "N", n, k, nl))   # F - L C
    res = []
    for opa, opb, M, N, K in shapes:
        A = torch.randn((K, M) if opa == "N" else (M, K), dtype=torch.complex128, device=dev)
        B = torch.randn((N, K), dtype=torch.complex128, device=dev)
        C = torch.empty((N, M), dtype=torch.complex128, device=dev)
        flops = 8.0 * M * N * K
        reps = int(max(3, min(50, 4e-3 * 30e12 / flops)))

        def timed():
            eng.zgemm(opa, opb, M, N, K, 1.0, A, B, 0.0, C)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                eng.zgemm(opa, opb, M, N, K, 1.0, A, B, 0.0, C)
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps

        cfg, spl = ctypes.c_int(), ctypes.c_int()
        lib.chfsi_gemm_override(-1, 0)
        lib.chfsi_gemm_plan(eng.h, 0 if opa == "N" else 1, 0, 0, M, N, K, ctypes.byref(cfg),
                            ctypes.byref(spl))
        auto_ms = timed()
        res.append({"op": opa + opb, "M": M, "N": N, "K": K, "cfg": -1, "split": 0,
                    "ms": auto_ms, "plan": [cfg.value, spl.value]})
        best = (1e9, None)
        for c in range(NCFG if opa == "N" else 7):
            for s in [1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64]:
                if (K // 8) // s < 4:
                    continue
                lib.chfsi_gemm_override(c, s)
                ms = timed()
                res.append({"op": opa + opb, "M": M, "N": N, "K": K, "cfg": c, "split": s,
                            "ms": ms})
                best = min(best, (ms, (c, s)))
        lib.chfsi_gemm_override(-1, 0)
        print(f"{opa}{opb} M={M} N={N} K={K}: auto {flops / auto_ms / 1e9:.2f} TF plan "
              f"{cfg.value},{spl.value}; best {flops / best[0] / 1e9:.2f} TF {best[1]}  "
              f"[{time.time() - t_start:.0f}s]", flush=True)
        del A, B, C
    json.dump(res, open("gpurun_out/sweep_gemm.json", "w"))


if os.environ.get("SWEEP_MODE") == "gemm":
    gemm_sweep()
    sys.exit(0)

for n, widths in SIZES.items():
    if only and n not in only:
        continue
    H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
    for k in widths:
        Y1 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
        Y0 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
        flops = 8.0 * n * n * k
        reps = int(max(3, min(50, 4e-3 * 30e12 / flops)))

        def timed():
            eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, Y0)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, Y0)
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps

        cfg, spl = ctypes.c_int(), ctypes.c_int()
        lib.chfsi_gemm_override(-1, 0)
        lib.chfsi_gemm_plan(eng.h, 0, 0, 1, n, k, n, ctypes.byref(cfg), ctypes.byref(spl))
        auto_ms = timed()
        out.append({"n": n, "k": k, "cfg": -1, "split": 0, "ms": auto_ms,
                    "plan": [cfg.value, spl.value]})
        best = (1e9, None)
        for c in range(NCFG):
            for s in SPLITS:
                if s > 1 and (n // 8) // s < 4:
                    continue
                if k >= 1000 and s > 2:
                    continue
                lib.chfsi_gemm_override(c, s)
                ms = timed()
                out.append({"n": n, "k": k, "cfg": c, "split": s, "ms": ms})
                best = min(best, (ms, (c, s)))
        lib.chfsi_gemm_override(-1, 0)
        print(f"n={n} k={k}: auto {flops / auto_ms / 1e9:.2f} TF plan {cfg.value},{spl.value}; "
              f"best {flops / best[0] / 1e9:.2f} TF {best[1]}  [{time.time() - t_start:.0f}s]",
              flush=True)
        del Y1, Y0
    del H
    torch.cuda.empty_cache()
    json.dump(out, open("gpurun_out/sweep.json", "w"))
json.dump(out, open("gpurun_out/sweep.json", "w"))
