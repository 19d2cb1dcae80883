"""Sweep the DMMA GEMM tile configs over filter widths on the GPU.

    python scripts/tune_gemm.py [n] > gpurun_out/tune.txt
Prints TFLOP/s of the fused filter step per (width, config, split) and the plan the
cost model picks.
"""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import _native, device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
widths = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else \
    [16, 26, 32, 48, 64, 96, 128, 210, 275, 512, 1100, 2200]
dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
lib = _native.load()
g = torch.Generator(device=dev)
g.manual_seed(0)
H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
res = {}
for k in widths:
    Y1 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
    Y0 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
    cfg, spl = ctypes.c_int(), ctypes.c_int()
    lib.chfsi_gemm_override(-1, 0)
    lib.chfsi_gemm_plan(eng.h, 0, 0, 1, n, k, n, ctypes.byref(cfg), ctypes.byref(spl))
    row = {"plan": [cfg.value, spl.value]}
    reps = max(1, min(10, int(3e12 / (8.0 * n * n * k))))
    for c in range(11):
        for s in ((1, 2, 3, 4) if k <= 300 else (1,)):
            lib.chfsi_gemm_override(c, s)
            eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, Y0)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, Y0)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            row[f"c{c}s{s}"] = round(8.0 * n * n * k / ms / 1e9, 2)
    lib.chfsi_gemm_override(-1, 0)
    eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, Y0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, Y0)
    b.record()
    torch.cuda.synchronize()
    row["auto"] = round(8.0 * n * n * k / (a.elapsed_time(b) / reps) / 1e9, 2)
    best = max((v, kk) for kk, v in row.items() if kk.startswith("c"))
    print(k, "auto", row["auto"], "plan", row["plan"], "best", best, flush=True)
    res[k] = row
    del Y1, Y0
json.dump(res, open("gpurun_out/tune.json", "w"), indent=1)
