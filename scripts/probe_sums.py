"""Filter calls with 3M operand-sum planes: per-step TFLOP/s of every sum-reading config
(14, 15) x split-K over filter widths, beside the in-loop-sum 3M configs (11, 12) and the
cost model's pick. H is declared (chfsi_declare_operator), as in a solve.

    python scripts/probe_sums.py [n] [widths] > gpurun_out/probe_sums.json
"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import _native, device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
widths = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else \
    [26, 64, 128, 210, 275, 550, 1100, 2200]
dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
lib = _native.load()
g = torch.Generator(device=dev)
g.manual_seed(0)
H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
eng.declare_operator(H)
DEG = 4


def run(k, Y, W):
    eng.filter(H, Y, W, DEG, -1.0, 1.0, -2.0)
    torch.cuda.synchronize()
    reps = max(1, min(5, int(4e12 / (8.0 * n * n * k * DEG))))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        eng.filter(H, Y, W, DEG, -1.0, 1.0, -2.0)
    b.record()
    torch.cuda.synchronize()
    return 8.0 * n * n * k * DEG / (a.elapsed_time(b) / reps * 1e-3) / 1e12


out = {"n": n, "degree": DEG, "widths": {}}
for k in widths:
    Y = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g) * 1e-3
    W = torch.empty_like(Y)
    row = {}
    splits = (1, 2, 3, 4, 6, 8, 12, 17) if k <= 300 else (1, 2, 3) if k <= 1200 else (1,)
    for c in (tuple(int(x) for x in os.environ["CFGS"].split(",")) if os.environ.get("CFGS") else (14, 15, 16) if os.environ.get("SUMS_ONLY") else (11, 12, 14, 15, 16)):
        for s in splits:
            lib.chfsi_gemm_override(c, s)
            row[f"c{c}s{s}"] = round(run(k, Y, W), 2)
    lib.chfsi_gemm_override(-1, 0)
    row["auto"] = round(run(k, Y, W), 2)
    best = max((v, kk) for kk, v in row.items() if kk.startswith("c"))
    print(json.dumps({"k": k, "auto": row["auto"], "best": best}), file=sys.stderr, flush=True)
    out["widths"][k] = row
eng.declare_operator(None)
print(json.dumps(out, indent=1))
