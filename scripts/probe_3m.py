"""3M vs 4M complex products in the fused filter step on the GPU.

    python scripts/probe_3m.py [n] [widths] > gpurun_out/probe_3m.json

For each width k: TFLOP/s (conventional 8 n^2 k flop per step) of the TMA configs
with four real products (cfg 7, 10) and with 3M (cfg 11, 12) over split-K factors,
the cost model's pick in each mode, and the deviation of the 3M result from the 4M
result and from torch (cuBLAS ZGEMM) relative to ||H|| ||Y1||.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import _native, device as D  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
widths = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else \
    [26, 64, 210, 275, 1100, 2200]
dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
lib = _native.load()
g = torch.Generator(device=dev)
g.manual_seed(0)
H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
H = (H + H.mH) * 0.5
hn = float(torch.linalg.matrix_norm(H, ord=2)) if n <= 4096 else float(torch.linalg.norm(H))


def timed(reps, fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


out = {"n": n, "widths": {}}
for k in widths:
    Y1 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
    Y0 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
    C = torch.empty_like(Y0)
    reps = max(1, min(10, int(3e12 / (8.0 * n * n * k))))
    row = {}
    splits = (1, 2, 3, 4, 6, 8, 12, 17) if k <= 300 else (1, 2) if k <= 1200 else (1,)
    for c in (7, 10, 11, 12, 13):
        for s in splits:
            lib.chfsi_gemm_override(c, s)
            ms = timed(reps, lambda: eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, C))
            row[f"c{c}s{s}"] = round(8.0 * n * n * k / ms / 1e9, 2)
    lib.chfsi_gemm_override(-1, 0)
    for mul in (4, 3):
        lib.chfsi_set_complex_mul(mul)
        ms = timed(reps, lambda: eng.filter_step(H, Y1, 0.5, -0.1, Y0, 0.2, C))
        row[f"auto{mul}"] = round(8.0 * n * n * k / ms / 1e9, 2)
    # accuracy: plain product (alpha = 1, beta = gamma = 0)
    C4 = torch.empty_like(C)
    C3 = torch.empty_like(C)
    lib.chfsi_set_complex_mul(4)
    eng.filter_step(H, Y1, 1.0, 0.0, None, 0.0, C4)
    lib.chfsi_set_complex_mul(3)
    eng.filter_step(H, Y1, 1.0, 0.0, None, 0.0, C3)
    ref = Y1 @ H  # tensor rows are columns: C^T = Y^T H^T, and H is stored as H^T
    scale = float(torch.linalg.norm(H)) * float(torch.linalg.norm(Y1))
    colscale = torch.linalg.norm(Y1, dim=1) * float(torch.linalg.norm(H))
    row["err_3m_vs_ref"] = float(torch.linalg.norm(C3 - ref)) / scale
    row["err_4m_vs_ref"] = float(torch.linalg.norm(C4 - ref)) / scale
    row["maxabs_3m_vs_ref_rel_col"] = float(((C3 - ref).abs().amax(dim=1) / colscale).max())
    row["maxabs_4m_vs_ref_rel_col"] = float(((C4 - ref).abs().amax(dim=1) / colscale).max())
    best4 = max((v, kk) for kk, v in row.items() if kk[:3] in ("c7s", "c10"))
    best3 = max((v, kk) for kk, v in row.items() if kk[:3] in ("c11", "c12", "c13"))
    row["best4"], row["best3"] = best4, best3
    print(json.dumps({"k": k, **{x: row[x] for x in ("auto4", "auto3", "best4", "best3",
                                                      "err_3m_vs_ref", "err_4m_vs_ref")}}),
          file=sys.stderr, flush=True)
    out["widths"][k] = row
    del Y1, Y0, C, C3, C4, ref
print(json.dumps(out, indent=1))
