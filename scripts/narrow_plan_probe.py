"""Sustained degree-25 filter calls at a narrow shard width (default k = 26, the 8-GPU
tail shard of the reference-interval c4 solve) for several forced plans
(chfsi_gemm_override cfg x split-K), with nvidia-smi SM clocks sampled during each.

    python scripts/narrow_plan_probe.py [k] > out.json
"""
import json
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1305_5120_b200 import _native, device as D  # noqa: E402
from paper_1305_5120_b200 import workloads as Wl  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 26
n = int(os.environ.get("N_ORDER", "20000"))
dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
lib = _native.load()
H, lam = Wl.spectrum_matrix_torch(0, n, dev)
g = torch.Generator(device=dev)
g.manual_seed(1)
eng.declare_operator(H)
a, b, lr = float(lam[n // 10]), 1.01 * float(lam[-1]), float(lam[0])
Y0 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
Y, W = Y0.clone(), torch.empty_like(Y0)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
rows = []
plans = [(-1, 0)] + [(c, s) for c in (14, 15, 16) for s in (4, 8, 12, 16, 24)]
if os.environ.get("PLANS"):  # "cfg:split,cfg:split,..."
    plans = [tuple(int(v) for v in x.split(":")) for x in os.environ["PLANS"].split(",")]
for cfg, split in plans:
    lib.chfsi_gemm_override(cfg, split)
    eng.filter(H, Y.copy_(Y0), W, 25, a, b, lr)
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                            "--format=csv,noheader,nounits", "-lms", "100"],
                           stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    ev[0].record()
    calls = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 3.0:
        Y.copy_(Y0)
        eng.filter(H, Y, W, 25, a, b, lr)
        calls += 1
        torch.cuda.synchronize()
    ev[1].record()
    torch.cuda.synchronize()
    smi.terminate()
    lines = [ln.split(",") for ln in smi.communicate()[0].strip().splitlines() if "," in ln]
    clk = sorted(float(x[0]) for x in lines)
    pw = sorted(float(x[1]) for x in lines)
    ms = ev[0].elapsed_time(ev[1]) / (calls * 25)
    rows.append({"cfg": cfg, "split": split, "ms_per_step": ms,
                 "sm_mhz_median": clk[len(clk) // 2] if clk else None,
                 "power_w_median": pw[len(pw) // 2] if pw else None})
    print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
lib.chfsi_gemm_override(-1, 0)
eng.declare_operator(None)
print(json.dumps({"k": k, "n": n, "rows": rows}))
