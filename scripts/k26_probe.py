"""Filter step time at narrow widths (k = 26, 51, 101, 201; n = 20000) for degree-5 and
degree-25 calls, start blocks of scale 1 and 7e-6, on the c4 matrix and on a random
Hermitian one: the sustained narrow-width slowdown traced to the board power cap
(profiles/r02/narrow_plans.json). python scripts/k26_probe.py"""
import sys, math, json, torch, numpy as np
sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D
from paper_1305_5120_b200 import workloads as Wl
dev = torch.device("cuda", 0); eng = D.Engine.get(dev); n = 20000
g = torch.Generator(device=dev); g.manual_seed(0)
Hc, lam = Wl.spectrum_matrix_torch(0, n, dev)
Hr = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
Hr = ((Hr + Hr.T.conj()) * (0.5 / (3.0 * math.sqrt(n)))).resolve_conj().contiguous()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
def t(H, k, deg, scale, a, b, lr):
    Y0 = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g) * scale
    Y = Y0.clone(); W = torch.empty_like(Y)
    eng.filter(H, Y, W, deg, a, b, lr); torch.cuda.synchronize()
    ev[0].record()
    for _ in range(3):
        Y.copy_(Y0); eng.filter(H, Y, W, deg, a, b, lr)
    ev[1].record(); torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / 3 / deg
out = []
for name, H, a, b, lr in (("c4", Hc, float(lam[2000]), 1.01*float(lam[-1]), float(lam[0])), ("rand", Hr, -1.0, 1.0, -2.0)):
    eng.declare_operator(H)
    for k in (26, 51, 101, 201):
        for deg in (5, 25):
            for scale in (1.0, 1e-3 / math.sqrt(n)):
                out.append({"H": name, "k": k, "deg": deg, "scale": scale, "ms_per_step": t(H, k, deg, scale, a, b, lr)})
                print(json.dumps(out[-1]), flush=True)
    eng.declare_operator(None)
