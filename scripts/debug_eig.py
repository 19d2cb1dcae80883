import sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D
import oracle.chfsi_oracle as O
eng = D.Engine.get(torch.device("cuda", 0)); dev = eng.device
n, m = 20000, 25
rng = np.random.default_rng(7)
lam = np.sort(np.concatenate([rng.uniform(-1.0, 0.0, n // 5), 10.0 ** rng.uniform(0.0, 2.0, n - n // 5)]))
g = torch.Generator(device=dev); g.manual_seed(7)
q, _ = torch.linalg.qr(torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g))
print("orth", torch.linalg.norm(q[:, :8].conj().T @ q[:, :8] - torch.eye(8, device=dev, dtype=q.dtype)).item())
lt = torch.as_tensor(lam, dtype=torch.complex128, device=dev)
h = (q * lt) @ q.conj().T
cols = [0, 1, 1999, 2000, 2199, n - 1]
qc = q[:, cols]
print("eig resid (torch)", [torch.linalg.norm(h @ qc[:, r] - lam[cols[r]] * qc[:, r]).item() for r in range(6)])
hb = ((h + h.conj().T) / 2).conj().contiguous()
del h
y = qc.T.contiguous()
hy = torch.zeros_like(y)
eng.zgemm("N", "N", n, 6, n, 1.0, hb, y, 0.0, hy)
print("eig resid (ours)", [torch.linalg.norm(hy[r] - lam[cols[r]] * y[r]).item() for r in range(6)])
a, b, lr = float(lam[2000]), float(lam[-1]) * 1.01, float(lam[0])
for deg in (1, 2, 5, 25):
    w = torch.empty_like(y)
    out = eng.filter(hb, y.clone(), w, deg, a, b, lr)
    gain = O.filter_gain(deg, lam[cols], a, b, lr)
    errs = [torch.linalg.norm(out[r] - float(gain[r]) * y[r]).item() for r in range(6)]
    print("deg", deg, "gain", np.array2string(gain, precision=3), "errs", np.array2string(np.array(errs), precision=2))
