"""Bandwidth-bound kernels at c4 sizes for ncu (n = 20000): residual norms, column dots,
Hermitian norms / symmetrise, and the tail CholQR Gram / CGS2 projection (k = 210,
2000 locked)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1305_5120_b200 import device as D

dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
n = 20000
g = torch.Generator(device=dev)
g.manual_seed(0)
for k in (210, 2200):
    hz = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
    z = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
    lam = np.linspace(-1, 1, k)
    for _ in range(3):
        eng.residual_norms(hz, z, lam)
    out = torch.empty((k,), dtype=torch.complex128, device=dev)
    del hz, z
a = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
for _ in range(2):
    eng.hermitian_norms(a)
    eng.hermitize(a)
del a
# tail QR pieces: F (210 cols) against L (2000 locked)
f = torch.randn((210, n), dtype=torch.complex128, device=dev, generator=g)
L = torch.linalg.qr(torch.randn((n, 2000), dtype=torch.complex128, device=dev, generator=g))[0]
L = L.T.conj().resolve_conj().contiguous().conj().resolve_conj()  # (2000, n) column-major block
t = torch.empty_like(f)
q = torch.empty_like(f)
for _ in range(2):
    eng.project_out(f, L)
    eng.orthonormalize(f, None, t, q)
torch.cuda.synchronize()
print("bw workload done")
