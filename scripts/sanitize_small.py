"""Small end-to-end workload for `compute-sanitizer --tool memcheck`: every GEMM
config/split on ragged shapes (TMA zero-fill edges), the 3M sum-plane filter configs
(forced, every split, ragged widths, padded leading dims, declared operator, the width
rule at n = 8192), the fused filter, CholQR2 with locked vectors, Rayleigh-Ritz, a small
solve and a generalized solve."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1305_5120_b200 as G  # noqa: E402
from paper_1305_5120_b200 import _native, device as D  # noqa: E402

eng = D.Engine.get(torch.device("cuda", 0))
lib = _native.load()
rng = np.random.default_rng(0)


def crand(*s):
    return rng.standard_normal(s) + 1j * rng.standard_normal(s)


for cfg in range(14):
    for split in (1, 2):
        lib.chfsi_gemm_override(cfg, split)
        for (m, n, k) in [(13, 5, 27), (70, 33, 9)]:
            ops = [("N", "N")] if cfg >= 7 else [("N", "N"), ("C", "N"), ("N", "C")]
            for opa, opb in ops:
                A = crand(m, k) if opa == "N" else crand(k, m)
                B = crand(k, n) if opb == "N" else crand(n, k)
                C = D.to_device(crand(m, n), eng.device)
                eng.zgemm(opa, opb, m, n, k, 1.0, D.to_device(A, eng.device),
                          D.to_device(B, eng.device), 0.5, C)
lib.chfsi_gemm_override(-1, 0)
# sum-plane filter configs (n % 8 == 0), ragged widths, forced splits
for cfg in (14, 15, 16, 17, 18, -1):  # 17 / 18: the B-sum-only kernels
    for split in (1, 3, 0):
        lib.chfsi_gemm_override(cfg, split)
        for (n, k) in [(136, 5), (64, 37), (200, 26)]:
            hh = crand(n, n)
            hh = (hh + hh.conj().T) / 2
            dH = D.to_device(hh, eng.device)
            eng.filter(dH, D.to_device(crand(n, k), eng.device), D.zeros(n, k, eng.device), 3,
                       -1.0, 1.0, -2.0)
lib.chfsi_gemm_override(-1, 0)
# padded leading dims + declared operator + apply_operator
Hbuf = torch.randn((96, 120), dtype=torch.complex128, device=eng.device)
Hv = Hbuf[:, :96]
Ybuf = torch.randn((20, 104), dtype=torch.complex128, device=eng.device)
eng.declare_operator(Hv)
eng.filter(Hv, Ybuf[:, :96], torch.empty((20, 96), dtype=torch.complex128, device=eng.device),
           4, -1.0, 1.0, -2.0)
eng.apply_operator(Hv, Ybuf[:, :96], torch.empty((20, 96), dtype=torch.complex128,
                                                  device=eng.device))
eng.declare_operator(None)
# the width rule (M >= 8192) on a narrow block
Hbig = torch.randn((8192, 8192), dtype=torch.complex128, device=eng.device)
eng.filter(Hbig, torch.randn((26, 8192), dtype=torch.complex128, device=eng.device),
           torch.empty((26, 8192), dtype=torch.complex128, device=eng.device), 2, -1.0, 1.0, -2.0)
# round 2: the narrow rule's B-sum-only kernels (17-64 columns: one and two tiles, 24-
# and 32-wide) and a block just past the rule
for kk in (20, 40, 51, 70):
    eng.filter(Hbig, torch.randn((kk, 8192), dtype=torch.complex128, device=eng.device),
               torch.empty((kk, 8192), dtype=torch.complex128, device=eng.device), 2, -1.0, 1.0,
               -2.0)
del Hbig
# round 2: the HBM-bound GEMV (N = 1) with a padded leading dimension, and the Lanczos bound
Abuf = torch.randn((300, 310), dtype=torch.complex128, device=eng.device)
x = torch.randn((1, 300), dtype=torch.complex128, device=eng.device)
y = torch.randn((1, 300), dtype=torch.complex128, device=eng.device)
eng.zgemm("N", "N", 300, 1, 300, 0.5 + 0.1j, Abuf[:, :300], x, -0.2, y)
hl = (Abuf[:, :300] + Abuf[:, :300].T.conj()).resolve_conj().contiguous()
eng.lanczos_bound(hl, x[0], 10)
# round 2: triangular operand at an unaligned offset with a forced split (element-masked)
lib.chfsi_gemm_override(-1, 3)
L = torch.tril(torch.randn((64, 64), dtype=torch.complex128, device=eng.device)).T.contiguous()
eng.zgemm("N", "N", 20, 17, 64, 1.0, torch.randn((64, 20), dtype=torch.complex128,
                                                  device=eng.device),
          L[3:20], 0.0, torch.empty((17, 20), dtype=torch.complex128, device=eng.device),
          tri=eng.TRI_B_LOWER, tri_offset=3)
lib.chfsi_gemm_override(-1, 0)
# round 2: pageable upload through the staging ring (> 8 MB, several chunks)
big = np.asfortranarray(crand(3000, 400))
t = D.to_device(big, eng.device)
assert np.array_equal(D.to_host(t), big)
from paper_1305_5120_b200.workloads import baseline_matrix  # noqa: E402
h, lam, _ = baseline_matrix(1, 120)
lam_g, v, rep = G.chfsi_solve(h, None, G.SolverConfig(nev=10, buffer=6, degree=12,
                                                      max_outer_iters=5000,
                                                      interval="block_top"), seed=1)
a = crand(40, 40)
a = (a + a.conj().T) / 2
b = crand(40, 40)
b = b.conj().T @ b + 40 * np.eye(40)
G.solve_generalized(a, b, None, G.SolverConfig(nev=4), seed=2)
torch.cuda.synchronize()
print("sanitize workload done", rep.outer_iterations)
