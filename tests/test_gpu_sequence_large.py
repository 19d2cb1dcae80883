"""Generalized reuse sequences at BASELINE sizes (c2: n = 5000, c3: n = 10000) beyond
problem 1: every problem's eigenvalues against an independent dense eigensolver of
the explicitly reduced problem (test-only: torch.linalg.cholesky / solve_triangular /
eigvalsh, i.e. cuSOLVER through torch -- not this repo's kernels), plus generalized
residuals and B-orthonormality (north_star: eigenvalues within 1e-10 relative,
residuals below tol, the same number of converged pairs).

The reference's own CPU run of these sequences would take 10+ hours, so problem 1
of c2 is pinned against the reference itself (tests/test_golden_full.py) and the
later problems against this dense oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sequence(n, problems, seed):
    """BASELINE c2-c4 recipe on the GPU (workloads.spectrum_matrix_torch for A_1,
    S = I + 0.1 B^H B / ||B^H B||, A_{l+1} = A_l + 1e-3 ||A_1|| E_l)."""
    import torch
    from paper_1305_5120_b200 import device as D
    from paper_1305_5120_b200.workloads import spectrum_matrix_torch
    dev = torch.device("cuda", 0)
    eng = D.Engine.get(dev)
    a, lam = spectrum_matrix_torch(seed, n, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(seed + 1)
    b = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
    s = torch.empty_like(b)
    eng.zgemm("C", "N", n, n, n, 1.0, b, b, 0.0, s)
    del b
    eng.hermitize(s)
    s.mul_(0.1 / float(torch.linalg.eigvalsh(s.T.conj())[-1]))
    s.diagonal().add_(1.0)
    delta = 1e-3 * max(abs(lam[0]), abs(lam[-1]))
    mats = [a]
    for ell in range(1, problems):
        g.manual_seed(seed + 100 + ell)
        e = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
        e = ((e + e.conj().T) / 2).conj().resolve_conj().contiguous()
        w = torch.linalg.eigvalsh(e.T)
        e.mul_(delta / float(torch.max(w.abs())))
        mats.append(mats[-1] + e)
    return mats, s


def _dense_eigvalsh(a_blk, s_blk, nev):
    """lambda(A, S) by explicit reduction L^-1 A L^-H (torch/cuSOLVER, test oracle)."""
    import torch
    # (cols, rows) blocks: row j = column j, i.e. the tensor is A^T = conj(A)
    A = a_blk.T
    S = s_blk.T
    L = torch.linalg.cholesky(S)
    X = torch.linalg.solve_triangular(L, A, upper=False)
    H = torch.linalg.solve_triangular(L, X.conj().T, upper=False).conj().T
    H = (H + H.conj().T) / 2
    return torch.linalg.eigvalsh(H)[:nev].cpu().numpy()


def _check(mats, s, rep, cfg, nev):
    import torch
    from paper_1305_5120_b200 import device as D
    eng = D.Engine.get(torch.device("cuda", 0))
    for i, a in enumerate(mats):
        lam = rep.eigenvalues[i]
        assert len(lam) == nev
        ref = _dense_eigvalsh(a, s, nev)
        assert np.max(np.abs(lam - ref) / np.abs(ref)) <= 1e-10, i
        vb = rep.vectors[i].device_block()
        n, k = vb.shape[1], vb.shape[0]
        av, sv = torch.empty_like(vb), torch.empty_like(vb)
        eng.zgemm("N", "N", n, k, n, 1.0, a, vb, 0.0, av)
        eng.zgemm("N", "N", n, k, n, 1.0, s, vb, 0.0, sv)
        lt = torch.as_tensor(lam, device=vb.device).to(vb.dtype)
        res = torch.linalg.vector_norm(av - sv * lt[:, None], dim=1)
        norm1 = float(torch.linalg.matrix_norm(a.T, ord=1) + torch.linalg.matrix_norm(s.T, ord=1))
        assert float(res.max()) <= cfg.tol * norm1, i
        gram = torch.empty((k, k), dtype=vb.dtype, device=vb.device)
        eng.zgemm("C", "N", k, k, n, 1.0, vb, sv, 0.0, gram)
        eye = torch.eye(k, dtype=vb.dtype, device=vb.device)
        assert float(torch.linalg.matrix_norm(gram - eye)) <= 1e-9, i


def _solve(mats, s, cfg, nev, seed):
    import paper_1305_5120_b200 as G
    smat = G.HermitianDenseMatrix.from_device(s, trusted=True)
    seq = G.ProblemSequence(
        spec=G.SequenceSpec(n=mats[0].shape[0], N=len(mats), nev=nev, seed=seed,
                            kind="generalized"),
        problems=[(G.HermitianDenseMatrix.from_device(a, trusted=True), smat) for a in mats])
    return G.solve_sequence(seq, cfg, "reuse", angles=False)


def test_c2_generalized_sequence_reference_semantics_vs_dense():
    """BASELINE c2 (n = 5000, nev = 500, nex = 50, m = 20), 3 problems with reuse and the
    reference's own interval placement."""
    import paper_1305_5120_b200 as G
    mats, s = _sequence(5000, 3, seed=20)
    cfg = G.SolverConfig(nev=500, buffer=50, degree=20, max_outer_iters=20000)
    rep = _solve(mats, s, cfg, 500, seed=20)
    _check(mats, s, rep, cfg, 500)


def test_c3_generalized_sequence_block_top_vs_dense():
    """BASELINE c3 (n = 10000, nev = 1000, nex = 100, m = 25), 2 problems with reuse,
    opt-in block_top interval."""
    import paper_1305_5120_b200 as G
    mats, s = _sequence(10000, 2, seed=30)
    cfg = G.SolverConfig(nev=1000, buffer=100, degree=25, max_outer_iters=2000,
                         interval="block_top")
    rep = _solve(mats, s, cfg, 1000, seed=30)
    _check(mats, s, rep, cfg, 1000)
