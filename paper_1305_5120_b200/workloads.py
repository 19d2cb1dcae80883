"""Seeded synthetic problems with BASELINE.json's recipes.

The reference measures on no public dataset (the paper's FLEUR matrices are
not available), so these generators stand in for it:

  c0  n=1000  standard, lambda: 20 % uniform in [-1, 0], 80 % log-uniform in
      [1, 100]; H = Q diag(lambda) Q^H with Q from QR of a complex Gaussian.
  c1  n=2000  sequence of 5: H_{i+1} = H_i + delta E_i, E_i = (G+G^H)/2 scaled
      to ||E_i||_2 = 1, delta = 1e-3 ||H_1||_2.
  c2-c4       generalized sequences: S = I + 0.1 B^H B / ||B^H B||_2 (one S per
      sequence), A_i built as in c1.

Host generation uses numpy's Generator (the same stream order the reference's
conftest/sequence helpers use); ``spectrum_matrix_torch`` builds the n=20000
c4 matrix on the GPU for the benchmark (data generation only, not the
measured path).
"""

from dataclasses import dataclass

import numpy as np

CONFIGS = {
    # name: (n, nev, nex, degree, n_problems, generalized)
    "c0": (1000, 100, 20, 15, 1, False),
    "c1": (2000, 200, 40, 20, 5, False),
    "c2": (5000, 500, 50, 20, 10, True),
    "c3": (10000, 1000, 100, 25, 10, True),
    "c4": (20000, 2000, 200, 25, 10, True),
}


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    nev: int
    nex: int
    degree: int
    n_problems: int
    generalized: bool
    tol: float = 1e-10

    @property
    def k(self):
        return self.nev + self.nex


def workload(name, n=None):
    n0, nev, nex, m, N, gen = CONFIGS[name]
    if n is not None and n != n0:
        scale = n / n0
        nev = max(1, int(round(nev * scale)))
        nex = max(1, int(round(nex * scale)))
        n0 = n
    return Workload(name, n0, nev, nex, m, N, gen)


def baseline_spectrum(rng, n):
    """Lowest 20 % uniform in [-1, 0], the rest log-uniform in [1, 100], sorted."""
    n_lo = n // 5
    lo = rng.uniform(-1.0, 0.0, n_lo)
    hi = 10.0 ** rng.uniform(0.0, 2.0, n - n_lo)
    return np.sort(np.concatenate([lo, hi]))


def complex_gaussian(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def spectrum_matrix(rng, evals):
    """Hermitian matrix with exactly the given eigenvalues, H = Q diag Q^H (host)."""
    evals = np.asarray(evals, dtype=np.float64)
    n = evals.size
    q, _ = np.linalg.qr(complex_gaussian(rng, (n, n)))
    h = (q * evals) @ q.conj().T
    h = (h + h.conj().T) / 2.0
    return np.asfortranarray(h), q


def baseline_matrix(seed, n):
    """c0 recipe: returns (H F-order, exact eigenvalues ascending, exact eigenvectors)."""
    rng = np.random.default_rng(seed)
    lam = baseline_spectrum(rng, n)
    h, q = spectrum_matrix(rng, lam)
    return h, lam, q


def unit_hermitian_perturbation(rng, n):
    """E = (G + G^H)/2 rescaled to ||E||_2 = 1."""
    g = complex_gaussian(rng, (n, n))
    e = (g + g.conj().T) / 2.0
    w = np.linalg.eigvalsh(e)
    return e / max(abs(w[0]), abs(w[-1]))


def spd_metric(rng, n):
    """S = I + 0.1 B^H B / ||B^H B||_2 (cond(S) <= 1.1)."""
    b = complex_gaussian(rng, (n, n))
    bhb = b.conj().T @ b
    bhb = (bhb + bhb.conj().T) / 2.0
    top = np.linalg.eigvalsh(bhb)[-1]
    s = np.eye(n, dtype=np.complex128) + 0.1 * bhb / top
    return np.asfortranarray((s + s.conj().T) / 2.0)


def baseline_sequence(seed, n, n_problems, generalized=False, rel_delta=1e-3):
    """List of (A, S or None) following BASELINE configs c1-c4 (host numpy)."""
    rng = np.random.default_rng(seed)
    lam = baseline_spectrum(rng, n)
    a, _ = spectrum_matrix(rng, lam)
    delta = rel_delta * max(abs(lam[0]), abs(lam[-1]))
    s = spd_metric(rng, n) if generalized else None
    out = [(a, s)]
    for _ in range(1, n_problems):
        a = a + delta * unit_hermitian_perturbation(rng, n)
        a = np.asfortranarray((a + a.conj().T) / 2.0)
        out.append((a, s))
    return out


def spectrum_matrix_torch(seed, n, device):
    """GPU construction of the c0-recipe matrix at large n (c4: n=20000).

    Returns (H as a column-major block: torch (n, n) complex128 whose row j is
    column j of H, exact eigenvalues as numpy). Uses torch (cuSOLVER QR,
    cuBLAS matmul) purely to synthesise test data.
    """
    import torch

    rng = np.random.default_rng(seed)
    lam = baseline_spectrum(rng, n)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    z = torch.randn((n, n), dtype=torch.complex128, device=device, generator=g)
    q, _ = torch.linalg.qr(z)
    del z
    lt = torch.as_tensor(lam, dtype=torch.float64, device=device).to(torch.complex128)
    h = (q * lt) @ q.conj().T
    del q
    h = (h + h.conj().T) / 2
    # h is Hermitian: its row-major storage is conj(H) column-major; store H^T = conj(H)
    # rows so that row j of the tensor is column j of H. (conj() is a lazy view in
    # torch: resolve_conj() writes the conjugated values to memory.)
    hc = h.conj().resolve_conj().contiguous()
    del h
    return hc, lam
