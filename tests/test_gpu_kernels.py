"""GPU parity of the individual native kernels against the oracle (oracle/chfsi_oracle.py)
and closed forms. Tolerances are relative, FP64 (DMMA accumulation order differs
from OpenBLAS, so 1e-13 instead of bit equality)."""

import numpy as np
import pytest

from conftest import rand_hermitian, rand_spd, spectrum_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import torch
    from paper_1305_5120_b200 import device as D
    return D.Engine.get(torch.device("cuda", 0))


def crand(rng, *s):
    return rng.standard_normal(s) + 1j * rng.standard_normal(s)


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (37, 19, 53), (128, 64, 256), (70, 3, 1000),
                                   (5, 7, 4000), (300, 260, 77), (513, 129, 65), (64, 0, 8),
                                   (16, 16, 0)])
@pytest.mark.parametrize("opa,opb", [("N", "N"), ("C", "N"), ("N", "C"), ("C", "C")])
def test_zgemm_all_ops(eng, m, n, k, opa, opb):
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    A = crand(rng, m, k) if opa == "N" else crand(rng, k, m)
    B = crand(rng, k, n) if opb == "N" else crand(rng, n, k)
    C = crand(rng, m, n)
    al, be = 0.7 - 0.2j, -0.3 + 0.5j
    ref = al * ((A if opa == "N" else A.conj().T) @ (B if opb == "N" else B.conj().T)) + be * C
    dA, dB, dC = D.to_device(A, eng.device), D.to_device(B, eng.device), D.to_device(C, eng.device)
    eng.zgemm(opa, opb, m, n, k, al, dA, dB, be, dC)
    got = D.to_host(dC)
    if ref.size:
        assert np.linalg.norm(got - ref) <= 1e-13 * max(1.0, np.linalg.norm(ref))


def test_zgemm_deterministic_splitk(eng):
    """Gram-shaped product (split-K path) is bit-identical run to run."""
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(3)
    A = crand(rng, 20000, 24)
    dA = D.to_device(A, eng.device)
    outs = []
    for _ in range(3):
        dC = D.zeros(24, 24, eng.device)
        eng.zgemm("C", "N", 24, 24, 20000, 1.0, dA, dA, 0.0, dC)
        outs.append(D.to_host(dC))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])
    ref = A.conj().T @ A
    assert np.linalg.norm(outs[0] - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("m", [1, 2, 5, 20, 50])
def test_filter_matches_scalar_closed_form(eng, m):
    """Diagonal H: p_m(H) e_j = p_m(lam_j) e_j (reference test_filter.py:54-67 idea)."""
    import oracle.chfsi_oracle as O
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(40 + m)
    lam = np.concatenate([np.sort(rng.uniform(0.0, 4.0, 8)), np.sort(rng.uniform(5.0, 10.0, 24))])
    h = np.diag(lam).astype(complex)
    a, b, lam_ref = 4.8, 10.2, float(lam[0])
    dH = D.to_device(h, eng.device)
    dY = D.to_device(np.eye(32, dtype=complex), eng.device)
    dW = D.zeros(32, 32, eng.device)
    out = D.to_host(eng.filter(dH, dY, dW, m, a, b, lam_ref))
    got = np.real(np.diag(out))
    ref = O.filter_gain(m, lam, a, b, lam_ref)
    assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)) <= 1e-12
    assert np.linalg.norm(out - np.diag(np.diag(out))) <= 1e-12 * np.linalg.norm(out)


@pytest.mark.parametrize("n,k,m", [(200, 24, 15), (513, 37, 20), (1000, 120, 25)])
def test_filter_matches_oracle_recurrence(eng, n, k, m):
    import oracle.chfsi_oracle as O
    from paper_1305_5120_b200 import device as D
    from paper_1305_5120_b200.workloads import baseline_matrix
    h, lam, _ = baseline_matrix(n, n)
    rng = np.random.default_rng(n + k)
    y = crand(rng, n, k)
    a, b, lam_ref = float(lam[k]), float(lam[-1]) * 1.05, float(lam[0])
    ref = O.cheb_filter(h, y, m, a, b, lam_ref)
    dH = D.to_device(h, eng.device)
    dY = D.to_device(y, eng.device)
    dW = D.zeros(n, k, eng.device)
    got = D.to_host(eng.filter(dH, dY, dW, m, a, b, lam_ref))
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("n,k,m,panels", [(513, 37, 7, 3), (1000, 120, 12, 0), (1000, 120, 5, 16),
                                          (200, 1, 3, 1)])
def test_filter_streamed_matches_oracle(eng, n, k, m, panels):
    """Host-H filter (upload overlapped with the first degree step, row panels, ragged
    last panel) against the oracle recurrence; H lands on the device unchanged."""
    import oracle.chfsi_oracle as O
    from paper_1305_5120_b200 import device as D
    from paper_1305_5120_b200.workloads import baseline_matrix
    h, lam, _ = baseline_matrix(n, n)
    h = np.asfortranarray(h)
    rng = np.random.default_rng(n + 3 * k)
    y = crand(rng, n, k)
    a, b, lam_ref = float(lam[min(k, n - 1)]), float(lam[-1]) * 1.05, float(lam[0])
    ref = O.cheb_filter(h, y, m, a, b, lam_ref)
    dH = D.empty(n, n, eng.device)
    dY = D.to_device(y, eng.device)
    dW = D.zeros(n, k, eng.device)
    got = D.to_host(eng.filter_streamed(h, dH, dY, dW, m, a, b, lam_ref, panels=panels))
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.array_equal(D.to_host(dH), h)


@pytest.mark.parametrize("n,k,m,panels", [(512, 37, 7, 3), (1000, 120, 1, 4), (1000, 64, 2, 0),
                                          (136, 1, 3, 1)])
def test_filter_streamed_to_host(eng, n, k, m, panels):
    """Host-to-host filter (H streamed in, the last degree step by row panels with each
    panel read back under the next): the host result equals the device result bit for
    bit and the oracle recurrence to rounding; degree 1 reads back the first step's
    panels."""
    import oracle.chfsi_oracle as O
    from paper_1305_5120_b200 import device as D
    from paper_1305_5120_b200.workloads import baseline_matrix
    h, lam, _ = baseline_matrix(n, n)
    h = np.asfortranarray(h)
    rng = np.random.default_rng(n + 5 * k + m)
    y = crand(rng, n, k)
    a, b, lam_ref = float(lam[min(k, n - 1)]), float(lam[-1]) * 1.05, float(lam[0])
    ref = O.cheb_filter(h, y, m, a, b, lam_ref)
    dH = D.empty(n, n, eng.device)
    dev_out, host = eng.filter_streamed_to_host(h, dH, D.to_device(y, eng.device),
                                                D.zeros(n, k, eng.device), m, a, b, lam_ref,
                                                panels=panels)
    assert np.array_equal(host, D.to_host(dev_out))
    assert np.linalg.norm(host - ref) <= 1e-12 * np.linalg.norm(ref)


def test_public_filter_host_operator_to_host(eng):
    """chebyshev_filter(ndarray H >= 4096, ndarray Y) -- the bench's e2e path: entries are
    already on the host when the call returns and match the oracle."""
    import oracle.chfsi_oracle as O
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.workloads import baseline_matrix
    n, k, m = 4096, 24, 3
    h, lam, _ = baseline_matrix(n, n)
    y = crand(np.random.default_rng(8), n, k)
    spec = G.FilterSpec(degree=m, a=float(lam[k]), b=float(lam[-1]) * 1.05, lam_ref=float(lam[0]))
    out = G.chebyshev_filter(np.asfortranarray(h), y, spec)
    assert out._host is not None
    ref = O.cheb_filter(h, y, m, spec.a, spec.b, spec.lam_ref)
    assert np.linalg.norm(out.entries - ref) <= 1e-12 * np.linalg.norm(ref)


def test_filter_streamed_bit_identical_without_split(eng):
    """With split-K off, every panel step sums each output over K in the order of the
    full-height step: the streamed filter equals the resident one bit for bit."""
    from paper_1305_5120_b200 import _native
    from paper_1305_5120_b200 import device as D
    from paper_1305_5120_b200.workloads import baseline_matrix
    n, k, m = 1536, 96, 6
    h, lam, _ = baseline_matrix(n, n)
    h = np.asfortranarray(h)
    y = crand(np.random.default_rng(5), n, k)
    a, b, lam_ref = float(lam[k]), float(lam[-1]) * 1.05, float(lam[0])
    lib = _native.load()
    assert lib.chfsi_gemm_override(-1, 1) == 0
    try:
        dH = D.to_device(h, eng.device)
        full = D.to_host(eng.filter(dH, D.to_device(y, eng.device), D.zeros(n, k, eng.device),
                                    m, a, b, lam_ref))
        dH2 = D.empty(n, n, eng.device)
        got = D.to_host(eng.filter_streamed(h, dH2, D.to_device(y, eng.device),
                                            D.zeros(n, k, eng.device), m, a, b, lam_ref, panels=4))
    finally:
        lib.chfsi_gemm_override(-1, 0)
    assert np.array_equal(got, full)


def test_chebyshev_filter_host_path_streams(eng, monkeypatch):
    """The public chebyshev_filter(ndarray H, ...) takes the streamed path above the size
    threshold and returns the same block as with H already wrapped on the device."""
    import paper_1305_5120_b200 as G
    import paper_1305_5120_b200.core as C
    from paper_1305_5120_b200.workloads import baseline_matrix
    n, k = 700, 40
    h, lam, _ = baseline_matrix(n, n)
    y = crand(np.random.default_rng(8), n, k)
    spec = G.FilterSpec(degree=9, a=float(lam[k]), b=float(lam[-1]) * 1.05, lam_ref=float(lam[0]))
    monkeypatch.setattr(C, "_STREAM_MIN_N", 512)
    calls = []
    orig = C._filter_streamed
    monkeypatch.setattr(C, "_filter_streamed", lambda *a: calls.append(1) or orig(*a))
    got = G.chebyshev_filter(h, y, spec).entries
    assert calls == [1]
    ref = G.chebyshev_filter(G.HermitianDenseMatrix(h), y, spec).entries
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    with pytest.raises(G.ContractViolation):
        G.chebyshev_filter(h, y[:-1], spec)


def test_lanczos_bound_matches_oracle(eng):
    import oracle.chfsi_oracle as O
    import paper_1305_5120_b200 as G
    rng = np.random.default_rng(30)
    h = rand_hermitian(rng, 100, scale=2.0)
    lam_max = np.linalg.eigvalsh(h)[-1]
    for seed in range(10):
        got = G.lanczos_upper_bound(h, 10, seed=seed)
        ref, _ = O.lanczos_bound(h, 10, np.random.default_rng(seed))
        assert abs(got - ref) <= 1e-10 * abs(ref)
        assert got >= lam_max


def test_lanczos_breakdown_and_clipping():
    import paper_1305_5120_b200 as G
    b = G.lanczos_upper_bound(3.0 * np.eye(12, dtype=complex), 10, seed=0)
    assert 3.0 <= b <= 3.0 + 1e-10
    b = G.lanczos_upper_bound(np.diag(np.arange(1.0, 11.0)).astype(complex), 10, seed=1)
    assert 10.0 <= b <= 10.0 + 1e-6
    assert G.lanczos_upper_bound(np.diag([1.0, 2, 3, 4, 5]).astype(complex), 10, seed=2) >= 5.0


def test_residual_norms_match_numpy(eng):
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(59)
    n, k = 777, 13
    hy, y = crand(rng, n, k), crand(rng, n, k)
    lam = rng.uniform(-1, 1, k)
    got = eng.residual_norms(D.to_device(hy, eng.device), D.to_device(y, eng.device), lam)
    ref = np.linalg.norm(hy - y * lam, axis=0)
    assert np.max(np.abs(got - ref) / ref) <= 1e-14


@pytest.mark.parametrize("n,k,nl", [(300, 20, 0), (300, 20, 15), (5000, 64, 100), (1000, 250, 40)])
def test_orthonormalize_cgs2_cholqr2(eng, n, k, nl):
    import torch
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(n + k + nl)
    L = np.linalg.qr(crand(rng, n, nl))[0] if nl else None
    F = crand(rng, n, k) * np.logspace(0, 6, k)  # graded columns
    dF = D.to_device(F, eng.device)
    dL = D.to_device(L, eng.device) if nl else None
    dT, dQ = D.zeros(n, k, eng.device), D.zeros(n, k, eng.device)
    eng.orthonormalize(dF, dL, dT, dQ)
    Q = D.to_host(dQ)
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(k)) <= 1e-12 * np.sqrt(k)
    W = F - L @ (L.conj().T @ F) if nl else F
    if nl:
        assert np.linalg.norm(L.conj().T @ Q) <= 1e-12
    # same span as the projected block
    qw = np.linalg.qr(W)[0]
    assert np.linalg.norm(qw - Q @ (Q.conj().T @ qw)) <= 1e-9


def test_orthonormalize_rank_collapse_reports_column(eng):
    from paper_1305_5120_b200 import device as D
    from paper_1305_5120_b200.errors import RankDeficient
    rng = np.random.default_rng(13)
    F = crand(rng, 50, 4)
    F[:, 2] = F[:, 0]
    dF = D.to_device(F, eng.device)
    with pytest.raises(RankDeficient) as exc:
        eng.orthonormalize(dF, None, D.zeros(50, 4, eng.device), D.zeros(50, 4, eng.device))
    assert exc.value.column == 2


def test_rayleigh_ritz_matches_oracle(eng):
    import oracle.chfsi_oracle as O
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(58)
    n, k = 400, 30
    h = spectrum_matrix(rng, np.linspace(-3.0, 5.0, n))
    q = np.linalg.qr(crand(rng, n, k))[0]
    w_ref, z_ref, hz_ref = O.ritz(h, q)
    dH, dQ = D.to_device(h, eng.device), D.to_device(q, eng.device)
    dHQ, dZ, dHZ = (D.zeros(n, k, eng.device) for _ in range(3))
    w = eng.rayleigh_ritz(dH, dQ, dHQ, dZ, dHZ)
    assert np.max(np.abs(w - w_ref)) <= 1e-12 * np.max(np.abs(w_ref))
    Z, HZ = D.to_host(dZ), D.to_host(dHZ)
    assert np.linalg.norm(HZ - h @ Z) <= 1e-12 * np.linalg.norm(HZ)
    # Ritz vectors agree up to phase
    ov = np.abs(np.sum(Z.conj() * z_ref, axis=0))
    assert np.all(ov > 1 - 1e-9)


def test_hermitian_norms_and_hermitize(eng):
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(0)
    for n in (1, 31, 32, 33, 100, 257):
        a = crand(rng, n, n)
        d = D.to_device(a, eng.device)
        fro, devn = eng.hermitian_norms(d)
        assert abs(fro - np.linalg.norm(a)) <= 1e-13 * np.linalg.norm(a)
        assert abs(devn - np.linalg.norm(a - a.conj().T)) <= 1e-13 * np.linalg.norm(a)
        eng.hermitize(d)
        got = D.to_host(d)
        ref = (a + a.conj().T) / 2.0
        np.fill_diagonal(ref, ref.diagonal().real)
        assert np.array_equal(got, got.conj().T)
        assert np.max(np.abs(got - ref)) <= 1e-15 * np.max(np.abs(ref))


def test_cholesky_trtri_heevd(eng):
    from paper_1305_5120_b200 import device as D
    from paper_1305_5120_b200.errors import NotPositiveDefinite
    rng = np.random.default_rng(16)
    for n in (7, 64, 300, 1030):
        b = rand_spd(rng, n, shift=1.0)
        d = D.to_device(b, eng.device)
        eng.cholesky(d)
        lf = D.to_host(d)
        assert np.linalg.norm(np.triu(lf, 1)) == 0.0
        assert np.all(lf.diagonal().imag == 0) and np.all(lf.diagonal().real > 0)
        assert np.linalg.norm(lf @ lf.conj().T - b) <= 1e-12 * np.linalg.norm(b)
        x = D.zeros(n, n, eng.device)
        eng.trtri_lower(d, x)
        xi = D.to_host(x)
        assert np.linalg.norm(xi @ lf - np.eye(n)) <= 1e-11 * np.sqrt(n)
        assert np.linalg.norm(np.triu(xi, 1)) == 0.0
    with pytest.raises(NotPositiveDefinite) as exc:
        eng.cholesky(D.to_device(np.diag([1.0, 1.0, -1.0]).astype(complex), eng.device))
    assert exc.value.pivot == 3
    h = rand_hermitian(rng, 200)
    d = D.to_device(h, eng.device)
    w = eng.heevd(d)
    assert np.max(np.abs(w - np.linalg.eigvalsh(h))) <= 1e-13 * np.max(np.abs(w))


@pytest.mark.parametrize("cfg", [-1, 1, 3, 7, 10])
@pytest.mark.parametrize("split", [0, 1, 3])
def test_triangle_skipping_gemm_and_reduction(eng, cfg, split):
    """Linv A (row tile m reads k < m + BM) and W Linv^H (column tile j reads k < j + BN)
    skip Linv's zero triangle; the products equal the dense ones, including ragged
    orders, forced configs and split-K chunks that fall entirely in the zero block."""
    from paper_1305_5120_b200 import _native, device as D
    lib = _native.load()
    rng = np.random.default_rng(77 + cfg + 5 * split)
    try:
        assert lib.chfsi_gemm_override(cfg, split) == 0
        for n in (1, 37, 130, 301):
            a = crand(rng, n, n)
            a = a + a.conj().T
            linv = np.tril(crand(rng, n, n))
            dA, dL = D.to_device(a, eng.device), D.to_device(linv, eng.device)
            w, h = D.empty(n, n, eng.device), D.empty(n, n, eng.device)
            eng.reduce_to_standard(dA, dL, w, h)
            ref_w = linv @ a
            ref_h = ref_w @ linv.conj().T
            assert np.linalg.norm(D.to_host(w) - ref_w) <= 1e-13 * np.linalg.norm(ref_w), n
            assert np.linalg.norm(D.to_host(h) - ref_h) <= 1e-13 * np.linalg.norm(ref_h), n
    finally:
        lib.chfsi_gemm_override(-1, 0)


@pytest.mark.parametrize("cfg", [-1, 0, 1, 3, 5])
@pytest.mark.parametrize("split", [0, 1, 4])
def test_lower_only_gram(eng, cfg, split):
    """TRI_C_LOWER: the Gram X^H X computes only tiles touching the lower triangle (the
    CholQR Gram); its lower triangle equals the dense product."""
    from paper_1305_5120_b200 import _native, device as D
    lib = _native.load()
    rng = np.random.default_rng(5 + cfg + split)
    try:
        assert lib.chfsi_gemm_override(cfg, split) == 0
        for k, n in ((1, 50), (40, 700), (130, 2000), (257, 900)):
            x = crand(rng, n, k)
            g = D.zeros(k, k, eng.device)
            eng.zgemm("C", "N", k, k, n, 1.0, D.to_device(x, eng.device),
                      D.to_device(x, eng.device), 0.0, g, tri=eng.TRI_C_LOWER)
            got = np.tril(D.to_host(g))
            ref = np.tril(x.conj().T @ x)
            assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref), k
    finally:
        lib.chfsi_gemm_override(-1, 0)


def test_cholesky_inverse_step(eng):
    """chfsi_cholesky_inverse (replicated k x k step of a sharded CholQR pass):
    symmetrise, shift, factor, invert; diag(L), trace and the zpotrf pivot."""
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(21)
    for k in (1, 33, 300):
        x = crand(rng, 4 * k, k)
        g = x.conj().T @ x
        g_asym = g + 1e-13 * np.linalg.norm(g) * crand(rng, k, k)  # gathered, not Hermitian
        dG, dLi = D.to_device(g_asym, eng.device), D.empty(k, k, eng.device)
        diag, tr, info = eng.cholesky_inverse(dG, dLi, shift=0.5)
        gh = (g_asym + g_asym.conj().T) / 2 + 0.5 * np.eye(k)
        lo = np.linalg.cholesky(gh)
        assert info == 0
        assert abs(tr - np.trace(g_asym).real) <= 1e-12 * abs(tr)
        assert np.allclose(diag, np.diag(lo).real, rtol=1e-12, atol=0)
        li = D.to_host(dLi)
        assert np.array_equal(np.triu(li, 1), np.zeros((k, k)))
        assert np.linalg.norm(li @ lo - np.eye(k)) <= 1e-11 * k
    bad = np.diag([4.0, 1.0, -1.0, 2.0]).astype(complex)
    _, _, info = eng.cholesky_inverse(D.to_device(bad, eng.device), D.empty(4, 4, eng.device))
    assert info == 3


def test_trtri_blocked_matches_inverse(eng):
    """Recursive triangular inverse (its GEMMs skip the zero blocks of X11 / X22)."""
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(12)
    for n in (255, 600, 1100):
        lo = np.tril(crand(rng, n, n)) * 0.05 + np.diag(2.0 + rng.random(n))
        x = D.empty(n, n, eng.device)
        eng.trtri_lower(D.to_device(lo, eng.device), x)
        got = D.to_host(x)
        assert np.array_equal(np.triu(got, 1), np.zeros((n, n)))
        assert np.linalg.norm(got @ lo - np.eye(n)) <= 1e-12 * n


# every tile configuration and split factor the cost model can pick, on ragged shapes
_NCFG = 19
_TMA_FIRST = 7
_SUMS_FIRST = 14  # 3M kernels reading operand-sum planes: filter calls only
_BSUMS_FIRST = 17  # 3M kernels reading the B-sum plane only (narrow blocks)


@pytest.mark.parametrize("cfg", list(range(_SUMS_FIRST)))
@pytest.mark.parametrize("split", [1, 3])
def test_every_gemm_config_and_split(eng, cfg, split):
    from paper_1305_5120_b200 import _native, device as D
    lib = _native.load()
    rng = np.random.default_rng(100 + cfg * 7 + split)
    ops = [("N", "N")] if cfg >= _TMA_FIRST else [("N", "N"), ("C", "N"), ("N", "C"), ("C", "C")]
    try:
        assert lib.chfsi_gemm_override(cfg, split) == 0
        for (m, n, k) in [(70, 37, 203), (8, 8, 8), (129, 1, 300), (5, 66, 1029)]:
            for opa, opb in ops:
                A = crand(rng, m, k) if opa == "N" else crand(rng, k, m)
                B = crand(rng, k, n) if opb == "N" else crand(rng, n, k)
                C = crand(rng, m, n)
                ref = (0.3 + 0.1j) * ((A if opa == "N" else A.conj().T) @
                                      (B if opb == "N" else B.conj().T)) + (0.5 - 0.2j) * C
                dC = D.to_device(C, eng.device)
                eng.zgemm(opa, opb, m, n, k, 0.3 + 0.1j, D.to_device(A, eng.device),
                          D.to_device(B, eng.device), 0.5 - 0.2j, dC)
                got = D.to_host(dC)
                assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref), (m, n, k, opa, opb)
            # fused filter epilogue (square A, in place over Y0)
            if m == k or cfg >= 0:
                H = crand(rng, m, m)
                Y1, Y0 = crand(rng, m, n), crand(rng, m, n)
                dY0 = D.to_device(Y0, eng.device)
                eng.filter_step(D.to_device(H, eng.device), D.to_device(Y1, eng.device),
                                0.7, -0.2, dY0, 0.1, dY0)
                ref = 0.7 * (H @ Y1) - 0.2 * Y1 + 0.1 * Y0
                assert np.linalg.norm(D.to_host(dY0) - ref) <= 1e-13 * np.linalg.norm(ref)
    finally:
        lib.chfsi_gemm_override(-1, 0)


@pytest.mark.parametrize("cfg", [-1, _SUMS_FIRST, _SUMS_FIRST + 1, _SUMS_FIRST + 2, _BSUMS_FIRST,
                                 _BSUMS_FIRST + 1, 7, 11])
@pytest.mark.parametrize("split", [0, 1, 3])
def test_filter_with_sum_planes(eng, cfg, split):
    """chfsi_filter with 3M operand-sum planes (Hs, and per block the plane its step's
    epilogue or split-K reduce wrote): every sum-reading config and split against the
    oracle recurrence, ragged n and k; a forced config that reads no planes (7, 11) still
    leaves correct planes for the next step (separate sum pass); the B-sum-only configs
    (17, 18) with their packed tail blocks."""
    import oracle.chfsi_oracle as O
    from paper_1305_5120_b200 import _native, device as D
    from paper_1305_5120_b200.workloads import baseline_matrix
    lib = _native.load()
    try:
        assert lib.chfsi_gemm_override(cfg, split) == 0
        # sum planes need n % 8 == 0 (3-D A boxes); a ragged n takes the plain 3M kernels
        sizes = [(304, 37, 6), (1000, 120, 5), (136, 1, 3), (8, 1, 4), (16, 3, 2), (24, 40, 3)]
        if cfg < _SUMS_FIRST:
            sizes.append((301, 37, 6))
        if cfg >= _BSUMS_FIRST:
            # packed tail block (last live 8-column block with 1-4 columns) at every live
            # block count of a 32- and a 24-wide tile, and the unpacked 5-column tail
            sizes += [(64, 26, 3), (200, 20, 3), (72, 12, 2), (128, 33, 2), (128, 28, 2),
                      (128, 4, 2), (128, 29, 2)]
        for (n, k, m) in sizes:
            h, lam, _ = baseline_matrix(n, n)
            rng = np.random.default_rng(n + k + cfg)
            y = crand(rng, n, k)
            a, b, lam_ref = float(lam[min(k, n - 1)]), float(lam[-1]) * 1.05, float(lam[0])
            ref = O.cheb_filter(h, y, m, a, b, lam_ref)
            dW = D.zeros(n, k, eng.device)
            got = D.to_host(eng.filter(D.to_device(h, eng.device), D.to_device(y, eng.device),
                                       dW, m, a, b, lam_ref))
            assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref), (n, k, m)
    finally:
        lib.chfsi_gemm_override(-1, 0)


def test_filter_width_rule_large_operator(eng):
    """Operators of order >= 8192 plan their sum-plane filter steps by the width rule
    (24- or 32-column tiles, split-K to ~20000 CTAs): ragged and tiny widths against a
    torch (cuBLAS ZGEMM) product step by step, and the rule's plans are the ones used."""
    import ctypes
    import torch
    from paper_1305_5120_b200 import _native
    n = 8192
    dev = eng.device
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
    H = (H + H.mH) * 0.5
    H = H.contiguous()
    eng.declare_operator(H)
    try:
        # (20 / 25 / 28 / 33 / 42 / 57 / 60: packed tail blocks of 1-4 columns at every
        # live-block count of the 32- and 24-wide narrow kernels)
        for k in (1, 8, 20, 25, 26, 28, 33, 40, 42, 51, 57, 60, 100, 101, 201, 550):
            cfg, split = ctypes.c_int(), ctypes.c_int()
            _native.call("chfsi_gemm_plan", eng.h, 0, 0, 2, n, k, n, ctypes.byref(cfg),
                         ctypes.byref(split))
            # narrow blocks: the B-sum-only 3M kernels (cfg 17 / 18), which do not stream
            # H's sum plane (the power-capped regime, zgemm.cu)
            if 16 < k <= 64:
                assert cfg.value >= _BSUMS_FIRST, (k, cfg.value)
            else:
                assert _SUMS_FIRST <= cfg.value < _BSUMS_FIRST, (k, cfg.value)
            Y = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
            W = torch.empty_like(Y)
            a, b, lam_ref = -1.0, 1.0, -2.0
            # degree-2 filter: Y1 = s1/e (H - c) Y, Y2 = 2 s2/e (H - c) Y1 - s1 s2 Y
            c, e = (a + b) / 2, (b - a) / 2
            s1 = e / (lam_ref - c)
            s2 = 1.0 / (2.0 / s1 - s1)
            ref1 = (s1 / e) * (Y @ H - c * Y)  # (k, n) rows are columns: (H Y)^T = Y^T H^T
            ref2 = (2 * s2 / e) * (ref1 @ H - c * ref1) - s1 * s2 * Y
            out = eng.filter(H, Y.clone(), W, 2, a, b, lam_ref)
            err = float(torch.linalg.norm(out - ref2) / torch.linalg.norm(ref2))
            assert err <= 1e-13, (k, err)
            # the Rayleigh-Ritz product H Q on the declared operator takes the same plans
            # with the plain store epilogue
            HQ = torch.empty_like(Y)
            eng.apply_operator(H, Y, HQ)
            ref = Y @ H
            err = float(torch.linalg.norm(HQ - ref) / torch.linalg.norm(ref))
            assert err <= 1e-13, (k, err)
    finally:
        eng.declare_operator(None)


def test_narrow_kernels_every_width(eng):
    """Every block width the narrow-block rule takes (17-64 columns: 32- and 24-wide tiles,
    each live-block count, packed and plain tail blocks), one fused degree step and one
    split-K plan each, against a torch (cuBLAS ZGEMM) product."""
    import torch
    n = 8192
    dev = eng.device
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
    H = ((H + H.mH) * 0.5).contiguous()
    eng.declare_operator(H)
    try:
        for k in range(17, 65):
            Y = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
            W = torch.empty_like(Y)
            a, b, lam_ref = -1.0, 1.0, -2.0
            c, e = (a + b) / 2, (b - a) / 2
            s1 = e / (lam_ref - c)
            ref = (s1 / e) * (Y @ H - c * Y)
            out = eng.filter(H, Y.clone(), W, 1, a, b, lam_ref)
            err = float(torch.linalg.norm(out - ref) / torch.linalg.norm(ref))
            assert err <= 1e-13, (k, err)
            # column by column too: a wrong pairing in a packed block would hide in a norm
            cerr = torch.linalg.norm(out - ref, dim=1) / torch.linalg.norm(ref, dim=1)
            assert float(cerr.max()) <= 1e-13, (k, int(cerr.argmax()), float(cerr.max()))
    finally:
        eng.declare_operator(None)


@pytest.mark.parametrize("declared", [False, True])
def test_filter_sum_planes_with_padded_leading_dims(eng, declared):
    """Sum-plane filter steps on views with ld > n (H, Y and W inside larger buffers):
    the 3-D A box, the grouped H plane and the block planes honour the leading dims."""
    import torch
    n, k, pad = 1024, 50, 24
    dev = eng.device
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    Hbuf = torch.randn((n, n + pad), dtype=torch.complex128, device=dev, generator=g)
    H = Hbuf[:, :n]
    Hd = H.contiguous()
    Hd = (Hd + Hd.mH) * 0.5
    H.copy_(Hd)
    Ybuf = torch.randn((k, n + pad), dtype=torch.complex128, device=dev, generator=g)
    Y = Ybuf[:, :n]
    Wbuf = torch.zeros((k, n + 2 * pad), dtype=torch.complex128, device=dev)
    W = Wbuf[:, pad:pad + n]
    a, b, lam_ref = -1.0, 1.0, -2.0
    c, e = (a + b) / 2, (b - a) / 2
    s1 = e / (lam_ref - c)
    s2 = 1.0 / (2.0 / s1 - s1)
    Y0 = Y.clone()
    ref1 = (s1 / e) * (Y0 @ Hd - c * Y0)
    ref2 = (2 * s2 / e) * (ref1 @ Hd - c * ref1) - s1 * s2 * Y0
    if declared:
        eng.declare_operator(H)
    try:
        out = eng.filter(H, Y, W, 2, a, b, lam_ref)
    finally:
        if declared:
            eng.declare_operator(None)
    err = float(torch.linalg.norm(out - ref2) / torch.linalg.norm(ref2))
    assert err <= 1e-13, err
    assert torch.count_nonzero(Wbuf[:, :pad]) == 0 and torch.count_nonzero(Wbuf[:, pad + n:]) == 0


def test_declared_operator_filter_and_apply(eng):
    """chfsi_declare_operator: filter calls and H X products on the declared H reuse its
    sum plane (filter: the same result as undeclared, bit for bit; H X: the plan may
    differ in split-K, so to rounding); re-declaring after H changes picks up the new H;
    clearing returns to per-call planes."""
    import oracle.chfsi_oracle as O
    from paper_1305_5120_b200 import device as D
    from paper_1305_5120_b200.workloads import baseline_matrix
    n, k, m = 512, 40, 5
    h, lam, _ = baseline_matrix(n, n)
    rng = np.random.default_rng(9)
    y = crand(rng, n, k)
    a, b, lam_ref = float(lam[k]), float(lam[-1]) * 1.05, float(lam[0])
    dH = D.to_device(h, eng.device)

    def run():
        f = D.to_host(eng.filter(dH, D.to_device(y, eng.device), D.zeros(n, k, eng.device),
                                 m, a, b, lam_ref))
        hy = D.to_host(eng.apply_operator(dH, D.to_device(y, eng.device),
                                          D.zeros(n, k, eng.device)))
        return f, hy

    f0, hy0 = run()
    eng.declare_operator(dH)
    try:
        f1, hy1 = run()
        assert np.array_equal(f0, f1)
        assert np.linalg.norm(hy1 - hy0) <= 1e-15 * np.linalg.norm(hy0) * n ** 0.5
        ref = O.cheb_filter(h, y, m, a, b, lam_ref)
        assert np.linalg.norm(f1 - ref) <= 1e-12 * np.linalg.norm(ref)
        assert np.linalg.norm(hy1 - h @ y) <= 1e-14 * np.linalg.norm(h @ y)
        h2 = 2.0 * h
        dH.copy_(D.to_device(h2, eng.device))
        eng.declare_operator(dH)  # H changed: declare again
        _, hy2 = run()
        assert np.linalg.norm(hy2 - h2 @ y) <= 1e-14 * np.linalg.norm(h2 @ y)
    finally:
        eng.declare_operator(None)
    _, hy3 = run()
    assert np.linalg.norm(hy3 - hy2) <= 1e-15 * np.linalg.norm(hy2) * n ** 0.5


def test_sum_config_needs_planes(eng):
    """Forcing a sum-reading config on a product without planes is an argument error."""
    from paper_1305_5120_b200 import _native, device as D
    lib = _native.load()
    try:
        assert lib.chfsi_gemm_override(_SUMS_FIRST, 1) == 0
        x = D.zeros(64, 64, eng.device)
        st = lib.chfsi_zgemm(eng.h, 0, 0, 64, 64, 64, 1.0, 0.0, D.ptr(x), 64, D.ptr(x), 64, 0.0,
                             0.0, D.ptr(x), 64)
        assert st != 0 and b"sum planes" in lib.chfsi_last_error()
    finally:
        lib.chfsi_gemm_override(-1, 0)


def test_plan_is_tma_for_the_filter_shape(eng):
    import ctypes
    from paper_1305_5120_b200 import _native
    cfg, split = ctypes.c_int(), ctypes.c_int()
    _native.call("chfsi_gemm_plan", eng.h, 0, 0, 1, 20000, 2200, 20000, ctypes.byref(cfg),
                 ctypes.byref(split))
    assert cfg.value >= _TMA_FIRST and split.value == 1


@pytest.mark.parametrize("mul", [3, 4])
def test_complex_product_scheme(eng, mul):
    """3M (Ar Br, Ai Bi, (Ar+Ai)(Br+Bi)) and four-product TMA kernels give the same
    filter step and plain product to rounding, through the planner's own picks."""
    from paper_1305_5120_b200 import _native, device as D
    lib = _native.load()
    rng = np.random.default_rng(40 + mul)
    old = lib.chfsi_get_complex_mul()
    try:
        assert lib.chfsi_set_complex_mul(mul) == 0
        assert lib.chfsi_get_complex_mul() == mul
        for (n, k) in ((513, 26), (1000, 210), (2048, 64)):
            H = crand(rng, n, n)
            H = (H + H.conj().T) / 2
            Y1, Y0 = crand(rng, n, k), crand(rng, n, k)
            dY0 = D.to_device(Y0, eng.device)
            eng.filter_step(D.to_device(H, eng.device), D.to_device(Y1, eng.device),
                            0.7, -0.2, dY0, 0.1, dY0)
            ref = 0.7 * (H @ Y1) - 0.2 * Y1 + 0.1 * Y0
            assert np.linalg.norm(D.to_host(dY0) - ref) <= 1e-14 * np.linalg.norm(ref), (n, k)
            dC = D.zeros(n, k, eng.device)
            eng.zgemm("N", "N", n, k, n, 1.0, D.to_device(H, eng.device),
                      D.to_device(Y1, eng.device), 0.0, dC)
            ref = H @ Y1
            err = np.abs(D.to_host(dC) - ref).max(axis=0)
            # normwise per column: |C - HY|_max <= c eps ||H||_F ||y_j||
            bound = 4e-16 * np.linalg.norm(H) * np.linalg.norm(Y1, axis=0)
            assert np.all(err <= bound), (n, k, float((err / bound).max()))
        assert lib.chfsi_set_complex_mul(5) != 0
    finally:
        lib.chfsi_set_complex_mul(old)


def test_full_size_3m_matches_four_products(eng):
    """At the BASELINE c4 order (n = 20000) a filter call with 3M sum-plane kernels and
    one with four-product kernels agree to rounding on a 40-column block (the width
    rule's pick vs the cost model's four-product pick)."""
    import torch
    from paper_1305_5120_b200 import _native
    lib = _native.load()
    n, k, m = 20000, 40, 3
    dev = eng.device
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    H = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
    H = (H + H.mH) * 0.5
    Y = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
    old = lib.chfsi_get_complex_mul()
    outs = []
    try:
        for mul in (3, 4):
            assert lib.chfsi_set_complex_mul(mul) == 0
            W = torch.empty_like(Y)
            outs.append(eng.filter(H, Y.clone(), W, m, -1.0, 1.0, -2.0).clone())
    finally:
        lib.chfsi_set_complex_mul(old)
    del H
    err = float(torch.linalg.norm(outs[0] - outs[1]) / torch.linalg.norm(outs[1]))
    assert err <= 1e-13, err


def test_full_size_filter_on_exact_eigenvectors(eng):
    """Size-independent property at BASELINE c4 size (n = 20000): for an exact
    eigenvector q_j of H, p_m(H) q_j = p_m(lambda_j) q_j with the scalar closed form."""
    import torch
    import oracle.chfsi_oracle as O
    from paper_1305_5120_b200 import device as D
    n, m = 20000, 25
    dev = eng.device
    rng = np.random.default_rng(7)
    lam = np.sort(np.concatenate([rng.uniform(-1.0, 0.0, n // 5),
                                  10.0 ** rng.uniform(0.0, 2.0, n - n // 5)]))
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    q, _ = torch.linalg.qr(torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g))
    lt = torch.as_tensor(lam, dtype=torch.complex128, device=dev)
    h = (q * lt) @ q.conj().T
    hb = ((h + h.conj().T) / 2).conj().resolve_conj().contiguous()  # column-major block of H
    del h
    cols = [0, 1, 1999, 2000, 2199, n - 1]
    y = q[:, cols].T.contiguous()  # (k, n) block of exact eigenvectors
    w = torch.empty_like(y)
    a, b, lr = float(lam[2000]), float(lam[-1]) * 1.01, float(lam[0])
    out = eng.filter(hb, y.clone(), w, m, a, b, lr)
    got = out.cpu().numpy()
    qs = q[:, cols].T.cpu().numpy()
    gain = O.filter_gain(m, lam[cols], a, b, lr)
    errs = [float(np.linalg.norm(got[r] - gain[r] * qs[r])) for r in range(len(cols))]
    # FP64 budget: H = Q diag(lam) Q^H is exact only to ~1e-13 ||H|| at n = 20000, and
    # the normalised recurrence (|p| <= 1 on the spectrum) carries that forward
    assert max(errs) <= 1e-9, (errs, list(gain))


def test_shifted_cholqr3_on_ill_conditioned_block(eng):
    """cond(F) ~ 1e10: Cholesky of F^H F (cond ~ 1e20) breaks down, the shifted CholQR3
    path (Fukaya et al.) must still return an orthonormal basis of range(F)."""
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(5)
    n, k = 400, 12
    U = np.linalg.qr(crand(rng, n, k))[0]
    V = np.linalg.qr(crand(rng, k, k))[0]
    F = (U * np.logspace(0, -10, k)) @ V  # singular values 1 .. 1e-10
    dF = D.to_device(F, eng.device)
    dT, dQ = D.zeros(n, k, eng.device), D.zeros(n, k, eng.device)
    eng.orthonormalize(dF, None, dT, dQ)
    Q = D.to_host(dQ)
    assert np.linalg.norm(Q.conj().T @ Q - np.eye(k)) <= 1e-12 * np.sqrt(k)
    assert np.linalg.norm(U - Q @ (Q.conj().T @ U)) <= 1e-6  # same span (up to cond * eps)


def test_project_out_and_rr_from_hq(eng):
    """The split entry points used by the column-sharded solver: CGS2 projection on a
    column range equals projecting the full block; RR from a precomputed HQ equals RR."""
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(77)
    n, k, nl = 600, 24, 50
    L = np.linalg.qr(crand(rng, n, nl))[0]
    F = crand(rng, n, k)
    dL = D.to_device(L, eng.device)
    full = D.to_device(F, eng.device)
    eng.project_out(full, dL)
    part = D.to_device(F, eng.device)
    eng.project_out(part[5:17], dL)  # only columns 5..16
    ref = F - L @ (L.conj().T @ F)
    got_full, got_part = D.to_host(full), D.to_host(part)
    assert np.linalg.norm(got_full - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.linalg.norm(got_part[:, 5:17] - ref[:, 5:17]) <= 1e-12 * np.linalg.norm(ref)
    assert np.array_equal(got_part[:, :5], F[:, :5])
    h = spectrum_matrix(rng, np.linspace(-2.0, 3.0, n))
    q = np.linalg.qr(crand(rng, n, k))[0]
    dH, dQ = D.to_device(h, eng.device), D.to_device(q, eng.device)
    bufs = [D.zeros(n, k, eng.device) for _ in range(6)]
    w1, r1 = eng.rayleigh_ritz(dH, dQ, bufs[0], bufs[1], bufs[2], residuals=True)
    eng.zgemm("N", "N", n, k, n, 1.0, dH, dQ, 0.0, bufs[3])
    w2, r2 = eng.rayleigh_ritz_from_hq(dQ, bufs[3], bufs[4], bufs[5])
    assert np.array_equal(w1, w2) and np.array_equal(r1, r2)
    assert np.array_equal(D.to_host(bufs[1]), D.to_host(bufs[4]))


@pytest.mark.parametrize("off", [3, 8, 13])
@pytest.mark.parametrize("split", [0, 3])
def test_zgemm_tri_offsets_and_split(eng, off, split):
    """chfsi_zgemm_tri with every triangular flag at shard offsets that are and are not
    multiples of the 8-column K tile, auto and forced split-K: the TMA kernels load whole
    K tiles and cannot mask a triangular bound inside one, so unaligned offsets plan onto
    the element-masked kernels (a tile straddling two split-K chunks would otherwise be
    counted twice). Against numpy on factors whose zero triangle holds zeros."""
    from paper_1305_5120_b200 import _native, device as D
    lib = _native.load()
    rng = np.random.default_rng(900 + off + split)
    K, M, N = 600, 45, 37
    L = np.tril(crand(rng, K, K))
    X = crand(rng, K, 29)
    Y = crand(rng, 31, K)
    cases = [
        # (flag, opa, opb, A, B, m, n, reference)
        (eng.TRI_B_LOWER, "N", "N", Y, L[:, off:off + N], 31, N, Y @ L[:, off:off + N]),
        (eng.TRI_A_LOWER, "N", "N", L[off:off + M, :], X, M, 29, L[off:off + M, :] @ X),
        (eng.TRI_B_UPPER, "N", "C", Y, L[off:off + N, :], 31, N, Y @ L[off:off + N, :].conj().T),
        (eng.TRI_A_UPPER, "C", "N", L[:, off:off + M], X, M, 29, L[:, off:off + M].conj().T @ X),
    ]
    try:
        assert lib.chfsi_gemm_override(-1, split) == 0
        for flag, opa, opb, A, B, m, n, ref in cases:
            dC = D.zeros(m, n, eng.device)
            eng.zgemm(opa, opb, m, n, K, 1.0, D.to_device(A, eng.device),
                      D.to_device(B, eng.device), 0.0, dC, tri=flag, tri_offset=off)
            got = D.to_host(dC)
            assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref), (flag, off, split)
    finally:
        lib.chfsi_gemm_override(-1, 0)


@pytest.mark.parametrize("m,k,pad", [(256, 256, 0), (300, 1000, 5), (5003, 4001, 13), (20000, 64, 0)])
def test_zgemv_hbm_path(eng, m, k, pad):
    """Matrix-vector products (N = 1, op N x N: the Lanczos H v) take the HBM-bound GEMV
    (row per thread, column-split partials summed in fixed order): alpha/beta, a padded
    leading dimension, bit-identical repeats, against numpy."""
    import torch
    from paper_1305_5120_b200 import device as D
    rng = np.random.default_rng(m + k + pad)
    A = crand(rng, m, k)
    x = crand(rng, k, 1)
    y0 = crand(rng, m, 1)
    dA_full = D.zeros(m + pad, k, eng.device)
    dA_full[:, :m].copy_(torch.from_numpy(np.ascontiguousarray(A.T)).to(eng.device))
    dA = dA_full[:, :m] if pad else dA_full
    al, be = 0.6 + 0.3j, -0.25 + 0.1j
    outs = []
    for _ in range(2):
        dy = D.to_device(y0, eng.device)
        eng.zgemm("N", "N", m, 1, k, al, dA, D.to_device(x, eng.device), be, dy)
        outs.append(D.to_host(dy))
    ref = al * (A @ x) + be * y0
    assert np.array_equal(outs[0], outs[1])
    assert np.linalg.norm(outs[0] - ref) <= 1e-14 * np.linalg.norm(ref) * np.sqrt(k)
    n0 = eng.launch_count(reset=True)
    dy = D.to_device(y0, eng.device)
    eng.zgemm("N", "N", m, 1, k, 1.0, dA, D.to_device(x, eng.device), 0.0, dy)
    assert eng.launch_count(reset=True) == 2  # partial + fixed-order finish
    del n0


_STAGE_SCRIPT = r"""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
import oracle.chfsi_oracle as O
from paper_1305_5120_b200 import _native, device as D
from paper_1305_5120_b200.workloads import baseline_matrix
dev = torch.device("cuda", 0)
eng = D.Engine.get(dev)
rng = np.random.default_rng(5)
# pageable F-order block through the staging ring (4 MB slots -> 14 chunks, 3 workers)
a = np.asfortranarray(rng.standard_normal((5000, 700)) + 1j * rng.standard_normal((5000, 700)))
t = D.to_device(a, dev)
assert np.array_equal(D.to_host(t), a)
# strided source (ld > rows) through chfsi_upload, and a page-locked source
big = np.asfortranarray(rng.standard_normal((5003, 300)) + 1j * rng.standard_normal((5003, 300)))
out = torch.empty((300, 4990), dtype=torch.complex128, device=dev)
_native.call("chfsi_upload", eng.h, ctypes.c_void_p(big.ctypes.data), 5003, 4990, 300,
             ctypes.c_void_p(out.data_ptr()), 4990)
assert np.array_equal(D.to_host(out), big[:4990])
pin = torch.empty((300, 5003), dtype=torch.complex128, pin_memory=True)
pin.copy_(torch.from_numpy(np.ascontiguousarray(big.T)))
out2 = torch.empty((300, 5003), dtype=torch.complex128, device=dev)
_native.call("chfsi_upload", eng.h, ctypes.c_void_p(pin.data_ptr()), 5003, 5003, 300,
             ctypes.c_void_p(out2.data_ptr()), 5003)
assert torch.equal(out2.cpu(), pin)
# streamed filter with a pageable H of 64 MB: each row panel in many staged chunks
n, k, m = 2048, 40, 4
h, lam, _ = baseline_matrix(n, n)
h = np.asfortranarray(h)
y = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
aa, bb, lr = float(lam[k]), float(lam[-1]) * 1.05, float(lam[0])
ref = O.cheb_filter(h, y, m, aa, bb, lr)
dH = D.empty(n, n, dev)
got = D.to_host(eng.filter_streamed(h, dH, D.to_device(y, dev), D.zeros(n, k, dev), m, aa, bb,
                                    lr, panels=4))
assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
assert np.array_equal(D.to_host(dH), h)
print("staging ok")
"""


def test_pageable_staged_uploads():
    """Pageable host operands go through the native pinned staging ring (csrc/staging.cu):
    contiguous and strided sources, many chunks per panel (4 MB slots), a page-locked
    source taking the direct copy, and the streamed filter on a pageable H -- all
    bit-exact transfers."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CHFSI_STAGE_MB="4", CHFSI_STAGE_THREADS="3")
    out = subprocess.run([sys.executable, "-c", _STAGE_SCRIPT], capture_output=True, text=True,
                         timeout=600, cwd=root, env=env)
    assert out.returncode == 0 and "staging ok" in out.stdout, out.stderr[-3000:]
