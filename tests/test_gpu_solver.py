"""GPU parity of the full solver against the oracle (reference algorithm restated on the
CPU) on the same seeded inputs and start vectors.

Bar (BASELINE.json north_star): eigenvalues within 1e-10 relative, every residual below
tol, the same number of converged pairs, largest principal angle (sine formula) < 1e-8.
Iteration counts may differ by rounding-induced lock timing."""

import numpy as np
import pytest

from conftest import gapped_matrix, rand_hermitian, rand_spd, spectrum_matrix

pytestmark = pytest.mark.gpu


def _angle(u, v):
    import oracle.chfsi_oracle as O
    return O.largest_angle_sine(u, v)


def test_known_diagonal_spectrum():
    import paper_1305_5120_b200 as G
    h = np.diag(np.arange(1.0, 101.0)).astype(complex)
    cfg = G.SolverConfig(nev=5)
    lam, vecs, report = G.chfsi_solve(h, None, cfg, seed=0)
    assert np.max(np.abs(lam - np.arange(1.0, 6.0))) <= 1e-9
    assert np.all(G.residuals(h, vecs, lam) < cfg.tol)
    assert report.converged and vecs.orthonormal


@pytest.mark.parametrize("seed,n,nev", [(56, 150, 12), (52, 90, 9), (55, 80, 8), (7, 400, 40)])
def test_matches_oracle_same_start(seed, n, nev):
    import oracle.chfsi_oracle as O
    import paper_1305_5120_b200 as G
    h, evals = gapped_matrix(seed, n, nev)
    cfg = G.SolverConfig(nev=nev, max_outer_iters=200)
    lam, vecs, rep = G.chfsi_solve(h, None, cfg, seed=seed + 1)
    lam_o, v_o, rep_o = O.solve(h, None, nev, cfg.buffer_cols, cfg.degree, cfg.tol, 200,
                                seed=seed + 1)
    assert len(lam) == len(lam_o) == nev
    assert np.max(np.abs(lam - lam_o) / np.abs(lam_o).clip(1e-300)) <= 1e-10
    assert np.all(G.residuals(h, vecs, lam) < cfg.tol)
    assert _angle(vecs.entries, v_o) < 1e-8
    assert abs(rep.outer_iterations - len(rep_o["iterations"])) <= 2


def test_exact_start_single_iteration():
    import paper_1305_5120_b200 as G
    h, _ = gapped_matrix(50, 80, 8)
    cfg = G.SolverConfig(nev=8)
    lam_o, v_o = np.linalg.eigh(h)
    s = cfg.nev + cfg.buffer_cols
    lam, vecs, report = G.chfsi_solve(h, v_o[:, :s], cfg, seed=1)
    assert report.outer_iterations == 1
    assert np.max(np.abs(lam - lam_o[:8])) <= 1e-10


def test_dimension_guard_before_work():
    import paper_1305_5120_b200 as G
    h = np.diag([1.0, 2.0, 3.0]).astype(complex)
    G.reset_product_count()
    with pytest.raises(G.ContractViolation):
        G.chfsi_solve(h, None, G.SolverConfig(nev=3), seed=0)
    assert G.product_count() == 0


def test_not_converged_carries_partials():
    import paper_1305_5120_b200 as G
    h, _ = gapped_matrix(51, 60, 6, lo=4.0, hi_lo=4.2)
    cfg = G.SolverConfig(nev=6, degree=1, max_outer_iters=2)
    with pytest.raises(G.NotConverged) as exc:
        G.chfsi_solve(h, None, cfg, seed=2)
    err = exc.value
    assert err.report.outer_iterations == 2
    assert len(err.eigenvalues) < 6
    assert not err.report.converged


def test_determinism_bit_identical():
    import paper_1305_5120_b200 as G
    h, _ = gapped_matrix(53, 70, 7)
    cfg = G.SolverConfig(nev=7)
    lam1, v1, r1 = G.chfsi_solve(h, None, cfg, seed=4)
    lam2, v2, r2 = G.chfsi_solve(h, None, cfg, seed=4)
    assert np.array_equal(lam1, lam2)
    assert np.array_equal(v1.entries, v2.entries)
    assert r1.total_matmuls == r2.total_matmuls
    assert [s.max_resid for s in r1.iterations] == [s.max_resid for s in r2.iterations]


def test_work_accounting_matches_counter():
    import paper_1305_5120_b200 as G
    h, _ = gapped_matrix(55, 80, 8)
    cfg = G.SolverConfig(nev=8)
    G.reset_product_count()
    _, _, report = G.chfsi_solve(h, None, cfg, seed=6)
    assert G.product_count() == report.total_matmuls
    for it in report.iterations:
        assert it.matmuls == (cfg.degree + 1) * it.filtered_cols


def test_inverted_prior_raises_degenerate():
    import paper_1305_5120_b200 as G
    h = np.diag(np.arange(1.0, 31.0)).astype(complex)
    with pytest.raises(G.FilterDegenerate):
        G.chfsi_solve(h, None, G.SolverConfig(nev=4), prior=(9.0, 2.0), seed=0)


def test_locked_counts_monotone_and_recheck():
    import paper_1305_5120_b200 as G
    h, _ = gapped_matrix(52, 90, 9)
    lam, vecs, report = G.chfsi_solve(h, None, G.SolverConfig(nev=9), seed=3)
    counts = report.converged_counts
    assert all(b >= a for a, b in zip(counts, counts[1:]))
    assert counts[-1] == 9
    assert np.all(G.residuals(h, vecs, lam) < 1e-10)


def test_oracle_equivalence_random_problems():
    """Reference criterion 1 in miniature: random Hermitian problems vs a dense eigensolver."""
    import paper_1305_5120_b200 as G
    for i in range(12):
        rng = np.random.default_rng(5000 + i)
        n = int(rng.integers(20, 201))
        nev = int(rng.integers(1, max(1, int(0.2 * n)) + 1))
        h = rand_hermitian(rng, n, scale=2.0)
        cfg = G.SolverConfig(nev=nev, max_outer_iters=300)
        lam, vecs, _ = G.chfsi_solve(h, None, cfg, seed=rng)
        lam_o = np.linalg.eigvalsh(h)
        norm2 = max(abs(lam_o[0]), abs(lam_o[-1]))
        assert np.max(np.abs(lam - lam_o[:nev])) <= 10 * cfg.tol * norm2
        assert float(G.residuals(h, vecs, lam).max()) < cfg.tol


def test_generalized_matches_oracle():
    import oracle.chfsi_oracle as O
    import paper_1305_5120_b200 as G
    rng = np.random.default_rng(62)
    a = rand_hermitian(rng, 50, scale=3.0)
    b = rand_spd(rng, 50)
    nev = 8
    cfg = G.SolverConfig(nev=nev, max_outer_iters=200)
    lam, c, rep = G.solve_generalized(a, b, None, cfg, seed=10)
    lam_o, c_o, _ = O.solve_generalized(a, b, None, nev, cfg.buffer_cols, max_it=200, seed=10)
    assert np.max(np.abs(lam - lam_o) / np.abs(lam_o)) <= 1e-10
    ce = c.entries
    res = a @ ce - (b @ ce) * lam
    bound = cfg.tol * (np.linalg.norm(a, 1) + np.linalg.norm(b, 1))
    assert np.max(np.linalg.norm(res, axis=0)) <= bound
    assert np.linalg.norm(ce.conj().T @ b @ ce - np.eye(nev)) <= 1e-9


def test_generalized_b_identity_and_a_multiple_of_b():
    import paper_1305_5120_b200 as G
    rng = np.random.default_rng(60)
    a = spectrum_matrix(rng, np.concatenate([np.linspace(0.0, 3.0, 6), np.linspace(5.0, 9.0, 34)]))
    cfg = G.SolverConfig(nev=6)
    lam_g, v_g, _ = G.solve_generalized(a, np.eye(40, dtype=complex), None, cfg, seed=8)
    lam_s, v_s, _ = G.chfsi_solve(a, None, cfg, seed=8)
    assert np.max(np.abs(lam_g - lam_s)) <= 1e-13
    b = rand_spd(np.random.default_rng(61), 30)
    lam, c, _ = G.solve_generalized(2.0 * b, b, None, G.SolverConfig(nev=5), seed=9)
    assert np.max(np.abs(lam - 2.0)) <= 1e-10


def test_generalized_warm_start_single_iteration():
    import paper_1305_5120_b200 as G
    rng = np.random.default_rng(64)
    a = rand_hermitian(rng, 40, scale=3.0)
    b = rand_spd(rng, 40)
    cfg = G.SolverConfig(nev=5)
    lam1, c1, _ = G.solve_generalized(a, b, None, cfg, seed=12)
    pad_rng = np.random.default_rng(65)
    s = cfg.nev + cfg.buffer_cols
    y0 = np.hstack([c1.entries, pad_rng.standard_normal((40, s - 5)) +
                    1j * pad_rng.standard_normal((40, s - 5))])
    lam2, _, rep2 = G.solve_generalized(a, b, y0, cfg, prior=(float(lam1[0]), float(lam1[-1]) + 0.5),
                                        seed=13)
    assert rep2.outer_iterations == 1
    assert np.max(np.abs(lam2 - lam1)) <= 1e-10


def test_indefinite_b_rejected():
    import paper_1305_5120_b200 as G
    rng = np.random.default_rng(66)
    a = rand_hermitian(rng, 10)
    bad = np.diag(np.concatenate([np.ones(9), [-1.0]])).astype(complex)
    with pytest.raises(G.NotPositiveDefinite) as exc:
        G.solve_generalized(a, bad, None, G.SolverConfig(nev=2), seed=0)
    assert exc.value.pivot == 10


# ----------------------------------------------------------------------
# parity against fixtures produced by the reference itself (tests/golden)

def _gold(name):
    import os
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name))


@pytest.mark.parametrize("gs,n,nev,ss", [(56, 150, 12, 7), (52, 90, 9, 3), (55, 80, 8, 6),
                                          (53, 70, 7, 4)])
def test_small_problems_match_reference_golden(gs, n, nev, ss):
    import paper_1305_5120_b200 as G
    g = _gold("solver_small.npz")
    key = f"g{gs}_n{n}_nev{nev}_s{ss}"
    h, _ = gapped_matrix(gs, n, nev)
    lam, v, rep = G.chfsi_solve(h, None, G.SolverConfig(nev=nev), seed=ss)
    ref = g[key + "_lam"]
    assert np.max(np.abs(lam - ref) / np.abs(ref)) <= 1e-10
    assert _angle(v.entries, g[key + "_v"]) < 1e-8
    assert len(lam) == len(ref)
    assert abs(rep.outer_iterations - len(g[key + "_it_converged"])) <= 2


def test_baseline_c0_matches_reference_golden():
    """BASELINE config 0 in full (n=1000, nev=100, nex=20, m=15, tol 1e-10, random
    start; generator seed 0, solver seed 1) against the reference's own result."""
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.workloads import baseline_matrix
    g = _gold("c0.npz")
    h, lam_true, _ = baseline_matrix(0, 1000)
    cfg = G.SolverConfig(nev=100, buffer=20, degree=15, max_outer_iters=20000)
    lam, v, rep = G.chfsi_solve(h, None, cfg, seed=1)
    ref = g["lam"]
    assert len(lam) == len(ref) == 100
    assert np.max(np.abs(lam - ref) / np.abs(ref)) <= 1e-10
    assert np.max(G.residuals(h, v, lam)) < cfg.tol
    assert _angle(v.entries, g["v"]) < 1e-8
    # iteration trace: the reference needed len(it_converged) iterations
    n_ref = len(g["it_converged"])
    assert abs(rep.outer_iterations - n_ref) <= max(5, n_ref // 50)


def test_reuse_sequence_matches_reference_golden():
    """BASELINE c1 recipe at n=200 (3 problems, reuse), driven like the reference's
    solve_sequence (same pad / solver Generator seeds)."""
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.workloads import baseline_sequence
    g = _gold("sequence_small.npz")
    probs = baseline_sequence(5, 200, 3)
    spec = G.SequenceSpec(n=200, N=3, nev=20, seed=5)
    seq = G.ProblemSequence(spec=spec, problems=[(G.HermitianDenseMatrix(a, rtol=1e-10), None)
                                                 for a, _ in probs])
    cfg = G.SolverConfig(nev=20, buffer=4, degree=20, max_outer_iters=5000)
    rep = G.solve_sequence(seq, cfg, "reuse")
    for i in range(3):
        ref = g[f"lam{i}"]
        assert np.max(np.abs(rep.eigenvalues[i] - ref) / np.abs(ref)) <= 1e-10
        assert _angle(rep.vectors[i].entries, g[f"v{i}"]) < 1e-8
        assert abs(rep.reports[i].outer_iterations - int(g[f"iters{i}"])) <= 3


def test_generalized_matches_reference_golden():
    import paper_1305_5120_b200 as G
    g = _gold("generalized.npz")
    lam, c, rep = G.solve_generalized(g["a"], g["b"], None, G.SolverConfig(nev=8), seed=10)
    assert np.max(np.abs(lam - g["lam"]) / np.abs(g["lam"])) <= 1e-10
    b = g["b"]
    ce = c.entries
    assert np.linalg.norm(ce.conj().T @ b @ ce - np.eye(8)) <= 1e-9
    assert _angle(ce, g["c"]) < 1e-8


def test_filter_and_lanczos_match_reference_golden():
    import paper_1305_5120_b200 as G
    g = _gold("filter.npz")
    deg, a, b, lr = g["rand_spec"]
    out = G.chebyshev_filter(g["rand_h"], g["rand_y"], G.FilterSpec(int(deg), a, b, lr)).entries
    ref = g["rand_out"]
    assert np.linalg.norm(out - ref) <= 1e-13 * np.linalg.norm(ref)
    gl = _gold("lanczos.npz")
    for s, bref in enumerate(gl["bounds"]):
        assert abs(G.lanczos_upper_bound(gl["h"], 10, seed=s) - bref) <= 1e-12 * abs(bref)


def test_generalized_baseline_recipe_sequence():
    """c2-style generalized reuse sequence (S = I + 0.1 B^H B/||B^H B||) at n=400:
    every cycle converges, B-orthonormal, generalized residual below the scaled bound,
    and eigenvalues agree with the oracle's explicit reduction."""
    import oracle.chfsi_oracle as O
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.workloads import baseline_sequence
    probs = baseline_sequence(8, 400, 3, generalized=True)
    seq = G.ProblemSequence(spec=G.SequenceSpec(n=400, N=3, nev=40, seed=8),
                            problems=[(a, s) for a, s in probs])
    cfg = G.SolverConfig(nev=40, buffer=4, degree=20, max_outer_iters=20000)
    rep = G.solve_sequence(seq, cfg, "reuse")
    for (a, s), lam, c in zip(probs, rep.eigenvalues, rep.vectors):
        ce = c.entries
        res = np.linalg.norm(a @ ce - (s @ ce) * lam, axis=0)
        assert np.max(res) <= cfg.tol * (np.linalg.norm(a, 1) + np.linalg.norm(s, 1))
        assert np.linalg.norm(ce.conj().T @ s @ ce - np.eye(40)) <= 1e-9
        lf = O.cholesky(s)
        ref = np.linalg.eigvalsh(O.reduce_standard(a, lf))[:40]
        assert np.max(np.abs(lam - ref) / np.abs(ref)) <= 1e-10


def test_reduction_at_scale_matches_oracle():
    """reduce_to_standard / back_transform at n = 3000 (blocked recursive triangular
    inverse: several recursion levels) against the oracle's LAPACK ztrsm route."""
    import oracle.chfsi_oracle as O
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.workloads import spd_metric
    n = 3000
    rng = np.random.default_rng(31)
    a = rand_hermitian(rng, n, scale=5.0)
    s = spd_metric(rng, n)
    lf_o = O.cholesky(s)
    h_o = O.reduce_standard(a, lf_o)
    lf = G.cholesky_factor(s)
    assert np.linalg.norm(lf.entries - lf_o) <= 1e-13 * np.linalg.norm(lf_o)
    h = G.reduce_to_standard(a, lf).entries
    assert np.linalg.norm(h - h_o) <= 1e-12 * np.linalg.norm(h_o)
    y = rng.standard_normal((n, 7)) + 1j * rng.standard_normal((n, 7))
    c = G.back_transform(y, lf).entries
    c_o = O.tri_solve(lf_o, y, side="left", adjoint=True)
    assert np.linalg.norm(c - c_o) <= 1e-12 * np.linalg.norm(c_o)


@pytest.mark.parametrize("n,nev,nex", [(2, 1, 1), (5, 1, 1), (9, 3, 6), (16, 4, 12), (33, 1, 2)])
def test_edge_sizes_including_full_search_space(n, nev, nex):
    """Tiny orders, nev = 1, and nev + buffer == n (the search block is the whole space)."""
    import paper_1305_5120_b200 as G
    rng = np.random.default_rng(n * 10 + nev)
    evals = np.sort(rng.uniform(-3.0, 3.0, n))
    h = spectrum_matrix(rng, evals)
    cfg = G.SolverConfig(nev=nev, buffer=nex, degree=8, max_outer_iters=500)
    lam, vecs, rep = G.chfsi_solve(h, None, cfg, seed=1)
    assert lam.shape == (nev,) and (vecs.n, vecs.s) == (n, nev)
    assert np.max(np.abs(lam - evals[:nev])) <= 1e-9 * max(1.0, np.max(np.abs(evals)))
    assert np.all(G.residuals(h, vecs, lam) < cfg.tol)


def test_wrapper_inputs_and_device_start_block():
    """HermitianDenseMatrix / VectorBlock inputs (device-resident) give the same answer as
    raw ndarrays; a VectorBlock start block is used without a host round trip."""
    import paper_1305_5120_b200 as G
    h, _ = gapped_matrix(71, 120, 10)
    hm = G.HermitianDenseMatrix(h)
    cfg = G.SolverConfig(nev=10)
    lam_a, v_a, _ = G.chfsi_solve(h, None, cfg, seed=2)
    lam_b, v_b, _ = G.chfsi_solve(hm, None, cfg, seed=2)
    assert np.max(np.abs(lam_a - lam_b)) <= 1e-12 * np.max(np.abs(lam_a))
    s = cfg.nev + cfg.buffer_cols
    y0 = G.VectorBlock(np.linalg.qr(np.random.default_rng(3).standard_normal((120, s)) + 0j)[0])
    lam_c, _, _ = G.chfsi_solve(hm, y0, cfg, prior=(float(lam_a[0]), float(lam_a[-1]) + 0.5), seed=4)
    assert np.max(np.abs(lam_c - lam_a)) <= 1e-9


def test_reference_config_object_is_accepted():
    """A config with the reference's field names (e.g. chfsi.core.SolverConfig) is accepted."""
    import paper_1305_5120_b200 as G

    class RefConfig:
        nev, tol, max_outer_iters, degree, lanczos_steps, buffer = 6, 1e-10, 200, 20, 10, None
        buffer_cols = 1

    h, _ = gapped_matrix(72, 60, 6)
    lam, v, rep = G.chfsi_solve(h, None, RefConfig(), seed=5)
    assert len(lam) == 6 and rep.converged


def test_generalized_fixed_metric_factor_is_cached():
    """A HermitianDenseMatrix metric keeps (L, L^-1): the second solve reuses them."""
    import paper_1305_5120_b200 as G
    rng = np.random.default_rng(73)
    a = rand_hermitian(rng, 80, scale=3.0)
    s = G.HermitianDenseMatrix(rand_spd(rng, 80))
    cfg = G.SolverConfig(nev=5)
    lam1, c1, _ = G.solve_generalized(a, s, None, cfg, seed=1)
    lf, linv = s._factor
    lam2, c2, _ = G.solve_generalized(a, s, None, cfg, seed=1)
    assert s._factor[0] is lf and s._factor[1] is linv
    assert np.array_equal(lam1, lam2)


def test_rank_collapse_in_start_block_is_replaced_like_the_reference():
    """Duplicate start columns make the bootstrap QR rank-deficient; like core.py:375-381
    the collapsed column is replaced by a fresh random vector from the solver's
    Generator, and the solve converges to the oracle's (same replacement semantics)."""
    import oracle.chfsi_oracle as O
    import paper_1305_5120_b200 as G
    h, evals = gapped_matrix(81, 100, 8)
    cfg = G.SolverConfig(nev=8, buffer=3, max_outer_iters=300)
    rng0 = np.random.default_rng(3)
    y0 = rng0.standard_normal((100, 11)) + 1j * rng0.standard_normal((100, 11))
    y0[:, 5] = y0[:, 2]
    lam, v, rep = G.chfsi_solve(h, y0, cfg, seed=4)
    lam_o, v_o, _ = O.solve(h, y0, 8, 3, cfg.degree, cfg.tol, 300, seed=4)
    assert np.max(np.abs(lam - lam_o) / np.abs(lam_o)) <= 1e-10
    assert np.max(np.abs(lam - evals[:8]) / np.abs(evals[:8])) <= 1e-10
    assert _angle(v.entries, v_o) < 1e-8


def test_linalg_dropin_semantics():
    """Reference test_linalg.py behaviours on the GPU-backed linalg layer."""
    import paper_1305_5120_b200 as G
    rng = np.random.default_rng(15)
    h = rand_hermitian(rng, 8)
    with pytest.raises(G.OracleNoConvergence):
        G.oracle_eig(h, max_sweeps=0)
    lam, v = G.oracle_eig(np.diag([3.0, 1.0, 2.0]).astype(complex))
    assert np.array_equal(lam, [1.0, 2.0, 3.0])
    assert np.allclose(np.abs(v.entries), np.eye(3)[:, [1, 2, 0]], atol=1e-14)
    lam, _ = G.oracle_eig(np.array([[2.0, 1.0 - 1j], [1.0 + 1j, 3.0]]))
    assert np.allclose(lam, [1.0, 4.0], atol=1e-14)
    # gemm: alpha = 0 keeps C and counts nothing; square A counted; vector operand
    G.reset_product_count()
    x = rng.standard_normal((4, 3)) + 1j * rng.standard_normal((4, 3))
    out = G.gemm(0.0, np.eye(4, dtype=complex), x, beta=1.0, c=x)
    assert np.array_equal(out, x) and G.product_count() == 0
    sq = rng.standard_normal((6, 6)) + 0j
    blk = rng.standard_normal((6, 3)) + 0j
    G.gemm(1.0, sq, blk)
    assert G.product_count() == 3
    G.gemm(1.0, rng.standard_normal((4, 6)) + 0j, blk)
    assert G.product_count() == 3
    v5 = rng.standard_normal(5) + 1j * rng.standard_normal(5)
    a5 = rng.standard_normal((5, 5)) + 1j * rng.standard_normal((5, 5))
    assert G.gemm(1.0, a5, v5).shape == (5,)
    assert np.allclose(G.gemm(1.0, a5, v5), a5 @ v5, rtol=1e-14, atol=0)
    with pytest.raises(G.DimensionMismatch):
        G.gemm(1.0, np.ones((3, 4), dtype=complex), np.ones((3, 2), dtype=complex))
    with pytest.raises(G.ContractViolation):
        G.gemm(1.0, np.eye(2, dtype=complex), np.eye(2, dtype=complex), beta=1.0)
    # QR rank collapse names the column; Cholesky pivot is 1-based
    y = rng.standard_normal((10, 3)) + 1j * rng.standard_normal((10, 3))
    y[:, 2] = y[:, 0]
    with pytest.raises(G.RankDeficient) as exc:
        G.householder_qr(y)
    assert exc.value.column == 2
    with pytest.raises(G.NotPositiveDefinite) as exc:
        G.cholesky_factor(np.diag([1.0, -1.0]).astype(complex))
    assert exc.value.pivot == 2
    lf = G.cholesky_factor(np.diag([4.0, 9.0]).astype(complex))
    assert np.array_equal(lf.entries, np.diag([2.0, 3.0]).astype(complex))


@pytest.mark.parametrize("n", [5, 130, 700])
def test_triangular_solve_and_trmm_use_only_the_lower_triangle(n):
    """linalg.py:326-366: ztrsm / ztrmm with lower=1 read only the lower triangle of a raw
    factor; the device versions (triangle-skipping GEMMs on L^-1 or L) must too."""
    import paper_1305_5120_b200 as G
    rng = np.random.default_rng(n)
    lo = np.tril(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * 0.1
    lo[np.diag_indices(n)] = 1.0 + rng.random(n)
    raw = lo + np.triu(rng.standard_normal((n, n)), 1) * 7.0  # garbage above the diagonal
    x = rng.standard_normal((n, 9)) + 1j * rng.standard_normal((n, 9))
    xr = rng.standard_normal((9, n)) + 1j * rng.standard_normal((9, n))
    li = np.linalg.inv(lo)
    cases = [(x, "left", False, li @ x), (x, "left", True, li.conj().T @ x),
             (xr, "right", False, xr @ li), (xr, "right", True, xr @ li.conj().T)]
    for fac in (raw, G.LowerTriangularFactor(lo)):
        for blk, side, adj, ref in cases:
            got = G.triangular_solve(fac, blk, side=side, adjoint=adj)
            assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref), (side, adj)
        got = G.trmm_adjoint(fac, x)
        ref = lo.conj().T @ x
        assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


def test_criterion7_report_csv_deterministic():
    """Reference criterion 7 (test_acceptance.py:199-227): repeated runs give identical
    non-timing report columns, eigenvalues and vectors."""
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.report import report_csv_text
    rng = np.random.default_rng(9100)
    evals = np.concatenate([np.sort(rng.uniform(0, 4, 8)), np.sort(rng.uniform(6, 10, 92))])
    h = spectrum_matrix(rng, evals)
    cfg = G.SolverConfig(nev=8)

    def non_timing(rep):
        return [",".join(ln.split(",")[:5]) for ln in report_csv_text(rep).splitlines()]

    lam1, v1, r1 = G.chfsi_solve(h, None, cfg, seed=3)
    lam2, v2, r2 = G.chfsi_solve(h, None, cfg, seed=3)
    assert non_timing(r1) == non_timing(r2)
    assert np.array_equal(lam1, lam2) and np.array_equal(v1.entries, v2.entries)
