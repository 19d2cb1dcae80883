"""Host-side logic that needs no GPU: config/spec validation (core.py:59-115), error
types (errors.py), duck-typed configs, BASELINE workload generators, sequence specs."""

import numpy as np
import pytest

import paper_1305_5120_b200 as G
from paper_1305_5120_b200 import workloads as W


def test_solver_config_validation():
    with pytest.raises(G.ContractViolation):
        G.SolverConfig(nev=0)
    with pytest.raises(G.ContractViolation):
        G.SolverConfig(nev=4, tol=0.0)
    with pytest.raises(G.ContractViolation):
        G.SolverConfig(nev=4, lanczos_steps=1)
    with pytest.raises(G.ContractViolation):
        G.SolverConfig(nev=4, buffer=0)
    with pytest.raises(G.ContractViolation):
        G.SolverConfig(nev=4, max_outer_iters=0)
    with pytest.raises(G.ContractViolation):
        G.SolverConfig(nev=4, interval="weird")
    assert G.SolverConfig(nev=35).buffer_cols == 4
    assert G.SolverConfig(nev=4).buffer_cols == 1
    assert G.SolverConfig(nev=4, buffer=3).buffer_cols == 3


def test_filter_spec_validation():
    G.FilterSpec(degree=1, a=0.0, b=1.0, lam_ref=-1.0)
    with pytest.raises(G.ContractViolation):
        G.FilterSpec(degree=0, a=0.0, b=1.0, lam_ref=-1.0)
    with pytest.raises(G.ContractViolation):
        G.FilterSpec(degree=3, a=1.0, b=1.0, lam_ref=0.0)


def test_foreign_config_is_accepted_by_fields():
    from paper_1305_5120_b200.core import _as_config

    class RefLike:
        nev, tol, max_outer_iters, degree, lanczos_steps, buffer = 7, 1e-9, 11, 5, 4, 2

    cfg = _as_config(RefLike())
    assert (cfg.nev, cfg.tol, cfg.max_outer_iters, cfg.degree, cfg.buffer_cols) == (7, 1e-9, 11, 5, 2)
    with pytest.raises(G.ContractViolation):
        _as_config("not a config")


def test_error_attributes():
    assert G.NotPositiveDefinite(3).pivot == 3
    assert G.RankDeficient(2).column == 2
    e = G.NotConverged("m", np.zeros(1), np.zeros((2, 1)), "rep")
    assert e.report == "rep" and e.eigenvalues.shape == (1,)
    assert issubclass(G.DimensionMismatch, G.ContractViolation)
    assert issubclass(G.FilterDegenerate, G.ChfsiError)


def test_report_properties():
    r = G.SolveReport(n=3, nev=1)
    r.iterations.append(G.IterationStat(1, 4, 1, 0.0, 0.0, 84, 0.1, 0, 0, 0))
    r.iterations.append(G.IterationStat(2, 3, 2, 0.0, 0.0, 63, 0.1, 0, 0, 0))
    assert r.outer_iterations == 2
    assert r.converged_counts == [1, 2]


def test_baseline_spectrum_recipe():
    rng = np.random.default_rng(0)
    lam = W.baseline_spectrum(rng, 1000)
    assert np.all(np.diff(lam) >= 0)
    assert np.sum(lam < 0.5) == 200 and lam[0] >= -1.0 and lam[199] <= 0.0
    assert lam[200] >= 1.0 and lam[-1] <= 100.0


def test_baseline_matrix_has_exact_spectrum():
    h, lam, q = W.baseline_matrix(7, 120)
    assert np.allclose(np.linalg.eigvalsh(h), lam, atol=1e-12 * 100)
    assert np.array_equal(h, h.conj().T)


def test_baseline_sequence_perturbation_scale():
    probs = W.baseline_sequence(1, 80, 3)
    h1 = probs[0][0]
    delta = 1e-3 * np.max(np.abs(np.linalg.eigvalsh(h1)))
    d = np.linalg.norm(probs[1][0] - probs[0][0], 2)
    assert abs(d - delta) <= 1e-9 * delta
    gen = W.baseline_sequence(1, 40, 2, generalized=True)
    s = gen[0][1]
    w = np.linalg.eigvalsh(s)
    assert w[0] >= 1.0 - 1e-12 and w[-1] <= 1.1 + 1e-12


def test_workload_table():
    w = W.workload("c4")
    assert (w.n, w.nev, w.nex, w.degree, w.k, w.generalized) == (20000, 2000, 200, 25, 2200, True)
    w = W.workload("c0", n=500)
    assert (w.n, w.nev, w.nex) == (500, 50, 10)


def test_sequence_spec_validation():
    G.SequenceSpec(n=10, N=1, nev=2)
    for bad in (dict(n=10, N=0, nev=2), dict(n=10, N=2, nev=2, rho=1.0),
                dict(n=10, N=2, nev=2, delta0=-0.1), dict(n=10, N=2, nev=10),
                dict(n=10, N=2, nev=2, kind="banded"), dict(n=10, N=2, nev=2, spread=5.0)):
        with pytest.raises(G.ContractViolation):
            G.SequenceSpec(**bad)


def test_vector_angles_and_subspace_angle():
    rng = np.random.default_rng(70)
    y = rng.standard_normal((8, 3)) + 1j * rng.standard_normal((8, 3))
    y /= np.linalg.norm(y, axis=0)
    assert np.allclose(G.vector_angles(y, y * np.exp(1j * np.array([0.3, 1.1, -2.0]))), 0.0, atol=1e-7)
    e = np.eye(8, dtype=complex)
    assert np.allclose(G.vector_angles(e[:, :2], e[:, 2:4]), np.pi / 2, atol=1e-12)
    # sine-based angle resolves tiny angles the arccos form cannot
    eps = 1e-11
    v = e[:, :2] + eps * e[:, 2:4]
    assert abs(G.subspace_angle(e[:, :2], v) - eps) <= 1e-3 * eps


def test_device_ptr_rejects_lazy_conj_views():
    """torch's conj() is a lazy bit over shared storage: the C ABI must never see it."""
    import torch
    from paper_1305_5120_b200 import device as D
    t = torch.randn((3, 4), dtype=torch.complex128)
    with pytest.raises(ValueError):
        D.ptr(t.conj())
    assert D.ptr(t.conj().resolve_conj()).value is not None
    assert D.ptr(None).value is None


def test_block_layout_roundtrip():
    """numpy F-order (n, k) <-> (k, n) column-major block, no transposition of values."""
    import torch
    from paper_1305_5120_b200 import device as D
    a = np.arange(12, dtype=np.complex128).reshape(4, 3) * (1 + 2j)
    t = D.to_device(a, torch.device("cpu"))
    assert tuple(t.shape) == (3, 4) and D.rows(t) == 4 and D.cols(t) == 3 and D.ld(t) == 4
    assert np.array_equal(t[1].numpy(), a[:, 1])
    back = D.to_host(t)
    assert back.flags.f_contiguous and np.array_equal(back, a)


def test_report_csv_schema():
    from paper_1305_5120_b200 import report as R
    rep = G.SolveReport(n=10, nev=2)
    rep.iterations.append(G.IterationStat(1, 3, 1, 1.5e-3, 2e-11, 63, 0.01, 0.002, 0.003, 0.0))
    rep.iterations.append(G.IterationStat(2, 2, 2, 0.0, 0.0, 42, 0.01, 0.002, 0.003, 0.0))
    txt = R.report_csv_text(rep)
    lines = txt.strip().split("\n")
    assert lines[0] == "iter,filtered_cols,converged,max_resid,matmul_count,t_filter,t_qr,t_rr,t_resid"
    assert lines[1].startswith("1,3,1,1.500000e-03,63,")
    rows = R.phase_rows(rep, total_seconds=0.1, config_hash="abc")
    assert [r[0] for r in rows] == ["filter", "qr", "rayleigh_ritz", "residuals", "other"]
    assert abs(sum(float(r[2]) for r in rows) - 1.0) < 1e-5
    a = G.SequenceReport(mode="random", work=[10, 20], angles=[None, np.array([1e-3])])
    b = G.SequenceReport(mode="reuse", work=[10, 10], angles=[None, np.array([1e-4])])
    ratios = G.attach_work_ratios(a, b)
    seq = R.sequence_csv_text(a, b, ratios).strip().split("\n")
    assert seq[0] == "cycle,work_random,work_reuse,work_ratio,median_angle"
    assert seq[1] == "1,10,10,," and seq[2] == "2,20,10,2.0000,1.000000e-04"


def test_attach_work_ratios():
    a = G.SequenceReport(mode="random", work=[10, 20, 30])
    b = G.SequenceReport(mode="reuse", work=[10, 10, 10])
    assert G.attach_work_ratios(a, b) == [None, 2.0, 3.0]
    with pytest.raises(G.ContractViolation):
        G.attach_work_ratios(a, G.SequenceReport(mode="reuse", work=[1]))
