"""Sequence driver parity (reference sequence.py) on the GPU: the restated synthetic
generator reproduces the reference's matrices, and the reuse/random work of the
reference's acceptance preset (criterion 3, test_acceptance.py:27-38, 90-104) is
reproduced. Fixtures: tests/golden/reference_sequences.npz (written by the reference)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold():
    return np.load(os.path.join(GOLD, "reference_sequences.npz"))


def test_generate_sequence_matches_reference_generator():
    import paper_1305_5120_b200 as G
    g = gold()
    spec = G.SequenceSpec(n=30, N=3, nev=4, seed=21, kind="generalized", vary_b=True)
    seq = G.generate_sequence(spec)
    for i, (a, b) in enumerate(seq.problems):
        for got, ref in ((a.entries, g[f"a{i}"]), (b.entries, g[f"b{i}"])):
            assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_acceptance_preset_reuse_work_matches_reference():
    """Criterion 3 preset: n=500, N=13, nev=35, delta0=0.1, rho=0.5, seed=11."""
    import paper_1305_5120_b200 as G
    g = gold()
    spec = G.SequenceSpec(n=500, N=13, nev=35, delta0=0.1, rho=0.5, seed=11)
    seq = G.generate_sequence(spec)
    cfg = G.SolverConfig(nev=35)
    rand = G.solve_sequence(seq, cfg, "random")
    reuse = G.solve_sequence(seq, cfg, "reuse")
    ratios = G.attach_work_ratios(rand, reuse)
    tail = -(-len(ratios) // 3)
    assert all(r >= 2.0 for r in ratios[-tail:]), ratios
    assert all(r >= 1.0 for r in ratios[1:]), ratios
    # per-cycle work equals the reference's (iteration counts agree; allow one
    # rounding-induced lock shift per cycle)
    for mine, ref, name in ((rand.work, g["preset_work_random"], "random"),
                            (reuse.work, g["preset_work_reuse"], "reuse")):
        mine = np.array(mine)
        assert np.max(np.abs(mine - ref) / ref) <= 0.05, (name, mine, ref)
    lam_ref = g["preset_lam_last"]
    assert np.max(np.abs(reuse.eigenvalues[-1] - lam_ref) / np.abs(lam_ref)) <= 1e-10


def test_delta0_zero_reuse_hits_fixed_point():
    """Reference test_sequence.py:93-102: with no perturbation every reused cycle
    converges in one outer iteration."""
    import paper_1305_5120_b200 as G
    spec = G.SequenceSpec(n=96, N=4, nev=10, delta0=0.0, seed=9)
    seq = G.generate_sequence(spec)
    rep = G.solve_sequence(seq, G.SolverConfig(nev=10), "reuse")
    assert all(r.outer_iterations == 1 for r in rep.reports[1:])
    for lam in rep.eigenvalues[1:]:
        assert np.max(np.abs(lam - rep.eigenvalues[0])) <= 1e-10
    for med in rep.median_angles()[1:]:
        assert med <= 1e-7


def test_generalized_sequence_reuse_stays_b_orthonormal():
    import paper_1305_5120_b200 as G
    spec = G.SequenceSpec(n=64, N=3, nev=6, seed=17, kind="generalized")
    seq = G.generate_sequence(spec)
    cfg = G.SolverConfig(nev=6)
    rand = G.solve_sequence(seq, cfg, "random")
    reuse = G.solve_sequence(seq, cfg, "reuse")
    ratios = G.attach_work_ratios(rand, reuse)
    assert all(r >= 1.0 for r in ratios[1:])
    for (_, b), v in zip(seq.problems, reuse.vectors):
        gram = v.entries.conj().T @ b.entries @ v.entries
        assert np.linalg.norm(gram - np.eye(6)) <= 1e-9


def test_not_converged_aborts_with_partial_sequence_report():
    import paper_1305_5120_b200 as G
    spec = G.SequenceSpec(n=96, N=3, nev=10, seed=16)
    seq = G.generate_sequence(spec)
    cfg = G.SolverConfig(nev=10, degree=1, max_outer_iters=1)
    with pytest.raises(G.NotConverged) as exc:
        G.solve_sequence(seq, cfg, "random")
    assert isinstance(exc.value.report, G.SequenceReport)
    assert len(exc.value.report.reports) < 3
