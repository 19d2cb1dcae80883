"""Multi-GPU plumbing beyond the column shards (SURVEY.md sections 8b, 8e):

* the communicator layer (comm.py): torch.distributed groups and in-process
  thread cliques behind one interface;
* the cross-rank consistency guard on the replicated k x k decisions
  (distributed.ShardedPhases.agree / the fingerprints riding on the residual
  gather): a rank whose Gram differs by one ulp makes EVERY rank raise
  ChfsiError -- no hang, no silent divergence;
* the multi-GPU sequence driver (solve_sequence(group=) / (devices=)) against
  the single-GPU sequence (reference sequence.py:165-228);
* bench.py --gpus N starting its own N ranks.

CPU tests use gloo (world 2, 127.0.0.1) or CPU tensors in a thread clique; the
gpu-marked tests put two ranks on cuda:0 (gloo host staging, or the in-process
"local" clique) -- kernels of different ranks never wait on each other."""

import json
import os
import socket
import subprocess
import sys
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


# ------------------------------------------------------------------ CPU
def test_fingerprint_and_agreement():
    from paper_1305_5120_b200.distributed import check_agreement, fingerprint
    from paper_1305_5120_b200.errors import ChfsiError
    a = np.linspace(-1.0, 3.0, 17)
    b = a.copy()
    assert fingerprint(a) == fingerprint(b)
    b[5] = np.nextafter(b[5], np.inf)  # one ulp
    assert fingerprint(a) != fingerprint(b)
    assert float(int(fingerprint(a))) == fingerprint(a) < 2.0 ** 48
    check_agreement(np.array([[1.0, 2.0], [1.0, 2.0]]), "same")
    with pytest.raises(ChfsiError, match="cross-rank divergence in x"):
        check_agreement(np.array([[1.0, 2.0], [1.0, np.nextafter(2.0, 3.0)]]), "x")


def test_thread_clique_local_collectives_cpu():
    """ThreadComm ("local" backend) on CPU tensors: all-gather in rank order, broadcast
    from a root, barrier; an aborted clique raises instead of hanging."""
    from paper_1305_5120_b200.comm import ThreadComm, _Clique
    world = 3
    clique = _Clique([0] * world, "local")
    got = [None] * world
    errs = []

    def body(r):
        try:
            c = ThreadComm(clique, r)
            inp = torch.full((2, 3), float(r), dtype=torch.float64)
            out = torch.empty((world * 2, 3), dtype=torch.float64)
            c.all_gather_into_tensor(out, inp)
            t = torch.full((4,), float(10 + r), dtype=torch.float64)
            c.broadcast(t, src=1)
            c.barrier()
            got[r] = (out.clone(), t.clone())
        except Exception as exc:  # pragma: no cover - surfaced below
            errs.append(exc)

    ths = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=60)
    assert not errs, errs
    for r in range(world):
        out, t = got[r]
        assert torch.equal(out, torch.arange(world, dtype=torch.float64).repeat_interleave(2)
                           .reshape(-1, 1).expand(-1, 3))
        assert torch.equal(t, torch.full((4,), 11.0, dtype=torch.float64))
    from paper_1305_5120_b200.errors import ChfsiError
    clique2 = _Clique([0, 0], "local")
    clique2.abort()
    with pytest.raises(ChfsiError, match="aborted"):
        ThreadComm(clique2, 0).barrier()


def test_device_list_normalisation_and_default():
    from paper_1305_5120_b200 import comm
    assert comm.normalize_devices(3) == [0, 1, 2]
    assert comm.normalize_devices([2, 5]) == [2, 5]
    assert comm.choose_backend([0, 1]) == "nccl" and comm.choose_backend([0, 0]) == "local"
    with pytest.raises(ValueError):
        comm.normalize_devices(0)
    comm.set_devices(4)
    try:
        assert comm.get_devices() == [0, 1, 2, 3] and comm.default_devices() == [0, 1, 2, 3]
        with comm.inside_group():
            assert comm.default_devices() is None
    finally:
        comm.set_devices(None)
    assert comm.default_devices() is None


def _agree_worker(rank, world, port, out_dir):
    _init(rank, world, port)
    from paper_1305_5120_b200.distributed import ShardedPhases
    from paper_1305_5120_b200.errors import ChfsiError
    try:
        ph = ShardedPhases(dist.group.WORLD)
        like = torch.zeros(1, dtype=torch.float64)
        ph.agree("same", [1.0, 2.5], like)
        try:
            ph.agree("Ritz values", [1.0, 2.5 if rank == 0 else np.nextafter(2.5, 3.0)], like)
            res = "no error"
        except ChfsiError as exc:
            res = str(exc)
        with open(os.path.join(out_dir, f"a{rank}.txt"), "w") as f:
            f.write(res)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_agreement_guard_raises_on_every_rank(tmp_path):
    mp.spawn(_agree_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        msg = (tmp_path / f"a{r}.txt").read_text()
        assert "cross-rank divergence in Ritz values" in msg, msg


def test_layout_checks_reject_strided_blocks():
    from paper_1305_5120_b200 import device as D
    t = torch.zeros((4, 6), dtype=torch.complex128)
    assert D.ld(t) == 6 and D.ld(t[1:3]) == 6
    with pytest.raises(ValueError, match="row stride"):
        D.ld(t.t())
    with pytest.raises(ValueError, match="row stride"):
        D.ptr(t[:, ::2])
    assert D.ld(t[2:3]) == 6


def test_bench_launcher_argv():
    import bench
    argv = bench.launcher_argv(["--gpus", "4", "--steps", "2"], 4)
    assert argv[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in argv and "--master-addr=127.0.0.1" in argv
    assert argv[-4:] == ["--gpus", "4", "--steps", "2"]
    assert argv[-5].endswith("bench.py")


def test_bench_reference_arm_self_launches_n_ranks():
    """`bench.py --impl reference --gpus 2` without a launcher starts 2 ranks itself
    (torch.distributed.run); rank 0 alone prints the line, with n_gpus = 2."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
         "--steps", "1", "--warmup", "1", "--matrix-order", "300", "--block-cols", "40"],
        capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2


def test_bench_refuses_world_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
         "--steps", "1", "--warmup", "1", "--matrix-order", "200", "--block-cols", "20"],
        capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr


# ------------------------------------------------------------------ GPU
def _seq_problems(n=240, nprob=3):
    from paper_1305_5120_b200.workloads import baseline_sequence
    return baseline_sequence(8, n, nprob, generalized=True)


def _seq_cfg():
    import paper_1305_5120_b200 as G
    return G.SolverConfig(nev=24, buffer=6, degree=15, max_outer_iters=5000)


def _single_sequence():
    import paper_1305_5120_b200 as G
    probs = _seq_problems()
    seq = G.ProblemSequence(spec=G.SequenceSpec(n=240, N=3, nev=24, seed=8),
                            problems=[(a, s) for a, s in probs])
    return G.solve_sequence(seq, _seq_cfg(), "reuse", angles=False)


def _sharded_sequence(rank, world, port, out_dir):
    _init(rank, world, port)
    import paper_1305_5120_b200 as G
    try:
        torch.cuda.set_device(0)
        probs = _seq_problems()
        seq = G.ProblemSequence(spec=G.SequenceSpec(n=240, N=3, nev=24, seed=8),
                                problems=[(a, s) for a, s in probs])
        rep = G.solve_sequence(seq, _seq_cfg(), "reuse", angles=False, group=dist.group.WORLD)
        d = {}
        for i, (lam, v, r) in enumerate(zip(rep.eigenvalues, rep.vectors, rep.reports)):
            d[f"lam{i}"], d[f"v{i}"], d[f"it{i}"] = lam, v.entries, r.outer_iterations
        np.savez(os.path.join(out_dir, f"s{rank}.npz"), **d)
    finally:
        dist.destroy_process_group()


def _compare_sequences(got, ref, exact_iters=False):
    import oracle.chfsi_oracle as O
    for i in range(3):
        lam_ref = ref.eigenvalues[i]
        assert np.max(np.abs(got[f"lam{i}"] - lam_ref) / np.abs(lam_ref)) <= 1e-10, i
        assert O.largest_angle_sine(got[f"v{i}"], ref.vectors[i].entries) < 1e-8, i
        if exact_iters:
            assert int(got[f"it{i}"]) == ref.reports[i].outer_iterations


@pytest.mark.gpu
def test_gloo_world2_generalized_sequence_matches_single(tmp_path):
    """solve_sequence(..., group=) over 2 ranks (3 generalized c2-recipe problems, reuse):
    both ranks agree bit for bit and equal the single-GPU sequence (eigenvalues 1e-10,
    sine angle 1e-8)."""
    mp.spawn(_sharded_sequence, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    s0, s1 = np.load(tmp_path / "s0.npz"), np.load(tmp_path / "s1.npz")
    for i in range(3):
        assert np.array_equal(s0[f"lam{i}"], s1[f"lam{i}"])
        assert np.array_equal(s0[f"v{i}"], s1[f"v{i}"])
    _compare_sequences(s0, _single_sequence())


@pytest.mark.gpu
def test_in_process_sequence_two_ranks_matches_single():
    """solve_sequence(..., devices=[0, 0]): two rank threads in this process (the
    host-synchronised local clique, both on cuda:0) equal the single-GPU sequence."""
    import paper_1305_5120_b200 as G
    probs = _seq_problems()
    seq = G.ProblemSequence(spec=G.SequenceSpec(n=240, N=3, nev=24, seed=8),
                            problems=[(G.HermitianDenseMatrix(a), G.HermitianDenseMatrix(s))
                                      for a, s in probs])
    G.reset_product_count()
    rep = G.solve_sequence(seq, _seq_cfg(), "reuse", angles=False, devices=[0, 0])
    count = G.product_count()
    got = {}
    for i, (lam, v, r) in enumerate(zip(rep.eigenvalues, rep.vectors, rep.reports)):
        got[f"lam{i}"], got[f"v{i}"], got[f"it{i}"] = lam, v.entries, r.outer_iterations
    G.reset_product_count()
    ref = _single_sequence()
    _compare_sequences(got, ref)
    # the work is counted once (rank 0), as by the single-GPU run
    assert count == sum(ref.work)


@pytest.mark.gpu
def test_in_process_solve_two_ranks_and_default_devices():
    import oracle.chfsi_oracle as O
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.workloads import baseline_matrix
    h, lam_true, _ = baseline_matrix(21, 300)
    cfg = G.SolverConfig(nev=30, buffer=6, degree=15, max_outer_iters=3000)
    lam1, v1, rep1 = G.chfsi_solve(h, None, cfg, seed=5)
    lam2, v2, rep2 = G.chfsi_solve(h, None, cfg, seed=5, devices=[0, 0])
    assert np.max(np.abs(lam2 - lam1) / np.abs(lam1)) <= 1e-10
    assert O.largest_angle_sine(v2.entries, v1.entries) < 1e-8
    assert rep2.total_matmuls == rep1.total_matmuls or \
        abs(rep2.outer_iterations - rep1.outer_iterations) <= 3
    # the drop-in call unchanged, the GPU set from set_devices (CHFSI_DEVICES)
    G.set_devices([0, 0])
    try:
        rng = np.random.default_rng(5)
        lam3, v3, _ = G.chfsi_solve(h, None, cfg, seed=rng)
    finally:
        G.set_devices(None)
    assert np.array_equal(lam3, lam2)
    # the caller's Generator advanced as after a one-GPU solve
    rng_ref = np.random.default_rng(5)
    G.chfsi_solve(h, None, cfg, seed=rng_ref)
    assert rng.bit_generator.state == rng_ref.bit_generator.state


@pytest.mark.gpu
def test_in_process_solve_eight_ranks_ragged_and_empty_shards():
    """The north star's rank count: 8 rank threads (sharing cuda:0 here) on a problem whose
    active block shrinks below 8 columns before it converges (nev + nex = 13: shards of 2
    and 1 columns from the start, empty shards at the end), standard and generalized."""
    import oracle.chfsi_oracle as O
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.workloads import baseline_matrix
    h, lam_true, _ = baseline_matrix(31, 200)
    cfg = G.SolverConfig(nev=10, buffer=3, degree=12, max_outer_iters=4000)
    lam1, v1, rep1 = G.chfsi_solve(h, None, cfg, seed=7)
    lam8, v8, rep8 = G.chfsi_solve(h, None, cfg, seed=7, devices=[0] * 8)
    assert rep8.converged and rep1.converged and len(lam8) == len(lam1) == cfg.nev
    assert np.max(np.abs(lam8 - lam1) / np.abs(lam1)) <= 1e-10
    assert O.largest_angle_sine(v8.entries, v1.entries) < 1e-8
    assert float(G.residuals(h, v8, lam8).max()) < cfg.tol
    rng = np.random.default_rng(3)
    b = rng.standard_normal((200, 200)) + 1j * rng.standard_normal((200, 200))
    b = np.eye(200) + 0.1 * (b.conj().T @ b) / np.linalg.norm(b.conj().T @ b, 2)
    g1, c1, _ = G.solve_generalized(h, b, None, cfg, seed=7)
    g8, c8, _ = G.solve_generalized(h, b, None, cfg, seed=7, devices=[0] * 8)
    assert np.max(np.abs(g8 - g1) / np.abs(g1)) <= 1e-10
    gram = c8.entries.conj().T @ b @ c8.entries
    assert np.linalg.norm(gram - np.eye(cfg.nev)) <= 1e-9


@pytest.mark.gpu
def test_in_process_guard_fails_cleanly_on_divergent_rank():
    """Fault injection: rank 1's gathered Rayleigh-Ritz Gram gets a one-ulp change.
    Every rank must raise ChfsiError (cross-rank divergence), not hang."""
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200 import distributed as Dd
    from paper_1305_5120_b200.workloads import baseline_matrix
    h, _, _ = baseline_matrix(21, 300)
    cfg = G.SolverConfig(nev=30, buffer=6, degree=15, max_outer_iters=3000)

    def bump(W):
        v = torch.view_as_real(W)
        v[0, 0, 0] = float(np.nextafter(float(v[0, 0, 0]), np.inf))

    Dd.TEST_HOOKS["perturb_gram"] = (1, bump)
    try:
        result = {}

        def run():
            try:
                G.chfsi_solve(h, None, cfg, seed=5, devices=[0, 0])
                result["err"] = None
            except Exception as exc:  # noqa: BLE001
                result["err"] = exc

        t = threading.Thread(target=run)
        t.start()
        t.join(timeout=300)
        assert not t.is_alive(), "sharded solve hung after a divergent rank"
    finally:
        Dd.TEST_HOOKS.clear()
    assert isinstance(result["err"], G.ChfsiError), result["err"]
    assert "cross-rank divergence" in str(result["err"])


def _perturbed_solver(rank, world, port, out_dir):
    _init(rank, world, port)
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200 import distributed as Dd
    from paper_1305_5120_b200.workloads import baseline_matrix
    try:
        torch.cuda.set_device(0)

        def bump(W):
            v = torch.view_as_real(W)
            v[0, 0, 0] = float(np.nextafter(float(v[0, 0, 0]), np.inf))

        Dd.TEST_HOOKS["perturb_gram"] = (1, bump)
        h, _, _ = baseline_matrix(21, 300)
        cfg = G.SolverConfig(nev=30, buffer=6, degree=15, max_outer_iters=3000)
        try:
            G.chfsi_solve(h, None, cfg, seed=5, group=dist.group.WORLD)
            msg = "no error"
        except G.ChfsiError as exc:
            msg = str(exc)
        with open(os.path.join(out_dir, f"p{rank}.txt"), "w") as f:
            f.write(msg)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_world2_guard_fails_cleanly_on_divergent_rank(tmp_path):
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_perturbed_solver, args=(r, 2, port, str(tmp_path)))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    alive = [p.is_alive() for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert not any(alive), "a rank hung after the divergence"
    for r in range(2):
        msg = (tmp_path / f"p{r}.txt").read_text()
        assert "cross-rank divergence" in msg, msg


@pytest.mark.gpu
def test_nccl_clique_single_device_allgather():
    """The native NCCL clique (csrc/comm.cu, dlopen'ed libnccl) on the one GPU of the
    box: a world-1 clique all-gathers and broadcasts in place; duplicate devices are
    refused (they take the local clique instead)."""
    import ctypes
    from paper_1305_5120_b200 import _native
    from paper_1305_5120_b200.comm import ThreadComm, _Clique
    ver = ctypes.c_int(0)
    assert _native.load().chfsi_comm_available(ctypes.byref(ver)) == 1 and ver.value > 0
    torch.cuda.set_device(0)
    cl = _Clique([0], "nccl")
    try:
        c = ThreadComm(cl, 0)
        x = torch.arange(10, dtype=torch.float64, device="cuda")
        out = torch.empty(10, dtype=torch.float64, device="cuda")
        c.all_gather_into_tensor(out, x)
        c.broadcast(x, 0)
        torch.cuda.synchronize()
        assert torch.equal(out, x)
    finally:
        cl.close()
    devs = (ctypes.c_int * 2)(0, 0)
    hs = (ctypes.c_void_p * 2)()
    assert _native.load().chfsi_comm_init_all(2, devs, hs) != 0
    assert "distinct" in _native.last_error()


@pytest.mark.gpu
def test_bench_gpus2_self_launch_prints_n_gpus():
    """`python bench.py --gpus 2 --dist-backend gloo ...` with no launcher runs 2 ranks
    (sharing cuda:0 in gloo test mode) and reports n_gpus = 2."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo",
         "--matrix-order", "4096", "--block-cols", "440", "--degree", "10", "--steps", "3",
         "--warmup", "3", "--no-extras"],
        capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0


@pytest.mark.gpu
def test_bench_nccl_refuses_more_gpus_than_visible():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    n = torch.cuda.device_count() + 1
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--no-extras"],
        capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "visible GPUs" in out.stderr


@pytest.mark.gpu
def test_in_process_clique_is_reused_and_replaced_after_abort():
    """run_on_devices keeps the clique of a device set for the next call (NCCL
    communicator setup costs more than a small solve); a clique aborted by a failing
    rank is dropped and the next call gets a fresh one."""
    from paper_1305_5120_b200 import comm
    comm.release_devices()
    out1 = comm.run_on_devices([0, 0], lambda c: c.rank)
    c1 = comm._cliques[((0, 0), "local")]
    out2 = comm.run_on_devices([0, 0], lambda c: c.world)
    assert out1 == [0, 1] and out2 == [2, 2]
    assert comm._cliques[((0, 0), "local")] is c1 and not c1.broken

    def fail(c):
        if c.rank == 1:
            raise RuntimeError("rank 1 fails")
        c.barrier()  # rank 0 waits for rank 1: must be released by the abort

    with pytest.raises(RuntimeError, match="rank 1 fails"):
        comm.run_on_devices([0, 0], fail)
    assert ((0, 0), "local") not in comm._cliques and c1.broken
    assert comm.run_on_devices([0, 0], lambda c: c.rank) == [0, 1]
    comm.release_devices()
    assert not comm._cliques
