"""Multi-process (world_size 2, gloo, 127.0.0.1) tests of the column-sharding plumbing
(distributed.ColumnShards / all_gather_values) and of sharded filtering semantics
(SURVEY.md section 8e): filtering each rank's contiguous column shard and gathering
equals filtering the whole block, because core.py:276-283 is column-separable.

The CPU tests use the oracle's filter as the per-rank compute (tests may import the
oracle); the gpu-marked test runs the real sharded solver (2 ranks on cuda:0, gloo
staging through the host; kernels never wait on each other)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    import sys
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _plumbing(rank, world, port):
    _init(rank, world, port)
    from paper_1305_5120_b200.distributed import ColumnShards, all_gather_values
    try:
        for k, n in ((7, 5), (1, 3), (8, 4), (0, 2)):
            g = torch.Generator().manual_seed(k * 10 + n)
            full = torch.randn((k, n), dtype=torch.complex128, generator=g)
            sh = ColumnShards(k, world)
            lo, hi = sh.range(rank)
            got = sh.gather_block(full[lo:hi].clone())
            assert torch.equal(got, full), (k, n)
            vals = torch.arange(k, dtype=torch.float64) * 1.5
            v = all_gather_values(vals[lo:hi].clone(), sh)
            assert torch.equal(v, vals)
        # the reference's worker bounds (linalg.py:238-243)
        sh = ColumnShards(2200, 8)
        assert sh.bounds == [(2200 * i) // 8 for i in range(9)]
    finally:
        dist.destroy_process_group()


def _sharded_filter(rank, world, port):
    _init(rank, world, port)
    import oracle.chfsi_oracle as O
    from paper_1305_5120_b200.distributed import ColumnShards
    from paper_1305_5120_b200.workloads import baseline_matrix
    try:
        h, lam, _ = baseline_matrix(4, 160)
        rng = np.random.default_rng(9)
        y = rng.standard_normal((160, 13)) + 1j * rng.standard_normal((160, 13))
        a, b, lr = float(lam[16]), float(lam[-1]) * 1.1, float(lam[0])
        sh = ColumnShards(13, world)
        lo, hi = sh.range(rank)
        mine = O.cheb_filter(h, y[:, lo:hi], 12, a, b, lr)
        block = torch.from_numpy(np.ascontiguousarray(mine.T))  # (cols, rows)
        got = sh.gather_block(block).numpy().T
        ref = O.cheb_filter(h, y, 12, a, b, lr)
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    finally:
        dist.destroy_process_group()


def test_column_shards_single_process():
    from paper_1305_5120_b200.distributed import ColumnShards
    sh = ColumnShards(10, 3)
    assert sh.bounds == [0, 3, 6, 10]
    assert sh.widths == [3, 3, 4] and sh.padded == 4
    assert [sh.owner(c) for c in range(10)] == [0, 0, 0, 1, 1, 1, 2, 2, 2, 2]
    with pytest.raises(ValueError):
        ColumnShards(-1, 2)


def test_gloo_world2_gather_plumbing():
    mp.spawn(_plumbing, args=(2, _free_port()), nprocs=2, join=True)


def test_gloo_world2_sharded_filter_equals_full():
    mp.spawn(_sharded_filter, args=(2, _free_port()), nprocs=2, join=True)


def _sharded_solver(rank, world, port, out_dir):
    _init(rank, world, port)
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.workloads import baseline_matrix
    try:
        torch.cuda.set_device(0)
        h, lam_true, _ = baseline_matrix(21, 300)
        cfg = G.SolverConfig(nev=30, buffer=6, degree=15, max_outer_iters=3000)
        lam, v, rep = G.chfsi_solve(h, None, cfg, seed=5, group=dist.group.WORLD)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), lam=lam, v=v.entries,
                 iters=rep.outer_iterations)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_world2_sharded_solver_matches_single(tmp_path):
    import oracle.chfsi_oracle as O
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.workloads import baseline_matrix
    mp.spawn(_sharded_solver, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    # every rank reached the same result (identical gathered block -> identical decisions)
    assert np.array_equal(r0["lam"], r1["lam"]) and int(r0["iters"]) == int(r1["iters"])
    h, lam_true, _ = baseline_matrix(21, 300)
    cfg = G.SolverConfig(nev=30, buffer=6, degree=15, max_outer_iters=3000)
    lam, v, rep = G.chfsi_solve(h, None, cfg, seed=5)
    assert np.max(np.abs(r0["lam"] - lam) / np.abs(lam)) <= 1e-10
    assert O.largest_angle_sine(r0["v"], v.entries) < 1e-8
    assert np.max(np.abs(r0["lam"] - lam_true[:30]) / np.abs(lam_true[:30])) <= 1e-10
