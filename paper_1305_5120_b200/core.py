"""ChFSI solver on the B200, behind the reference's chfsi.core API
(reference pkg/src/chfsi/core.py:59-569).

The outer loop (locking, interval updates, RNG order, report, errors) is
restated here line for line from core.py:385-546 so traces stay comparable
with the reference; every n x n x k product, the QR, the Rayleigh-Ritz
projection and the residual norms run as CUDA kernels in libchfsi_b200.so on
device-resident blocks. Per outer iteration the host sees only the k Ritz
values, k residuals and (for the rank test) k diagonal entries.

Buffers (all column-major complex128, n x (nev+buffer)): two filter blocks,
HQ, Z, HZ, plus the locked block (n x nev); H stays resident.
"""

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import device as dev
from .errors import ContractViolation, FilterDegenerate, NotConverged, RankDeficient
from .linalg import (
    HermitianDenseMatrix,
    LowerTriangularFactor,
    VectorBlock,
    _count_products,
    cholesky_factor,
    default_device,
    engine,
    solve_triangular_device,
    to_block,
)

__all__ = [
    "FilterSpec", "SolverConfig", "SolveReport", "IterationStat", "reduce_to_standard",
    "back_transform", "lanczos_upper_bound", "chebyshev_filter", "rayleigh_ritz",
    "residuals", "chfsi_solve", "solve_generalized",
]


# ----------------------------------------------------------------------
# configuration and reporting types (core.py:59-165)


@dataclass(frozen=True)
class FilterSpec:
    """Chebyshev filter parameters (core.py:59-79)."""

    degree: int
    a: float
    b: float
    lam_ref: float

    def __post_init__(self):
        if self.degree < 1:
            raise ContractViolation(f"filter degree must be >= 1, got {self.degree}")
        if not self.a < self.b:
            raise ContractViolation(f"filter interval requires a < b, got a={self.a}, b={self.b}")


@dataclass(frozen=True)
class SolverConfig:
    """Solver knobs (core.py:82-115). ``interval`` is a B200-build extension:
    "reference" (default) puts the filter's lower edge at Ritz value nev+1
    exactly like core.py:507-509; "block_top" puts it at the largest Ritz value
    of the search block (ChASE-style, SURVEY.md section 7 ii), opt-in only."""

    nev: int
    tol: float = 1e-10
    max_outer_iters: int = 30
    degree: int = 20
    lanczos_steps: int = 10
    buffer: int | None = None
    interval: str = "reference"

    def __post_init__(self):
        if self.nev < 1:
            raise ContractViolation(f"nev must be >= 1, got {self.nev}")
        if not self.tol > 0:
            raise ContractViolation(f"tol must be > 0, got {self.tol}")
        if self.max_outer_iters < 1:
            raise ContractViolation("max_outer_iters must be >= 1")
        if self.degree < 1:
            raise ContractViolation("degree must be >= 1")
        if self.lanczos_steps < 2:
            raise ContractViolation("lanczos_steps must be >= 2")
        if self.buffer is not None and self.buffer < 1:
            raise ContractViolation("buffer must be >= 1 when given")
        if self.interval not in ("reference", "block_top"):
            raise ContractViolation(f"unknown interval placement {self.interval!r}")

    @property
    def buffer_cols(self):
        if self.buffer is not None:
            return self.buffer
        return max(1, math.ceil(0.1 * self.nev))


def _as_config(config):
    """Accept our SolverConfig or any object with the reference's fields
    (e.g. the reference's own chfsi.core.SolverConfig, core.py:402-403)."""
    if isinstance(config, SolverConfig):
        return config
    fields = ("nev", "tol", "max_outer_iters", "degree", "lanczos_steps", "buffer")
    if all(hasattr(config, f) for f in fields):
        return SolverConfig(**{f: getattr(config, f) for f in fields})
    raise ContractViolation("config must be a SolverConfig")


@dataclass
class IterationStat:
    """Per-outer-iteration statistics (core.py:118-131)."""

    iteration: int
    filtered_cols: int
    converged: int
    max_resid: float
    min_resid: float
    matmuls: int
    t_filter: float
    t_qr: float
    t_rr: float
    t_resid: float


@dataclass
class SolveReport:
    """Solve statistics (core.py:134-165)."""

    n: int = 0
    nev: int = 0
    iterations: list = field(default_factory=list)
    setup_matmuls: int = 0
    total_matmuls: int = 0
    upper_bound: float = 0.0
    est_lam1: float = 0.0
    est_lam_next: float = 0.0
    t_lanczos: float = 0.0
    t_filter: float = 0.0
    t_qr: float = 0.0
    t_rr: float = 0.0
    t_resid: float = 0.0
    t_total: float = 0.0
    converged: bool = False
    # B200 build: filter FLOPs actually executed (8 n^2 m sum filtered_cols)
    filter_flops: float = 0.0

    @property
    def outer_iterations(self):
        return len(self.iterations)

    @property
    def converged_counts(self):
        return [it.converged for it in self.iterations]

    @property
    def filter_tflops(self):
        return self.filter_flops / self.t_filter / 1e12 if self.t_filter > 0 else 0.0


# ----------------------------------------------------------------------
# helpers


def _rng(seed):
    return seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)


def _hermitian(H, device=None):
    """Device-resident Hermitian operator for H (no re-validation for wrappers)."""
    if isinstance(H, HermitianDenseMatrix):
        return H
    if hasattr(H, "entries") and not isinstance(H, (VectorBlock, LowerTriangularFactor)):
        H = H.entries  # e.g. the reference's own HermitianDenseMatrix
    a = np.asarray(H, dtype=np.complex128)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ContractViolation(f"expected a square matrix, got shape {a.shape}")
    # the reference uses a raw ndarray as is (core.py:404 `_asarray`): upload unchanged
    block = dev.to_device(a, device if device is not None else default_device())
    return HermitianDenseMatrix.from_device(block, trusted=True)


def _host_block(x):
    if isinstance(x, (VectorBlock, LowerTriangularFactor, HermitianDenseMatrix)):
        return x.entries
    if hasattr(x, "entries"):
        return np.asarray(x.entries, dtype=np.complex128)
    return np.asarray(x, dtype=np.complex128)


def _rand_cols(rng, n, s):
    return rng.standard_normal((n, s)) + 1j * rng.standard_normal((n, s))


# ----------------------------------------------------------------------
# reduction to standard form (core.py:172-195)


def reduce_to_standard(A, L):
    """H = L^-1 A L^-H, re-symmetrised (core.py:172-188): triangular inverse
    plus two DMMA GEMMs; the result stays on the device."""
    lfac = L if isinstance(L, LowerTriangularFactor) else LowerTriangularFactor(L)
    ab = A.device_block() if isinstance(A, HermitianDenseMatrix) else to_block(_host_block(A))
    if dev.rows(ab) != lfac.n:
        raise ContractViolation(f"order mismatch: A is {(dev.rows(ab), dev.cols(ab))}, "
                                f"L is {(lfac.n, lfac.n)}")
    return HermitianDenseMatrix(_reduce_block(ab, lfac), rtol=1e-8)


def _reduce_block(ab, lfac, linv=None):
    eng = engine(ab.device)
    n = dev.rows(ab)
    if linv is None:
        linv = dev.empty(n, n, ab.device)
        eng.trtri_lower(lfac.device_block(ab.device), linv)
    w = dev.empty(n, n, ab.device)
    h = dev.empty(n, n, ab.device)
    return eng.reduce_to_standard(ab, linv, w, h)


def back_transform(Y, L):
    """C = L^-H Y (core.py:191-195)."""
    yb = Y.device_block() if isinstance(Y, VectorBlock) else to_block(_host_block(Y))
    return VectorBlock(solve_triangular_device(L, yb, side="left", adjoint=True))


# ----------------------------------------------------------------------
# building blocks


def lanczos_upper_bound(H, k, seed=0):
    """Upper bound for lambda_max(H) from k Lanczos steps (core.py:202-256).
    The start vector is drawn from ``seed``'s Generator exactly like the
    reference; the k GEMVs, dots and reorthogonalisation run on the GPU."""
    k = int(k)
    if k < 2:
        raise ContractViolation(f"lanczos steps must be >= 2, got {k}")
    hm = _hermitian(H)
    rng = _rng(seed)
    return _lanczos(hm, k, rng)


def _lanczos(hm, k, rng):
    n = hm.n
    v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    v /= np.linalg.norm(v)
    hb = hm.device_block()
    vb = dev.to_device(v, hb.device)
    bound, _, _ = engine(hb.device).lanczos_bound(hb, vb, min(k, n))
    _count_products(min(k, n))
    return bound


def chebyshev_filter(H, Y, spec, *, group=None, devices=None):
    """p_m(H) Y with the scaled Chebyshev recurrence (core.py:287-311).

    ``group`` (keyword-only, B200 extension): a torch.distributed process group with
    one process per GPU. Every rank passes the same H and Y; a host H is uploaded as
    one column slab per rank and all-gathered over NVLink, each rank filters its
    contiguous column range of Y, and the filtered shards are all-gathered, so every
    rank returns the full p_m(H) Y. ``devices`` (keyword-only): the same over several
    GPUs of THIS process (an int N or CUDA ordinals; one thread per GPU, NCCL clique);
    the result lives on the first device."""
    if devices is None and group is None:
        devices = _default_devices()
    if devices is not None:
        return _in_process(devices, group, lambda comm, _rng: chebyshev_filter(
            _localize(H), _localize(Y), spec, group=comm), None)
    if not isinstance(spec, FilterSpec):
        if all(hasattr(spec, f) for f in ("degree", "a", "b", "lam_ref")):
            spec = FilterSpec(spec.degree, spec.a, spec.b, spec.lam_ref)
        else:
            raise ContractViolation("spec must be a FilterSpec")
    if spec.lam_ref >= spec.a:
        raise FilterDegenerate(
            f"lam_ref = {spec.lam_ref} lies inside the unwanted interval [{spec.a}, {spec.b}]; "
            f"wanted and unwanted intervals overlap (a larger buffer improves the "
            f"lambda_nev+1 estimate)")
    if group is not None:
        from .distributed import world_info
        if world_info(group)[1] > 1:
            return _filter_sharded(H, Y, spec, group)
    host_h = _streamable_host(H)
    if host_h is not None:
        return _filter_streamed(host_h, Y, spec)
    hm = _hermitian(H)
    if isinstance(Y, VectorBlock):
        yb = Y.device_block(hm.device_block().device).clone()
    else:
        y = _host_block(Y)
        y2d = y if y.ndim == 2 else y.reshape(-1, 1)
        if y2d.shape[0] != hm.n:
            raise ContractViolation(
                f"filter operand mismatch: H is {(hm.n, hm.n)}, Y has {y2d.shape[0]} rows")
        yb = dev.to_device(y2d, hm.device_block().device)
    if dev.rows(yb) != hm.n:
        raise ContractViolation(f"filter operand mismatch: H is {(hm.n, hm.n)}, Y has {dev.rows(yb)} rows")
    w = torch.empty_like(yb)
    out = engine(yb.device).filter(hm.device_block(), yb, w, spec.degree, spec.a, spec.b,
                                   spec.lam_ref)
    _count_products(spec.degree * dev.cols(yb))
    return VectorBlock(out)


# Host operators at least this large are uploaded panel by panel under the first
# degree step (chfsi_filter_streamed) instead of before the filter.
_STREAM_MIN_N = 4096


def _streamable_host(H):
    """F-order complex128 host copy of a raw (reference-style ndarray) operator large
    enough to stream, else None. Wrapped operators are already resident."""
    if isinstance(H, (HermitianDenseMatrix, VectorBlock, LowerTriangularFactor, torch.Tensor)):
        return None
    if hasattr(H, "entries"):
        return None
    a = np.asarray(H)
    if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] < _STREAM_MIN_N:
        return None
    return np.asfortranarray(a, dtype=np.complex128)


def _filter_streamed(host_h, Y, spec):
    """chebyshev_filter for a host ndarray H: the upload of H overlaps the first degree
    step (core.py:304 uses the raw array as is; so does this -- no Hermitian check)."""
    n = host_h.shape[0]
    device = default_device()
    if isinstance(Y, VectorBlock):
        yb = Y.device_block(device).clone()
    else:
        y = _host_block(Y)
        y2d = y if y.ndim == 2 else y.reshape(-1, 1)
        if y2d.shape[0] != n:
            raise ContractViolation(
                f"filter operand mismatch: H is {(n, n)}, Y has {y2d.shape[0]} rows")
        yb = dev.to_device(y2d, device)
    if dev.rows(yb) != n:
        raise ContractViolation(f"filter operand mismatch: H is {(n, n)}, Y has {dev.rows(yb)} rows")
    hdev = dev.empty(n, n, device)
    w = torch.empty_like(yb)
    # the result comes back to the host panel by panel under the last degree step
    out, host = engine(device).filter_streamed_to_host(host_h, hdev, yb, w, spec.degree,
                                                       spec.a, spec.b, spec.lam_ref)
    _count_products(spec.degree * dev.cols(yb))
    vb = VectorBlock(out)
    host.setflags(write=False)
    object.__setattr__(vb, "_host", host)
    return vb


def _filter_sharded(H, Y, spec, group):
    """chebyshev_filter over the ranks of ``group`` (column-separable recurrence,
    core.py:276-283): H replicated (host slabs + all-gather), Y's columns sharded."""
    from .distributed import ColumnShards, replicate_from_host, world_info
    rank, world = world_info(group)
    device = default_device()
    if isinstance(H, HermitianDenseMatrix):
        hb = H.device_block(device)
    elif isinstance(H, torch.Tensor):
        hb = H
    else:
        if hasattr(H, "entries") and not isinstance(H, (VectorBlock, LowerTriangularFactor)):
            H = H.entries
        a = np.asarray(H)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ContractViolation(f"expected a square matrix, got shape {a.shape}")
        a = np.asfortranarray(a, dtype=np.complex128)
        hb = replicate_from_host(torch.from_numpy(a.T), device, group)
    n = dev.rows(hb)
    if isinstance(Y, VectorBlock):
        yfull = Y.device_block(device)
        k = dev.cols(yfull)
        if dev.rows(yfull) != n:
            raise ContractViolation(f"filter operand mismatch: H is {(n, n)}, Y has {dev.rows(yfull)} rows")
        sh = ColumnShards(k, world)
        lo, hi = sh.range(rank)
        yb = yfull[lo:hi].clone()
    else:
        y = _host_block(Y)
        y2d = y if y.ndim == 2 else y.reshape(-1, 1)
        if y2d.shape[0] != n:
            raise ContractViolation(
                f"filter operand mismatch: H is {(n, n)}, Y has {y2d.shape[0]} rows")
        k = y2d.shape[1]
        sh = ColumnShards(k, world)
        lo, hi = sh.range(rank)
        yb = dev.to_device(y2d[:, lo:hi], device)
    if hi > lo:
        w = torch.empty_like(yb)
        out = engine(device).filter(hb, yb, w, spec.degree, spec.a, spec.b, spec.lam_ref)
    else:
        out = yb
    full = sh.gather_block(out, group)
    _count_products(spec.degree * k)
    return VectorBlock(full)


def rayleigh_ritz(H, Q):
    """Ritz values (ascending) and rotated block Q W (core.py:333-344)."""
    hm = _hermitian(H)
    if isinstance(Q, VectorBlock):
        qb = Q.device_block(hm.device_block().device)
        if not Q.orthonormal:
            from .linalg import _orth_deviation
            devn = _orth_deviation(qb)
            if devn > 1e-10 * np.sqrt(Q.s):
                raise ContractViolation(f"rayleigh_ritz requires orthonormal columns, deviation {devn:.3e}")
    else:
        qb = dev.to_device(_host_block(Q), hm.device_block().device)
    n, k = dev.rows(qb), dev.cols(qb)
    hq, z, hz = (dev.empty(n, k, qb.device) for _ in range(3))
    w = engine(qb.device).rayleigh_ritz(hm.device_block(), qb, hq, z, hz)
    _count_products(k)
    return w, VectorBlock(z, orthonormal=True)


def residuals(H, Y, lambdas):
    """||H y_i - lambda_i y_i||_2 per column (core.py:347-358)."""
    hm = _hermitian(H)
    if isinstance(Y, VectorBlock):
        yb = Y.device_block(hm.device_block().device)
    else:
        y = _host_block(Y)
        y2d = y if y.ndim == 2 else y.reshape(-1, 1)
        yb = dev.to_device(y2d, hm.device_block().device)
    lam = np.asarray(lambdas, dtype=np.float64).ravel()
    if lam.shape[0] != dev.cols(yb):
        raise ContractViolation(f"{lam.shape[0]} eigenvalues for {dev.cols(yb)} columns")
    n, k = dev.rows(yb), dev.cols(yb)
    eng = engine(yb.device)
    hy = dev.empty(n, k, yb.device)
    eng.zgemm("N", "N", n, k, n, 1.0, hm.device_block(), yb, 0.0, hy)
    _count_products(k)
    return eng.residual_norms(hy, yb, lam)


# ----------------------------------------------------------------------
# the solver


class _Workspace:
    """Device buffers of one solve, reused across outer iterations."""

    def __init__(self, n, s_tot, nev, device):
        self.n, self.s, self.nev = n, s_tot, nev
        self.fa = dev.empty(n, s_tot, device)
        self.fb = dev.empty(n, s_tot, device)
        self.hq = dev.empty(n, s_tot, device)
        self.z = dev.empty(n, s_tot, device)
        self.hz = dev.empty(n, s_tot, device)
        self.locked = dev.empty(n, nev, device)


class DeviceSolver:
    """One ChFSI solve on a device-resident H (core.py:385-546)."""

    def __init__(self, hm, config, device=None, group=None):
        self.hm = hm
        self.cfg = config
        self.hb = hm.device_block(device)
        self.device = self.hb.device
        self.eng = engine(self.device)
        self.n = hm.n
        self.sharded = None
        if group is not None:
            from .distributed import ShardedPhases, world_info
            if world_info(group)[1] > 1:
                self.sharded = ShardedPhases(group)

    # -- phases -------------------------------------------------------
    def _filter(self, active, out_other, a_edge, b_up, lam_ref, locked=None):
        """Filter the active block in place (active is clobbered); returns the
        tensor with p_m(H) active: either ``active`` or ``out_other``. With a
        process group, each rank filters (and projects against ``locked``) its
        column shard and the shards are all-gathered (distributed.ShardedPhases)."""
        if self.sharded is not None:
            return self.sharded.filter_project(self.eng, self.hb, active, out_other,
                                               self.cfg.degree, a_edge, b_up, lam_ref, locked)
        return self.eng.filter(self.hb, active, out_other, self.cfg.degree, a_edge, b_up, lam_ref)

    def _orthonormalize(self, f, locked, t, q, rng, projected=False):
        """core.py:365-382 with rank-collapse replacement from the host RNG.
        ``projected``: f was already projected against ``locked`` (sharded path);
        only a replaced column needs the projection again."""
        n = self.n
        for _ in range(dev.cols(f) + 2):
            try:
                if self.sharded is not None:  # f is replicated and already projected
                    return self.sharded.orthonormalize(self.eng, f, t, q, rank_tol=1e-14)
                self.eng.orthonormalize(f, None if projected else locked, t, q, rank_tol=1e-14)
                return q
            except RankDeficient as exc:
                col = rng.standard_normal(n) + 1j * rng.standard_normal(n)
                f[exc.column].copy_(torch.from_numpy(col).to(self.device))
                if projected and locked is not None:
                    self.eng.project_out(f[exc.column:exc.column + 1], locked)
        raise RankDeficient(0)

    def _sync(self):
        self.eng.synchronize()

    def _phases(self, act, ws, nl, a_edge, b_up, lam_ref, rng, ev):
        """One outer iteration's arithmetic (core.py:459-477): filter the active block,
        orthonormalise against the locked block, Rayleigh-Ritz + residual norms.
        Phase times come from CUDA events on the solver stream: the iteration needs only
        two host syncs (rank test after CholQR2; Ritz values + residuals)."""
        ncols = dev.cols(act)
        locked = ws.locked[:nl] if nl else None
        ev[0].record(self.eng.stream)
        f = self._filter(act, ws.fb[:ncols], a_edge, b_up, lam_ref, locked)
        ev[1].record(self.eng.stream)
        _count_products(self.cfg.degree * ncols)
        q = self._orthonormalize(f, locked, ws.hq[:ncols], ws.fa[:ncols], rng,
                                 projected=self.sharded is not None)
        ev[2].record(self.eng.stream)
        wvec = None
        if self.sharded is not None:
            # f (in ws.fb) is dead after the QR: its buffer takes the own Ritz vectors
            w, res, wvec = self.sharded.rayleigh_ritz(self.eng, self.hb, q, ws.hq[:ncols],
                                                      ws.fb[:ncols], ws.hz[:ncols])
        else:
            w, res = self.eng.rayleigh_ritz(self.hb, q, ws.hq[:ncols], ws.z[:ncols],
                                            ws.hz[:ncols], residuals=True)
        ev[3].record(self.eng.stream)
        _count_products(ncols)
        ev[3].synchronize()
        tf = ev[0].elapsed_time(ev[1]) * 1e-3
        tq = ev[1].elapsed_time(ev[2]) * 1e-3
        trr = ev[2].elapsed_time(ev[3]) * 1e-3  # includes the fused residual norms
        return q, w, res, wvec, tf, tq, trr

    def probe_iterations(self, locked, active, iters, a_edge, b_up, lam_ref, seed=0):
        """Time ``iters`` outer iterations from a given state -- ``locked`` (n x L,
        orthonormal) and ``active`` (n x k) column-major device blocks -- without locking
        (every iteration filters the current Ritz block again). The per-iteration cost
        of a solve's long narrow tail (reference interval semantics, core.py:507-509: at
        c4 ~5000 iterations at k_a ~ 201 with 2000 locked) without running the ~2000 s
        solve; with a group the phases are sharded exactly as in a solve. Returns a list
        of (t_filter, t_qr, t_rr, t_wall) per iteration."""
        n = self.n
        nl, k = dev.cols(locked), dev.cols(active)
        ws = _Workspace(n, k, max(nl, 1), self.device)
        ws.locked[:nl].copy_(locked)
        ws.z[:k].copy_(active)
        rng = _rng(seed)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        out = []
        self.eng.declare_operator(self.hb)
        try:
            for _ in range(iters):
                t0 = time.perf_counter()
                q, w, res, wvec, tf, tq, trr = self._phases(ws.z[:k], ws, nl, a_edge, b_up,
                                                            lam_ref, rng, ev)
                if self.sharded is not None:
                    self.sharded.ritz_columns(self.eng, q, wvec, 0, None, ws.z[:k])
                out.append((tf, tq, trr, time.perf_counter() - t0))
        finally:
            self.eng.declare_operator(None)
        return out

    # -- driver -------------------------------------------------------
    def run(self, Y0, prior, rng, callback=None):
        # H is not written during the solve: its 3M sum plane is formed once here instead
        # of once per filter call (chfsi_declare_operator), and dropped at the end
        self.eng.declare_operator(self.hb)
        try:
            return self._run(Y0, prior, rng, callback)
        finally:
            self.eng.declare_operator(None)

    def _run(self, Y0, prior, rng, callback=None):
        cfg = self.cfg
        n, nev = self.n, cfg.nev
        s_tot = nev + cfg.buffer_cols
        ws = _Workspace(n, s_tot, nev, self.device)
        report = SolveReport(n=n, nev=nev)
        t_start = time.perf_counter()

        if Y0 is None or (isinstance(Y0, str) and Y0 == "random"):
            ws.z.copy_(dev.to_device(_rand_cols(rng, n, s_tot), self.device))
        elif isinstance(Y0, torch.Tensor):
            ws.z.copy_(Y0)
        else:
            ws.z.copy_(dev.to_device(Y0, self.device))

        # device time between events on the solver stream: work queued before the
        # solve (e.g. the generalized forward map) is not charged to Lanczos
        e_l0 = torch.cuda.Event(enable_timing=True)
        e_l1 = torch.cuda.Event(enable_timing=True)
        e_l0.record(self.eng.stream)
        b_up = _lanczos(self.hm, cfg.lanczos_steps, rng)
        e_l1.record(self.eng.stream)
        e_l1.synchronize()
        report.t_lanczos = e_l0.elapsed_time(e_l1) * 1e-3
        report.setup_matmuls += min(cfg.lanczos_steps, n)
        report.upper_bound = b_up

        if prior is not None:
            lam_ref, a_edge = float(prior[0]), float(prior[1])
        else:
            # bootstrap: one unfiltered Rayleigh-Ritz pass on the start block
            e_l0.record(self.eng.stream)
            q = self._orthonormalize(ws.z, None, ws.hq, ws.fa, rng)
            if self.sharded is not None:
                w, _, wvec = self.sharded.rayleigh_ritz(self.eng, self.hb, q, ws.hq, ws.fb, ws.hz)
                self.sharded.ritz_columns(self.eng, q, wvec, 0, None, ws.z)
            else:
                w = self.eng.rayleigh_ritz(self.hb, q, ws.hq, ws.z, ws.hz)
            e_l1.record(self.eng.stream)
            e_l1.synchronize()
            _count_products(s_tot)
            report.t_rr += e_l0.elapsed_time(e_l1) * 1e-3
            report.setup_matmuls += s_tot
            lam_ref, a_edge = float(w[0]), float(w[nev])
            if cfg.interval == "block_top":
                a_edge = float(w[-1])

        locked_vals = []
        nl = 0
        act = ws.z[:s_tot]  # the unconverged block, a contiguous column range of Z
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        for it in range(1, cfg.max_outer_iters + 1):
            if not lam_ref < a_edge:
                raise FilterDegenerate(
                    f"lambda_1 estimate {lam_ref} >= lambda_nev+1 estimate {a_edge}; "
                    f"interval placement ill-posed (increase buffer)")
            if not a_edge < b_up:
                b_up = a_edge + max(1.0, abs(a_edge)) * 1e-8
            ncols = dev.cols(act)

            q, w, res, wvec, tf, tq, trr = self._phases(act, ws, nl, a_edge, b_up, lam_ref,
                                                        rng, ev)
            report.filter_flops += 8.0 * n * n * cfg.degree * ncols
            tres = 0.0

            kk = 0
            while kk < len(w) and res[kk] < cfg.tol and len(locked_vals) < nev:
                locked_vals.append(float(w[kk]))
                kk += 1
            if self.sharded is not None:
                # newly locked vectors on every rank + this rank's next active shard
                self.sharded.ritz_columns(self.eng, q, wvec, kk, ws.locked[nl:nl + kk],
                                          ws.z[:ncols])
                nl += kk
            elif kk:
                ws.locked[nl:nl + kk].copy_(ws.z[:kk])
                nl += kk
            act = ws.z[kk:ncols]

            unconv = res[kk:]
            report.iterations.append(IterationStat(
                iteration=it, filtered_cols=ncols, converged=len(locked_vals),
                max_resid=float(unconv.max()) if unconv.size else 0.0,
                min_resid=float(unconv.min()) if unconv.size else 0.0,
                matmuls=(cfg.degree + 1) * ncols,
                t_filter=tf, t_qr=tq, t_rr=trr, t_resid=tres))
            report.t_filter += tf
            report.t_qr += tq
            report.t_rr += trr
            report.t_resid += tres
            if callback is not None:
                callback(report.iterations[-1])

            comb = np.sort(np.concatenate([locked_vals, w[kk:]]))
            lam_ref = float(comb[0])
            a_edge = float(comb[nev])
            if cfg.interval == "block_top":
                a_edge = float(comb[-1])
            report.est_lam1 = lam_ref
            report.est_lam_next = float(comb[nev])
            if len(locked_vals) >= nev:
                break

        report.total_matmuls = report.setup_matmuls + sum(i.matmuls for i in report.iterations)
        vecs = ws.locked[:nl]
        if len(locked_vals) < nev:
            report.t_total = time.perf_counter() - t_start
            raise NotConverged(
                f"{len(locked_vals)}/{nev} pairs converged after {cfg.max_outer_iters} outer "
                f"iterations", np.asarray(locked_vals),
                VectorBlock(vecs.clone()) if nl else dev.to_host(vecs), report)

        vals = np.asarray(locked_vals)
        e_l0.record(self.eng.stream)
        if self.sharded is not None:
            final_res = self.sharded.residual_check(self.eng, self.hb, vecs, vals, ws.hq[:nev])
        else:
            self.eng.apply_operator(self.hb, vecs, ws.hq[:nev])
            final_res = self.eng.residual_norms(ws.hq[:nev], vecs, vals)
        e_l1.record(self.eng.stream)
        e_l1.synchronize()
        _count_products(nev)
        report.t_resid += e_l0.elapsed_time(e_l1) * 1e-3
        report.total_matmuls += nev
        report.t_total = time.perf_counter() - t_start
        out = vecs.clone()
        del ws
        if np.any(final_res >= cfg.tol):
            raise NotConverged(f"final residual re-check failed: max {final_res.max():.3e}",
                               vals, VectorBlock(out), report)
        report.converged = True
        return vals, VectorBlock(out, orthonormal=True), report


def _localize(x, memo=None):
    """Per-rank view of an argument inside an in-process rank thread (``devices=``):
    device-resident matrices and blocks are copied to the thread's own GPU (over
    NVLink) and wrapped anew, so ranks never share (or flip) a wrapper's device cache;
    host arrays pass through (each rank uploads its own copy). ``memo`` maps id(x) to
    the local copy, so an object used by several problems (a sequence's fixed B, whose
    Cholesky factor is cached) is localised once per rank."""
    if memo is not None and id(x) in memo:
        return memo[id(x)]
    out = x
    d = default_device()
    if isinstance(x, HermitianDenseMatrix):
        if x._dev is not None:
            blk = x._dev if x._dev.device == d else x._dev.to(d)
            out = HermitianDenseMatrix.from_device(blk, trusted=True)
        else:
            out = HermitianDenseMatrix(x)  # host-backed: uploads on this rank's device
    elif isinstance(x, VectorBlock) and x._dev is not None:
        blk = x._dev if x._dev.device == d else x._dev.to(d)
        out = VectorBlock(blk)
        object.__setattr__(out, "orthonormal", x.orthonormal)
    elif isinstance(x, torch.Tensor) and x.is_cuda and x.device != d:
        out = x.to(d)
    if memo is not None:
        memo[id(x)] = out
    return out


def _default_devices():
    from .comm import default_devices
    return default_devices()


def _in_process(devices, group, fn, seed):
    """Run ``fn(comm, seed_copy)`` on one thread per GPU of ``devices`` (comm.py) and
    return rank 0's result. Every rank gets its own copy of the caller's Generator (the
    start block and rank-collapse columns are replicated draws); afterwards the
    caller's Generator is left where rank 0's ended, as after a one-GPU solve."""
    from .comm import clone_rng, normalize_devices, run_on_devices
    if group is not None:
        raise ContractViolation("give either group= (one process per GPU) or devices= "
                                "(several GPUs in this process), not both")
    devs = normalize_devices(devices)
    rngs = [clone_rng(seed) for _ in devs]
    if len(devs) == 1:
        from .comm import inside_group
        with torch.cuda.device(devs[0]), inside_group():
            out = fn(None, rngs[0])
    else:
        out = run_on_devices(devs, lambda comm: fn(comm, rngs[comm.rank]))[0]
    if isinstance(seed, np.random.Generator):
        seed.bit_generator.state = rngs[0].bit_generator.state
    return out


def chfsi_solve(H, Y0, config, prior=None, seed=0, *, group=None, devices=None,
                callback=None):
    """Run ChFSI on a standard Hermitian problem (core.py:385-546).

    Same signature, return types, report fields, RNG order and exceptions
    as the reference; arithmetic on the GPU. ``group`` (keyword-only, B200
    extension): a torch.distributed process group with one process per GPU;
    the filter columns are then sharded across its ranks (H replicated).
    ``devices`` (keyword-only): the same sharded solve over several GPUs of this
    process -- an int N (GPUs 0..N-1) or CUDA ordinals; one host thread per GPU and
    an NCCL clique (comm.py); results on the first device.
    ``callback`` (keyword-only, B200 extension): called with each IterationStat.
    """
    if devices is None and group is None:
        devices = _default_devices()
    if devices is not None:
        return _in_process(devices, group, lambda comm, rng: chfsi_solve(
            _localize(H), _localize(Y0), config, prior, rng, group=comm,
            callback=callback if comm is None or comm.rank == 0 else None), seed)
    config = _as_config(config)
    if isinstance(H, HermitianDenseMatrix):
        n = H.n
    else:
        hh = H.entries if hasattr(H, "entries") else np.asarray(H)
        if hh.ndim != 2 or hh.shape[0] != hh.shape[1]:
            raise ContractViolation(f"expected a square matrix, got shape {hh.shape}")
        n = hh.shape[0]
    nev = config.nev
    s_tot = nev + config.buffer_cols
    if s_tot > n:
        raise ContractViolation(f"nev + buffer = {s_tot} exceeds the matrix order {n}")
    rng = _rng(seed)
    y0 = None
    if Y0 is None or (isinstance(Y0, str) and Y0 == "random"):
        y0 = None
    elif isinstance(Y0, VectorBlock) and Y0._dev is not None:
        if (Y0.n, Y0.s) != (n, s_tot):
            raise ContractViolation(f"start block must be {n} x {s_tot}, got {(Y0.n, Y0.s)}")
        y0 = Y0._dev
    else:
        y = _host_block(Y0)
        if y.ndim != 2 or y.shape != (n, s_tot):
            raise ContractViolation(f"start block must be {n} x {s_tot}, got {y.shape}")
        y0 = y
    hm = _hermitian(H)
    return DeviceSolver(hm, config, group=group).run(y0, prior, rng, callback)


def solve_generalized(A, B, Y0, config, prior=None, seed=0, *, group=None, devices=None,
                      callback=None):
    """A c = lambda B c for the nev lowest pairs (core.py:549-569):
    B = L L^H (cuSOLVER zpotrf), H = L^-1 A L^-H (triangular inverse + DMMA
    GEMMs), ChFSI on H, C = L^-H Y. Returns B-orthonormal vectors.
    ``group`` / ``devices``: as for chfsi_solve."""
    if devices is None and group is None:
        devices = _default_devices()
    if devices is not None:
        return _in_process(devices, group, lambda comm, rng: solve_generalized(
            _localize(A), _localize(B), _localize(Y0), config, prior, rng, group=comm,
            callback=callback if comm is None or comm.rank == 0 else None), seed)
    config = _as_config(config)
    ab = A.device_block() if isinstance(A, HermitianDenseMatrix) else None
    bb = B.device_block() if isinstance(B, HermitianDenseMatrix) else None
    ah = None if ab is not None else _host_block(A)
    bh = None if bb is not None else _host_block(B)
    ashape = (A.n, A.n) if ab is not None else ah.shape
    bshape = (B.n, B.n) if bb is not None else bh.shape
    if tuple(ashape) != tuple(bshape):
        raise ContractViolation(f"A and B orders differ: {tuple(ashape)} vs {tuple(bshape)}")
    cached = getattr(B, "_factor", None) if bb is not None else None
    if cached is not None:
        lfac, linv = cached
    else:
        lfac = cholesky_factor(B if bb is not None else bh)
        linv = dev.empty(lfac.n, lfac.n, lfac.device_block().device)
        engine(linv.device).trtri_lower(lfac.device_block(), linv)
        if bb is not None:  # immutable B: keep (L, L^-1) for the next problem of a sequence
            object.__setattr__(B, "_factor", (lfac, linv))
    d = lfac.device_block().device
    if ab is None:
        ab = dev.to_device(ah, d)
    n = dev.rows(ab)
    eng = engine(d)
    from .distributed import reduce_sharded, upper_apply_sharded, world_info
    sharded = group is not None and world_info(group)[1] > 1
    if sharded:
        # column-sharded reduction + all-gather: every rank ends with the same H
        hb = reduce_sharded(eng, ab, linv, group)
    else:
        hb = _reduce_block(ab, lfac, linv)
    hm = HermitianDenseMatrix(hb, rtol=1e-8)
    y0 = Y0
    if Y0 is not None and not (isinstance(Y0, str) and Y0 == "random"):
        yb = Y0.device_block(d) if isinstance(Y0, VectorBlock) else to_block(_host_block(Y0), d)
        # forward map y = L^H c (core.py:565)
        if sharded:
            fwd = upper_apply_sharded(eng, lfac.device_block(), yb, group)
        else:
            fwd = dev.empty(dev.rows(yb), dev.cols(yb), d)
            eng.zgemm("C", "N", n, dev.cols(yb), n, 1.0, lfac.device_block(), yb, 0.0, fwd,
                      tri=eng.TRI_A_UPPER)
        y0 = VectorBlock(fwd)
    lam, yv, report = chfsi_solve(hm, y0, config, prior=prior, seed=seed, group=group,
                                  callback=callback)
    # back-transform C = L^-H Y (core.py:191-195)
    if sharded:
        c = upper_apply_sharded(eng, linv, yv.device_block(d), group)
    else:
        c = dev.empty(n, yv.s, d)
        eng.zgemm("C", "N", n, yv.s, n, 1.0, linv, yv.device_block(d), 0.0, c,
                  tri=eng.TRI_A_UPPER)
    return lam, VectorBlock(c), report
