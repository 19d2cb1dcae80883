"""ORACLE / TEST INFRASTRUCTURE ONLY.

CPU restatement (numpy + scipy LAPACK/BLAS + the C Jacobi in jacobi.c) of
the reference ChFSI algorithm of arXiv 1305.5120 as implemented in the
reference package /root/reference/pkg/src/chfsi (cited below as
core.py / linalg.py / sequence.py with line numbers).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker
or the timed CPU baseline -- never as the product path. Every numpy call
keeps the reference's operand order and memory layouts, so on the same
inputs it reproduces the reference to the last bit on the same BLAS build;
tests/test_oracle_golden.py pins it against fixtures produced by running
the reference itself (tests/golden/, scripts/make_golden.py).
"""

import ctypes
import math
import os
import subprocess
import time

import numpy as np
from scipy.linalg import blas as _sblas
from scipy.linalg import lapack as _slapack

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libjacobi_oracle.so")
_jac = None


class OracleError(Exception):
    """Raised where the reference raises one of its ChfsiError subclasses;
    ``kind`` names the reference class (errors.py)."""

    def __init__(self, kind, message, **info):
        self.kind = kind
        self.info = info
        super().__init__(f"{kind}: {message}")


def build():
    """Compile jacobi.c into oracle/_build (gcc, no FMA contraction)."""
    os.makedirs(os.path.dirname(_SO), exist_ok=True)
    src = os.path.join(_HERE, "jacobi.c")
    if os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(src):
        return _SO
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                           "-o", _SO, src, "-lm"])
    return _SO


def _lib():
    global _jac
    if _jac is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.oracle_jacobi_sweeps.restype = ctypes.c_int
        lib.oracle_jacobi_sweeps.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                             ctypes.POINTER(ctypes.c_int)]
        _jac = lib
    return _jac


# ---------------------------------------------------------------- Jacobi
def jacobi_eig(h, max_sweeps=30):
    """linalg.py:304-323 `_jacobi_raw`: ascending eigenvalues, F-order vectors."""
    h = np.asarray(h, dtype=np.complex128)
    n = h.shape[0]
    work = np.array(h, dtype=np.complex128, order="C")
    vec = np.eye(n, dtype=np.complex128)
    fro = np.linalg.norm(work)
    if n == 1 or fro == 0.0:
        d = work.diagonal().real.copy()
        idx = np.argsort(d, kind="stable")
        return d[idx], vec[:, idx]
    done = ctypes.c_int(0)
    ok = _lib().oracle_jacobi_sweeps(n, work.ctypes.data, vec.ctypes.data, n, int(max_sweeps),
                                     1e-13 * fro, ctypes.byref(done))
    if not ok:
        raise OracleError("OracleNoConvergence", f"{done.value} sweeps (n={n})")
    d = work.diagonal().real.copy()
    idx = np.argsort(d, kind="stable")
    return d[idx], np.asfortranarray(vec[:, idx])


# ---------------------------------------------------------------- products
class Tally:
    """Square-matrix x block product counter (linalg.py:49-82)."""

    def __init__(self):
        self.cols = 0


def product(alpha, a, b, tally, beta=0.0, c=None):
    """linalg.py:198-251 `gemm` at workers == 1: beta*C first, then += alpha*(A@B)."""
    b2 = b if b.ndim == 2 else b.reshape(-1, 1)
    if c is None:
        out = np.zeros((a.shape[0], b2.shape[1]), dtype=np.complex128, order="F")
    else:
        out = np.array(c, dtype=np.complex128, order="F") * beta
    if alpha != 0.0:
        if a.shape[0] == a.shape[1] and tally is not None:
            tally.cols += b2.shape[1]
        out += alpha * (a @ b2)
    return out[:, 0] if b.ndim == 1 else out


# ---------------------------------------------------------------- types
def hermitian(a, rtol=1e-13):
    """linalg.py:104-121 HermitianDenseMatrix construction (check + symmetrise)."""
    a = np.array(np.asarray(a, dtype=np.complex128), order="F")
    scale = np.linalg.norm(a)
    if scale > 0:
        dev = np.linalg.norm(a - a.conj().T)
        if dev > rtol * scale:
            raise OracleError("ContractViolation", f"not Hermitian: {dev:.3e}")
    a = (a + a.conj().T) / 2.0
    np.fill_diagonal(a, a.diagonal().real)
    return np.asfortranarray(a)


# ---------------------------------------------------------------- pieces
def lanczos_bound(h, k, rng, tally=None):
    """core.py:202-256 `lanczos_upper_bound`."""
    n = h.shape[0]
    k = min(int(k), n)
    v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    v /= np.linalg.norm(v)
    basis = np.zeros((n, k), dtype=np.complex128, order="F")
    basis[:, 0] = v
    diag, off = [], []
    for j in range(k):
        w = product(1.0, h, basis[:, j], tally)
        diag.append(np.vdot(basis[:, j], w).real)
        w -= diag[-1] * basis[:, j]
        if j > 0:
            w -= off[-1] * basis[:, j - 1]
        w -= basis[:, : j + 1] @ (basis[:, : j + 1].conj().T @ w)
        off.append(np.linalg.norm(w))
        if off[-1] < 1e-14 or j == k - 1:
            break
        basis[:, j + 1] = w / off[-1]
    m = len(diag)
    t = np.zeros((m, m), dtype=np.complex128)
    for i in range(m):
        t[i, i] = diag[i]
        if i + 1 < m:
            t[i, i + 1] = t[i + 1, i] = off[i]
    lam, _ = jacobi_eig(t)
    guard = 4.0 * m * np.finfo(np.float64).eps * max(abs(lam[0]), abs(lam[-1]))
    return float(lam[-1] + off[m - 1] + guard), m


def cheb_filter(h, y, degree, a, b, lam_ref, tally=None):
    """core.py:263-284 `_filter_raw` (scaled three-term recurrence)."""
    center, half = (a + b) / 2.0, (b - a) / 2.0
    s1 = half / (lam_ref - center)
    s = s1
    prev = y
    cur = product(s1 / half, h, y, tally, beta=-center * s1 / half, c=y)
    for _ in range(degree - 1):
        s_next = 1.0 / (2.0 / s1 - s)
        g = 2.0 * s_next / half
        nxt = product(g, h, cur, tally, beta=-center * g, c=cur)
        nxt -= (s * s_next) * prev
        prev, cur = cur, nxt
        s = s_next
    return cur


def orth_against(f, locked, rng):
    """core.py:365-382 `_qr_against_locked` (one projection pass + Householder QR,
    rank collapse -> fresh random column, at most ncols + 2 attempts)."""
    n = f.shape[0]
    for _ in range(f.shape[1] + 2):
        w = f
        if locked.shape[1]:
            w = w - locked @ (locked.conj().T @ w)
        q, r = np.linalg.qr(w)
        tiny = np.abs(np.diagonal(r)) < 1e-14 * np.linalg.norm(w)
        if not np.any(tiny):
            return q
        col = int(np.nonzero(tiny)[0][0])
        f = np.array(f)
        f[:, col] = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    raise OracleError("RankDeficient", "retries exhausted", column=0)


def ritz(h, q, tally=None):
    """core.py:318-330 `_rr_raw`: (ritz values, Z = QW, HZ = (HQ)W)."""
    hq = product(1.0, h, q, tally)
    g = q.conj().T @ hq
    g = (g + g.conj().T) / 2.0
    w, vec = jacobi_eig(g)
    return w, q @ vec, hq @ vec


def resid(h, y, lam, tally=None):
    """core.py:347-358 `residuals`."""
    y2 = y if y.ndim == 2 else y.reshape(-1, 1)
    hy = product(1.0, h, y2, tally)
    return np.linalg.norm(hy - y2 * np.asarray(lam, dtype=np.float64).ravel(), axis=0)


# ---------------------------------------------------------------- solver
def solve(h, y0, nev, nex=None, degree=20, tol=1e-10, max_it=30, lanczos_steps=10,
          prior=None, seed=0, tally=None):
    """core.py:385-546 `chfsi_solve` (standard Hermitian problem).

    Returns (eigenvalues, eigenvectors F-order, report dict). Raises
    OracleError("NotConverged", ..., eigenvalues=, eigenvectors=, report=)
    when the iteration budget is exhausted, like the reference.
    """
    tally = tally if tally is not None else Tally()
    h = np.asarray(h, dtype=np.complex128)
    n = h.shape[0]
    nex = max(1, math.ceil(0.1 * nev)) if nex is None else nex
    s_tot = nev + nex
    if s_tot > n:
        raise OracleError("ContractViolation", f"nev + buffer = {s_tot} > n = {n}")
    rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
    if y0 is None or (isinstance(y0, str) and y0 == "random"):
        y = rng.standard_normal((n, s_tot)) + 1j * rng.standard_normal((n, s_tot))
    else:
        y = np.array(np.asarray(y0, dtype=np.complex128), order="F")
        if y.shape != (n, s_tot):
            raise OracleError("ContractViolation", f"start block shape {y.shape}")
    rep = {"n": n, "nev": nev, "iterations": [], "setup_matmuls": 0}
    t_start = time.perf_counter()
    b_up, _ = lanczos_bound(h, lanczos_steps, rng, tally)
    rep["setup_matmuls"] += min(lanczos_steps, n)
    rep["upper_bound"] = b_up
    if prior is not None:
        lam_ref, a_edge = float(prior[0]), float(prior[1])
    else:
        q = orth_against(y, np.zeros((n, 0), dtype=np.complex128), rng)
        w, z, _ = ritz(h, q, tally)
        rep["setup_matmuls"] += s_tot
        lam_ref, a_edge = float(w[0]), float(w[nev])
        y = z
    vals = []
    vecs = np.zeros((n, 0), dtype=np.complex128, order="F")
    active = y
    for it in range(1, max_it + 1):
        if not lam_ref < a_edge:
            raise OracleError("FilterDegenerate", f"{lam_ref} >= {a_edge}")
        if not a_edge < b_up:
            b_up = a_edge + max(1.0, abs(a_edge)) * 1e-8
        ncols = active.shape[1]
        f = cheb_filter(h, active, degree, a_edge, b_up, lam_ref, tally)
        q = orth_against(f, vecs, rng)
        w, z, hz = ritz(h, q, tally)
        res = np.linalg.norm(hz - z * w, axis=0)
        kk = 0
        while kk < len(w) and res[kk] < tol and len(vals) < nev:
            vals.append(float(w[kk]))
            vecs = np.hstack([vecs, z[:, kk:kk + 1]])
            kk += 1
        active = z[:, kk:]
        left = res[kk:]
        rep["iterations"].append({
            "iteration": it, "filtered_cols": ncols, "converged": len(vals),
            "max_resid": float(left.max()) if left.size else 0.0,
            "min_resid": float(left.min()) if left.size else 0.0,
            "matmuls": (degree + 1) * ncols,
        })
        comb = np.sort(np.concatenate([vals, w[kk:]]))
        lam_ref, a_edge = float(comb[0]), float(comb[nev])
        rep["est_lam1"], rep["est_lam_next"] = lam_ref, a_edge
        if len(vals) >= nev:
            break
    rep["total_matmuls"] = rep["setup_matmuls"] + sum(r["matmuls"] for r in rep["iterations"])
    if len(vals) < nev:
        rep["t_total"] = time.perf_counter() - t_start
        raise OracleError("NotConverged", f"{len(vals)}/{nev}", eigenvalues=np.asarray(vals),
                          eigenvectors=vecs, report=rep)
    lam = np.asarray(vals)
    final = resid(h, vecs, lam, tally)
    rep["total_matmuls"] += nev
    rep["final_resid"] = final
    rep["t_total"] = time.perf_counter() - t_start
    if np.any(final >= tol):
        raise OracleError("NotConverged", "final re-check", eigenvalues=lam, eigenvectors=vecs,
                          report=rep)
    rep["converged"] = True
    return lam, vecs, rep


# ---------------------------------------------------------------- generalized
def cholesky(b):
    """linalg.py:254-270 `cholesky_factor` (zpotrf lower, clean, real diagonal)."""
    fac, info = _slapack.zpotrf(np.asarray(b, dtype=np.complex128), lower=1, clean=1,
                                overwrite_a=0)
    if info > 0:
        raise OracleError("NotPositiveDefinite", f"pivot {info}", pivot=int(info))
    fac = np.asfortranarray(fac)
    np.fill_diagonal(fac, fac.diagonal().real)
    return fac


def tri_solve(lf, x, side="left", adjoint=False):
    """linalg.py:326-355 `triangular_solve` (ztrsm, lower factor)."""
    x2 = x if x.ndim == 2 else x.reshape(-1, 1)
    z = _sblas.ztrsm(1.0, lf, np.asfortranarray(x2), side=0 if side == "left" else 1, lower=1,
                     trans_a=2 if adjoint else 0)
    return z[:, 0] if x.ndim == 1 else z


def reduce_standard(a, lf):
    """core.py:172-188 `reduce_to_standard`: H = L^-1 A L^-H, re-symmetrised (rtol 1e-8)."""
    w = tri_solve(lf, np.asarray(a, dtype=np.complex128), side="left")
    return hermitian(tri_solve(lf, w, side="right", adjoint=True), rtol=1e-8)


def solve_generalized(a, b, y0, nev, nex=None, degree=20, tol=1e-10, max_it=30,
                      lanczos_steps=10, prior=None, seed=0, tally=None):
    """core.py:549-569 `solve_generalized`."""
    lf = cholesky(b)
    h = reduce_standard(a, lf)
    if y0 is not None and not (isinstance(y0, str) and y0 == "random"):
        y0 = _sblas.ztrmm(1.0, lf, np.asfortranarray(np.asarray(y0, dtype=np.complex128)),
                          side=0, lower=1, trans_a=2)
    lam, y, rep = solve(h, y0, nev, nex, degree, tol, max_it, lanczos_steps, prior, seed, tally)
    return lam, tri_solve(lf, y, side="left", adjoint=True), rep


def solve_sequence_reuse(problems, seed, nev, nex=None, **kw):
    """sequence.py:165-228 `solve_sequence` in mode "reuse": cycle l starts from
    cycle l-1's vectors + random pad (rng [seed, 13, l]); solver rng [seed, 11, l];
    prior = (est_lam1, running min of est_lam_next)."""
    nex = max(1, math.ceil(0.1 * nev)) if nex is None else nex
    s_tot = nev + nex
    out = []
    prev, prior, running = None, None, None
    for ell, (a, b) in enumerate(problems, start=1):
        srng = np.random.default_rng([seed, 11, ell])
        y0, use_prior = None, None
        if prev is not None:
            prng = np.random.default_rng([seed, 13, ell])
            n = a.shape[0]
            pad = prng.standard_normal((n, s_tot - prev.shape[1])) + \
                1j * prng.standard_normal((n, s_tot - prev.shape[1]))
            y0 = np.hstack([prev, pad])
            use_prior = prior
        if b is None:
            lam, vecs, rep = solve(a, y0, nev, nex, prior=use_prior, seed=srng, **kw)
        else:
            lam, vecs, rep = solve_generalized(a, b, y0, nev, nex, prior=use_prior, seed=srng, **kw)
        out.append((lam, vecs, rep))
        prev = np.array(vecs)
        running = rep["est_lam_next"] if running is None else min(running, rep["est_lam_next"])
        prior = (rep["est_lam1"], running)
    return out


# ---------------------------------------------------------------- closed forms
def cheb_scalar(m, x):
    """C_m(x) by the cos/cosh closed form (reference test_filter.py:17-27 idea)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    inside = np.abs(x) <= 1.0
    out[inside] = np.cos(m * np.arccos(x[inside]))
    xo = x[~inside]
    out[~inside] = np.sign(xo) ** m * np.cosh(m * np.arccosh(np.abs(xo)))
    return out


def filter_gain(m, lam, a, b, lam_ref):
    c, e = (a + b) / 2.0, (b - a) / 2.0
    return cheb_scalar(m, (np.asarray(lam) - c) / e) / cheb_scalar(m, np.array([(lam_ref - c) / e]))[0]


def largest_angle_sine(u, v):
    """Largest principal angle between range(u) and range(v), sine formula
    arcsin ||V - Q(Q^H V)||_2 (exact below 1e-8)."""
    qu, _ = np.linalg.qr(np.asarray(u))
    qv, _ = np.linalg.qr(np.asarray(v))
    r = qv - qu @ (qu.conj().T @ qv)
    s = np.linalg.norm(r, 2)
    return float(np.arcsin(min(1.0, s)))
