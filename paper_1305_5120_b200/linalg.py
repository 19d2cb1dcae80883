"""Domain types and dense kernels, mirroring the reference's chfsi.linalg
(reference pkg/src/chfsi/linalg.py) with the arithmetic on the B200.

Types keep the reference contract (validation rules, read-only F-order
``entries``) but also carry a device copy, so a matrix uploaded once stays in
HBM across solves, filter calls and sequence cycles. Host copies are made
lazily and only when a caller reads ``entries``.
"""

import os
import threading

import numpy as np
import torch

from . import device as dev
from .errors import ContractViolation, DimensionMismatch, OracleNoConvergence, RankDeficient

__all__ = [
    "HermitianDenseMatrix", "VectorBlock", "LowerTriangularFactor", "gemm",
    "cholesky_factor", "householder_qr", "oracle_eig", "triangular_solve",
    "trmm_adjoint", "set_workers", "get_workers", "reset_product_count",
    "product_count",
]

# ----------------------------------------------------------------------
# worker setting and the square-product tally (linalg.py:49-82)

_lock = threading.Lock()
_workers = max(1, int(os.environ.get("CHFSI_WORKERS", "1")))
_product_columns = 0


def set_workers(count):
    """Kept for API compatibility (linalg.py:54). On the GPU path the
    parallelism is the grid; results do not depend on this value."""
    global _workers
    count = int(count)
    if count < 1:
        raise ContractViolation("worker count must be >= 1")
    _workers = count


def get_workers():
    return _workers


def reset_product_count():
    global _product_columns
    with _lock:
        _product_columns = 0


def product_count():
    """Columns pushed through n x n x s products so far (linalg.py:72-75)."""
    return _product_columns


def _count_products(cols):
    global _product_columns
    if dev.engine_tag() != 0:
        return  # in-process ranks (comm.py): the work is counted once, by rank 0
    with _lock:
        _product_columns += int(cols)


# ----------------------------------------------------------------------
# device helpers


def default_device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1305_5120_b200 requires a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def engine(device=None):
    return dev.Engine.get(device if device is not None else default_device())


def _asarray(x):
    """Host complex128 view of a wrapper type or array-like (linalg.py:89-93)."""
    if isinstance(x, (HermitianDenseMatrix, VectorBlock, LowerTriangularFactor)):
        return x.entries
    if isinstance(x, torch.Tensor):
        raise ContractViolation("pass device blocks through the wrapper types")
    return np.asarray(x, dtype=np.complex128)


def to_block(x, device=None):
    """Device column-major block (torch (k, n)) for a wrapper type or array."""
    device = device if device is not None else default_device()
    if isinstance(x, (HermitianDenseMatrix, VectorBlock, LowerTriangularFactor)):
        return x.device_block(device)
    a = np.asarray(x, dtype=np.complex128)
    return dev.to_device(a, device)


class _DeviceBacked:
    """Lazy host/device pair (host: read-only F-order ndarray; device: (k, n) tensor)."""

    __slots__ = ()

    def _init_storage(self, host, block):
        object.__setattr__(self, "_host", host)
        object.__setattr__(self, "_dev", block)

    @property
    def entries(self):
        if self._host is None:
            h = dev.to_host(self._dev)
            h.setflags(write=False)
            object.__setattr__(self, "_host", h)
        return self._host

    def device_block(self, device=None):
        device = torch.device(device) if device is not None else default_device()
        if self._dev is None or self._dev.device != device:
            object.__setattr__(self, "_dev", dev.to_device(self._host, device))
        return self._dev


class HermitianDenseMatrix(_DeviceBacked):
    """Square complex matrix with the Hermitian contract (linalg.py:96-126).

    Construction checks ||H - H^H||_F <= rtol ||H||_F and symmetrises
    (H <- (H + H^H)/2, real diagonal) -- on the GPU, where the matrix then
    stays resident. As a metric B of solve_generalized it also caches its
    Cholesky factor and the factor's inverse (the matrix is immutable), so a
    sequence with a fixed B factorises once (BASELINE c2-c4).
    """

    __slots__ = ("_host", "_dev", "n", "_factor")

    def __init__(self, entries, rtol=1e-13, device=None):
        if isinstance(entries, HermitianDenseMatrix):
            self._init_storage(entries._host, entries._dev)
            object.__setattr__(self, "n", entries.n)
            return
        if isinstance(entries, torch.Tensor):
            block = entries
            n0, n1 = block.shape[1], block.shape[0]
        else:
            a = _asarray(entries)
            if a.ndim != 2 or a.shape[0] != a.shape[1]:
                raise ContractViolation(f"expected a square matrix, got shape {a.shape}")
            block = dev.to_device(a, device if device is not None else default_device())
            n0, n1 = a.shape
        if n0 != n1:
            raise ContractViolation(f"expected a square matrix, got shape {(n0, n1)}")
        eng = engine(block.device)
        scale, devn = eng.hermitian_norms(block)
        if scale > 0 and devn > rtol * scale:
            raise ContractViolation(
                f"matrix is not Hermitian: deviation {devn:.3e} exceeds "
                f"{rtol:g} * ||H|| = {rtol * scale:.3e}")
        eng.hermitize(block)
        self._init_storage(None, block)
        object.__setattr__(self, "n", n0)

    @classmethod
    def from_device(cls, block, trusted=False, rtol=1e-13):
        """Wrap a device block; with trusted=True skip the check (already Hermitian)."""
        if not trusted:
            return cls(block, rtol=rtol)
        obj = cls.__new__(cls)
        obj._init_storage(None, block)
        object.__setattr__(obj, "n", block.shape[1])
        return obj

    def __setattr__(self, k, v):
        raise AttributeError("HermitianDenseMatrix is immutable")

    def __repr__(self):
        return f"HermitianDenseMatrix(n={self.n})"


def _orth_deviation(block):
    """||Q^H Q - I||_F computed on the device."""
    k = dev.cols(block)
    eng = engine(block.device)
    g = dev.empty(k, k, block.device)
    eng.zgemm("C", "N", k, k, dev.rows(block), 1.0, block, block, 0.0, g)
    g = g.transpose(0, 1)  # (row, col) indexing of the column-major k x k
    eye = torch.eye(k, dtype=dev.CDT, device=block.device)
    return float(torch.linalg.matrix_norm(g - eye).item())


class VectorBlock(_DeviceBacked):
    """n x s block of column vectors, 1 <= s <= n (linalg.py:129-166)."""

    __slots__ = ("_host", "_dev", "orthonormal", "n", "s")

    def __init__(self, entries, orthonormal=False):
        if isinstance(entries, VectorBlock):
            host, block = entries._host, entries._dev
            n, s = entries.n, entries.s
        elif isinstance(entries, torch.Tensor):
            host, block = None, entries if entries.dim() == 2 else entries.reshape(1, -1)
            n, s = block.shape[1], block.shape[0]
        else:
            a = np.array(_asarray(entries), order="F")
            if a.ndim == 1:
                a = a.reshape(-1, 1)
            if a.ndim != 2:
                raise ContractViolation(f"expected a 2-d block, got ndim={a.ndim}")
            a.setflags(write=False)
            host, block = a, None
            n, s = a.shape
        if not 1 <= s <= n:
            raise ContractViolation(f"block shape {(n, s)} violates 1 <= s <= n")
        self._init_storage(host, block)
        object.__setattr__(self, "n", n)
        object.__setattr__(self, "s", s)
        if orthonormal:
            if block is not None:
                devn = _orth_deviation(block)
            else:
                devn = np.linalg.norm(host.conj().T @ host - np.eye(s))
            if devn > 1e-12 * np.sqrt(s):
                raise ContractViolation(
                    f"block flagged orthonormal but ||Q^H Q - I|| = {devn:.3e}")
        object.__setattr__(self, "orthonormal", bool(orthonormal))

    def __setattr__(self, k, v):
        raise AttributeError("VectorBlock is immutable")

    def __repr__(self):
        return f"VectorBlock(n={self.n}, s={self.s}, orthonormal={self.orthonormal})"


class LowerTriangularFactor(_DeviceBacked):
    """Lower-triangular factor with real positive diagonal (linalg.py:169-191)."""

    __slots__ = ("_host", "_dev", "n")

    def __init__(self, entries, _trusted_block=None):
        if _trusted_block is not None:
            self._init_storage(None, _trusted_block)
            object.__setattr__(self, "n", _trusted_block.shape[1])
            return
        a = np.array(_asarray(entries), order="F")
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ContractViolation(f"expected a square factor, got shape {a.shape}")
        if np.linalg.norm(np.triu(a, 1)) != 0.0:
            raise ContractViolation("factor has nonzero entries above the diagonal")
        d = a.diagonal()
        if np.any(d.imag != 0.0) or np.any(d.real <= 0.0):
            raise ContractViolation("factor diagonal must be real positive")
        a.setflags(write=False)
        self._init_storage(a, None)
        object.__setattr__(self, "n", a.shape[0])

    def __setattr__(self, k, v):
        raise AttributeError("LowerTriangularFactor is immutable")

    def __repr__(self):
        return f"LowerTriangularFactor(n={self.n})"


# ----------------------------------------------------------------------
# kernels


def gemm(alpha, a, b, beta=0.0, c=None, workers=None):
    """C <- alpha A @ B + beta C on the DMMA GEMM (linalg.py:198-251).

    Host arrays in, host array out (drop-in); square-A products are tallied.
    """
    ah = a.entries if isinstance(a, (HermitianDenseMatrix, VectorBlock, LowerTriangularFactor)) else np.asarray(a, dtype=np.complex128)
    bh = b.entries if isinstance(b, (HermitianDenseMatrix, VectorBlock, LowerTriangularFactor)) else np.asarray(b, dtype=np.complex128)
    b2d = bh if bh.ndim == 2 else bh.reshape(-1, 1)
    if ah.ndim != 2 or b2d.ndim != 2 or ah.shape[1] != b2d.shape[0]:
        raise DimensionMismatch(f"gemm inner dimensions disagree: {ah.shape} x {bh.shape}")
    out_shape = (ah.shape[0], b2d.shape[1])
    if c is None:
        if beta != 0.0:
            raise ContractViolation("beta != 0 requires an explicit C operand")
        ch = None
    else:
        ch = _asarray(c)
        if ch.shape != out_shape:
            raise DimensionMismatch(f"gemm C operand has shape {ch.shape}, expected {out_shape}")
    d = default_device()
    eng = engine(d)
    m, n = out_shape
    k = ah.shape[1]
    dC = dev.to_device(ch, d) if ch is not None else dev.zeros(m, n, d)
    if alpha != 0.0:
        if ah.shape[0] == ah.shape[1]:
            _count_products(n)
        dA = to_block(a, d)
        dB = to_block(b2d if bh.ndim == 1 else b, d)
        eng.zgemm("N", "N", m, n, k, alpha, dA, dB, beta if ch is not None else 0.0, dC)
    elif ch is not None:
        eng.axpby(0.0, None, beta, dC)
    out = dev.to_host(dC)
    return out[:, 0] if bh.ndim == 1 else out


def cholesky_factor(B):
    """B = L L^H with L lower, real positive diagonal (linalg.py:254-270);
    cuSOLVER zpotrf on the device. Raises NotPositiveDefinite(pivot)."""
    if isinstance(B, HermitianDenseMatrix):
        n = B.n
        block = B.device_block().clone()
    else:
        b = _asarray(B)
        if b.ndim != 2 or b.shape[0] != b.shape[1]:
            raise ContractViolation(f"expected a square matrix, got shape {b.shape}")
        n = b.shape[0]
        block = dev.to_device(b, default_device())
    engine(block.device).cholesky(block)
    return LowerTriangularFactor(None, _trusted_block=block)


def householder_qr(Y):
    """Orthonormal basis of range(Y) (linalg.py:273-289). On the GPU this is
    CholQR2 (Householder is not a GPU-friendly algorithm); the rank test is
    the same: RankDeficient(column) when |R_jj| < 1e-14 ||Y||_F."""
    y = Y.device_block() if isinstance(Y, VectorBlock) else None
    if y is None:
        yh = _asarray(Y)
        if yh.ndim != 2:
            raise ContractViolation("householder_qr expects a 2-d block")
        y = dev.to_device(yh, default_device())
    f = y.clone()
    eng = engine(f.device)
    t = torch.empty_like(f)
    q = torch.empty_like(f)
    eng.orthonormalize(f, None, t, q, rank_tol=1e-14)
    return VectorBlock(q, orthonormal=True)


def oracle_eig(H, max_sweeps=30):
    """Full eigendecomposition, ascending (linalg.py:292-301); cuSOLVER zheevd
    on the device stands in for the reference's Jacobi oracle."""
    if isinstance(H, HermitianDenseMatrix):
        block = H.device_block().clone()
    else:
        h = _asarray(H)
        if h.ndim != 2 or h.shape[0] != h.shape[1]:
            raise ContractViolation(f"expected a square matrix, got shape {h.shape}")
        block = dev.to_device(h, default_device())
    if max_sweeps < 1 and dev.rows(block) > 1:
        # the reference's Jacobi with no sweep budget converges only if the input is
        # already diagonal to 1e-13 ||H||_F (_jacobi.py:21-28, linalg.py:312-318)
        fro = float(torch.linalg.vector_norm(block))
        off = float(torch.linalg.vector_norm(block - torch.diag_embed(torch.diagonal(block))))
        if fro > 0 and off > 1e-13 * fro:
            raise OracleNoConvergence(
                f"eigensolver: off-diagonal norm {off:.3e} above tolerance with a zero sweep "
                f"budget (n={dev.rows(block)})")
    w = engine(block.device).heevd(block)
    return w, VectorBlock(block)


def _factor_block(L):
    """Device copy of a lower-triangular factor with a zero upper triangle: like the
    reference's ztrsm/ztrmm (lower=1) only the lower triangle of a raw array is used."""
    if isinstance(L, LowerTriangularFactor):
        return L.device_block()
    return dev.to_device(np.tril(_asarray(L)), default_device())


def _inverse_factor(L):
    lb = _factor_block(L)
    n = dev.rows(lb)
    x = dev.empty(n, n, lb.device)
    engine(lb.device).trtri_lower(lb, x)
    return x


def triangular_solve(L, X, side="left", adjoint=False):
    """L^-1 X, L^-H X, X L^-1 or X L^-H (linalg.py:326-355), as a blocked
    triangular inverse followed by a DMMA GEMM."""
    if side not in ("left", "right"):
        raise ContractViolation(f"side must be 'left' or 'right', got {side!r}")
    xh = _asarray(X)
    x2d = xh if xh.ndim == 2 else xh.reshape(-1, 1)
    ln = L.n if isinstance(L, LowerTriangularFactor) else _asarray(L).shape[0]
    need = x2d.shape[0] if side == "left" else x2d.shape[1]
    if ln != need:
        raise DimensionMismatch(
            f"triangular_solve: factor order {ln} does not match block shape {x2d.shape} "
            f"on side {side!r}")
    out = dev.to_host(solve_triangular_device(L, to_block(x2d), side, adjoint))
    return out[:, 0] if xh.ndim == 1 else out


def solve_triangular_device(L, xb, side="left", adjoint=False, linv=None):
    """Device version: returns a new block op(L)^-1 X or X op(L)^-1."""
    linv = _inverse_factor(L) if linv is None else linv
    eng = engine(xb.device)
    m, n = dev.rows(xb), dev.cols(xb)
    out = dev.empty(m, n, xb.device)
    # linv is lower triangular with a zero upper triangle: skip its zero blocks
    if side == "left":
        eng.zgemm("C" if adjoint else "N", "N", m, n, m, 1.0, linv, xb, 0.0, out,
                  tri=eng.TRI_A_UPPER if adjoint else eng.TRI_A_LOWER)
    else:
        eng.zgemm("N", "C" if adjoint else "N", m, n, n, 1.0, xb, linv, 0.0, out,
                  tri=eng.TRI_B_UPPER if adjoint else eng.TRI_B_LOWER)
    return out


def trmm_adjoint(L, X):
    """L^H @ X (linalg.py:358-366)."""
    xh = _asarray(X)
    ln = L.n if isinstance(L, LowerTriangularFactor) else _asarray(L).shape[0]
    if ln != xh.shape[0]:
        raise DimensionMismatch(f"trmm: factor order {ln} vs block rows {xh.shape[0]}")
    x2d = xh if xh.ndim == 2 else xh.reshape(-1, 1)
    xb = to_block(x2d)
    lb = _factor_block(L)
    out = dev.empty(dev.rows(xb), dev.cols(xb), xb.device)
    eng = engine(xb.device)
    eng.zgemm("C", "N", ln, dev.cols(xb), ln, 1.0, lb, xb, 0.0, out, tri=eng.TRI_A_UPPER)
    res = dev.to_host(out)
    return res[:, 0] if xh.ndim == 1 else res
