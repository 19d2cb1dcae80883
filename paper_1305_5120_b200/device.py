"""Device-side plumbing: column-major complex128 blocks in HBM and the native engine.

A column-major n x k complex128 block lives in a torch tensor of shape (k, n)
with unit stride along rows: column j is row j of the tensor, the leading
dimension is ``t.stride(0)`` and a column range ``t[a:b]`` is a zero-copy
view. This is exactly the numpy F-order layout of the reference
(linalg.py:108,121), so host<->device transfers are plain byte copies.

torch provides allocation, streams and torch.distributed; all arithmetic is
in libchfsi_b200.so, reached through :class:`Engine`.
"""

import ctypes
import threading
import warnings

import numpy as np
import torch

from . import _native
from .errors import ContractViolation, NotPositiveDefinite, RankDeficient

CDT = torch.complex128


def rows(t):
    return t.shape[-1]


def cols(t):
    return t.shape[0] if t.dim() == 2 else 1


def _check_layout(t):
    """A (k, n) block must be column-major: unit stride along rows (the kernels read
    column j at data_ptr + j * ld) and ld >= n; a transposed or strided view would be
    read with the wrong layout. Empty blocks are not read (their strides are arbitrary)."""
    if t.numel() == 0:
        return
    if t.dim() == 2 and t.shape[1] > 1 and t.stride(1) != 1:
        raise ValueError(f"block has row stride {t.stride(1)}; the kernels need unit stride "
                         f"along rows (a (cols, rows) tensor with contiguous columns)")
    if t.dim() == 2 and t.shape[0] > 1 and t.stride(0) < t.shape[1]:
        raise ValueError(f"block leading dimension {t.stride(0)} < rows {t.shape[1]}")
    if t.dim() == 1 and t.shape[0] > 1 and t.stride(0) != 1:
        raise ValueError("vector must be contiguous")


def ld(t):
    _check_layout(t)
    if t.dim() != 2:
        return t.shape[0]
    # a single column's stride is arbitrary in torch: report the row count then
    return t.stride(0) if t.shape[0] > 1 else max(t.stride(0), t.shape[1])


def ptr(t):
    """Raw device pointer for the C ABI. torch's lazy conjugate/negative views share
    storage with their source (the bit is not applied to memory), so they must be
    materialised (``resolve_conj()``) before the kernels may read them."""
    if t is None:
        return ctypes.c_void_p(0)
    if t.is_conj() or t.is_neg():
        raise ValueError("tensor has a lazy conj/neg bit; call resolve_conj()/resolve_neg() first")
    _check_layout(t)
    return ctypes.c_void_p(t.data_ptr())


def empty(n, k, device):
    return torch.empty((k, n), dtype=CDT, device=device)


def zeros(n, k, device):
    return torch.zeros((k, n), dtype=CDT, device=device)


# pageable host blocks at least this large go through the native staged upload
_STAGED_MIN_BYTES = 8 << 20


def to_device(arr, device, pin=False):
    """numpy (n,) / (n, k) complex array -> device tensor (k, n) (column-major block).
    Large pageable arrays are uploaded by chfsi_upload (pinned staging ring filled by
    host worker threads, csrc/staging.cu) instead of the driver's pageable path."""
    a = np.asarray(arr, dtype=np.complex128)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    a = np.asfortranarray(a)
    if (not pin and a.nbytes >= _STAGED_MIN_BYTES and a.size
            and torch.device(device).type == "cuda"):
        out = torch.empty((a.shape[1], a.shape[0]), dtype=CDT, device=device)
        eng = Engine.get(out.device)
        _native.call("chfsi_upload", eng.h, ctypes.c_void_p(a.ctypes.data), a.shape[0],
                     a.shape[0], a.shape[1], ctypes.c_void_p(out.data_ptr()), a.shape[0])
        return out
    with warnings.catch_warnings():
        # read-only inputs (frozen VectorBlock.entries) are only read by the H2D copy
        warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
        host = torch.from_numpy(a.T)  # (k, n) C-contiguous view of the F-order data
    if pin:
        host = host.pin_memory()
    return host.to(device, non_blocking=pin)


_PINNED_MIN_BYTES = 1 << 20


def to_host(t):
    """device tensor (k, n) -> numpy (n, k) F-order complex128 array.

    Large results land in page-locked memory (torch's caching host allocator):
    on the B200 box a device->pageable copy ran at 2.2 GB/s, device->pinned at
    56.6 GB/s (scripts/h2d_probe.py). The numpy array views the pinned buffer."""
    t = t.detach()
    if t.is_cuda and t.numel() * t.element_size() >= _PINNED_MIN_BYTES:
        host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        host.copy_(t)
        return np.asfortranarray(host.numpy().T)
    return np.asfortranarray(t.to("cpu").numpy().T)


_tls = threading.local()


def set_engine_tag(tag):
    """Engines are per (device, tag); the in-process multi-GPU runner (comm.py) gives
    each rank thread its own tag, so ranks never share a handle's scratch arenas (two
    ranks may even share one GPU in the tests)."""
    _tls.tag = int(tag)


def engine_tag():
    return getattr(_tls, "tag", 0)


class Engine:
    """Native handle bound to one CUDA device and torch's current stream there."""

    _engines = {}
    _lock = threading.Lock()

    def __init__(self, device):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1305_5120_b200 needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device)
        self.index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.device = torch.device("cuda", self.index)
        self.lib = _native.load()
        with torch.cuda.device(self.index):
            self.stream = torch.cuda.current_stream(self.index)
        h = ctypes.c_void_p()
        _native.check("chfsi_create",
                      self.lib.chfsi_create(self.index, ctypes.c_void_p(self.stream.cuda_stream),
                                            ctypes.byref(h)))
        self.h = h

    @classmethod
    def get(cls, device=None):
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        device = torch.device(device)
        idx = device.index if device.index is not None else torch.cuda.current_device()
        key = (idx, engine_tag())
        eng = cls._engines.get(key)
        cur = torch.cuda.current_stream(idx)
        if eng is None:
            with cls._lock:
                eng = cls._engines.get(key)
                if eng is None:
                    eng = cls(torch.device("cuda", idx))
                    cls._engines[key] = eng
        if eng.stream.cuda_stream != cur.cuda_stream:
            eng.stream = cur
            _native.call("chfsi_set_stream", eng.h, ctypes.c_void_p(cur.cuda_stream))
        return eng

    # ------------------------------------------------------------ counters
    def launch_count(self, reset=False):
        return int(self.lib.chfsi_launch_count(self.h, 1 if reset else 0))

    def synchronize(self):
        _native.call("chfsi_synchronize", self.h)

    # ------------------------------------------------------------ kernels
    # triangular-operand flags of chfsi_zgemm_tri (include/chfsi_b200.h)
    TRI_A_LOWER, TRI_B_UPPER, TRI_B_LOWER, TRI_A_UPPER, TRI_C_LOWER = 1, 2, 4, 8, 16

    def zgemm(self, opa, opb, m, n, k, alpha, A, B, beta, C, tri=0, tri_offset=0):
        """C = alpha op(A) op(B) + beta C on column-major blocks (op: 'N' or 'C').
        ``tri``: triangular-operand flag (the zero blocks of the K range are skipped);
        ``tri_offset``: first row/column of C inside the triangular factor."""
        oa = 0 if opa == "N" else 1
        ob = 0 if opb == "N" else 1
        alpha = complex(alpha)
        beta = complex(beta)
        if tri:
            _native.call("chfsi_zgemm_tri", self.h, oa, ob, m, n, k, alpha.real, alpha.imag,
                         ptr(A), ld(A), ptr(B), ld(B), beta.real, beta.imag, ptr(C), ld(C),
                         int(tri), int(tri_offset))
        else:
            _native.call("chfsi_zgemm", self.h, oa, ob, m, n, k, alpha.real, alpha.imag,
                         ptr(A), ld(A), ptr(B), ld(B), beta.real, beta.imag, ptr(C), ld(C))
        return C

    def filter(self, H, Y, W, degree, a, b, lam_ref):
        """p_m(H) Y; Y is clobbered. Returns the tensor holding the result (Y or W)."""
        n, k = rows(Y), cols(Y)
        flag = ctypes.c_int(0)
        _native.call("chfsi_filter", self.h, n, k, int(degree), float(a), float(b),
                     float(lam_ref), ptr(H), ld(H), ptr(Y), ld(Y), ptr(W), ld(W),
                     ctypes.byref(flag))
        return W if flag.value else Y

    def filter_streamed(self, host_H, H, Y, W, degree, a, b, lam_ref, panels=0):
        """p_m(H) Y with H uploaded from the host F-order array ``host_H`` into the
        device block ``H`` while the first degree step runs panel by panel
        (chfsi_filter_streamed; it returns once host_H has been read, the GPU still busy);
        Y is clobbered. Returns the tensor holding the result (Y or W)."""
        if not (isinstance(host_H, np.ndarray) and host_H.dtype == np.complex128
                and host_H.flags.f_contiguous and host_H.ndim == 2):
            raise ValueError("filter_streamed: host_H must be an F-contiguous complex128 matrix")
        n, k = rows(Y), cols(Y)
        if host_H.shape != (n, n) or rows(H) != n or cols(H) != n:
            raise ValueError("filter_streamed: H must be n x n with n = rows(Y)")
        flag = ctypes.c_int(0)
        _native.call("chfsi_filter_streamed", self.h, n, k, int(degree), float(a), float(b),
                     float(lam_ref), host_H.ctypes.data, n, ptr(H), ld(H), ptr(Y), ld(Y),
                     ptr(W), ld(W), int(panels), ctypes.byref(flag))
        return W if flag.value else Y

    def filter_streamed_to_host(self, host_H, H, Y, W, degree, a, b, lam_ref, panels=0):
        """filter_streamed whose result also lands in a page-locked host array, panel by
        panel during the last degree step (chfsi_filter_streamed_to_host). Returns
        (device tensor holding the result, F-order (n, k) host array)."""
        if not (isinstance(host_H, np.ndarray) and host_H.dtype == np.complex128
                and host_H.flags.f_contiguous and host_H.ndim == 2):
            raise ValueError("filter_streamed: host_H must be an F-contiguous complex128 matrix")
        n, k = rows(Y), cols(Y)
        if host_H.shape != (n, n) or rows(H) != n or cols(H) != n:
            raise ValueError("filter_streamed: H must be n x n with n = rows(Y)")
        out = torch.empty((k, n), dtype=torch.complex128, pin_memory=True)
        flag = ctypes.c_int(0)
        _native.call("chfsi_filter_streamed_to_host", self.h, n, k, int(degree), float(a),
                     float(b), float(lam_ref), host_H.ctypes.data, n, ptr(H), ld(H), ptr(Y),
                     ld(Y), ptr(W), ld(W), int(panels), ctypes.c_void_p(out.data_ptr()), n,
                     ctypes.byref(flag))
        return (W if flag.value else Y), out.numpy().T

    @staticmethod
    def complex_mul():
        """Complex-product scheme of the TMA GEMMs: 3 (3M) or 4 real products."""
        return int(_native.load().chfsi_get_complex_mul())

    @staticmethod
    def set_complex_mul(mul):
        _native.call("chfsi_set_complex_mul", int(mul))

    def declare_operator(self, H):
        """H (device, n x n) stays unchanged until the next declaration; None clears.
        Filter calls on it reuse its 3M sum plane (chfsi_declare_operator)."""
        if H is None:
            _native.call("chfsi_declare_operator", self.h, 0, ctypes.c_void_p(0), 0)
        else:
            _native.call("chfsi_declare_operator", self.h, rows(H), ptr(H), ld(H))

    def apply_operator(self, H, X, Y):
        """Y = H X (reads H's 3M sum plane when H is the declared operator)."""
        n, k = rows(X), cols(X)
        _native.call("chfsi_apply_operator", self.h, n, k, ptr(H), ld(H), ptr(X), ld(X), ptr(Y),
                     ld(Y))
        return Y

    def filter_step(self, H, Y1, alpha, beta, Y0, gamma, C):
        n, k = rows(Y1), cols(Y1)
        _native.call("chfsi_filter_step", self.h, n, k, ptr(H), ld(H), ptr(Y1), ld(Y1),
                     float(alpha), float(beta), ptr(Y0), ld(Y0) if Y0 is not None else 0,
                     float(gamma), ptr(C), ld(C))
        return C

    def lanczos_bound(self, H, v0, steps):
        n = rows(H)
        kk = max(int(steps), 2)
        al = (ctypes.c_double * kk)()
        be = (ctypes.c_double * kk)()
        done = ctypes.c_int(0)
        bound = ctypes.c_double(0.0)
        _native.call("chfsi_lanczos_bound", self.h, n, int(steps), ptr(H), ld(H), ptr(v0), al, be,
                     ctypes.byref(done), ctypes.byref(bound))
        j = done.value
        return float(bound.value), np.array(al[:j]), np.array(be[:j])

    def orthonormalize(self, F, L, T, Q, rank_tol=1e-14):
        """CGS2 against L (may be None) + CholQR2; raises RankDeficient(column)."""
        n, k = rows(F), cols(F)
        nl = 0 if L is None else cols(L)
        bad = ctypes.c_int64(-1)
        fro = ctypes.c_double(0.0)
        st = self.lib.chfsi_orthonormalize(self.h, n, k, ptr(F), ld(F),
                                           ptr(L) if nl else ctypes.c_void_p(0),
                                           ld(L) if nl else n, nl, ptr(T), ld(T), ptr(Q), ld(Q),
                                           float(rank_tol), ctypes.byref(bad), ctypes.byref(fro))
        if st == _native.ERR_RANK:
            raise RankDeficient(int(bad.value))
        _native.check("chfsi_orthonormalize", st)
        return Q, float(fro.value)

    def rayleigh_ritz(self, H, Q, HQ, Z, HZ, residuals=False):
        """Ritz values (and, with residuals=True, ||HZ_j - w_j Z_j||) in one host sync."""
        n, k = rows(Q), cols(Q)
        w = np.empty(k, dtype=np.float64)
        res = np.empty(k, dtype=np.float64) if residuals else None
        pd = ctypes.POINTER(ctypes.c_double)
        _native.call("chfsi_rayleigh_ritz", self.h, n, k, ptr(H), ld(H), ptr(Q), ld(Q),
                     ptr(HQ), ld(HQ), ptr(Z), ld(Z), ptr(HZ), ld(HZ), w.ctypes.data_as(pd),
                     res.ctypes.data_as(pd) if residuals else None)
        return (w, res) if residuals else w

    def rayleigh_ritz_from_hq(self, Q, HQ, Z, HZ):
        """Rayleigh-Ritz given HQ = H Q: (Ritz values, residual norms), one host sync."""
        n, k = rows(Q), cols(Q)
        w = np.empty(k, dtype=np.float64)
        res = np.empty(k, dtype=np.float64)
        pd = ctypes.POINTER(ctypes.c_double)
        _native.call("chfsi_rayleigh_ritz_from_hq", self.h, n, k, ptr(Q), ld(Q), ptr(HQ), ld(HQ),
                     ptr(Z), ld(Z), ptr(HZ), ld(HZ), w.ctypes.data_as(pd), res.ctypes.data_as(pd))
        return w, res

    def project_out(self, F, L):
        """F <- F - L (L^H F), twice (CGS2); no-op when L is None."""
        if L is None or cols(L) == 0 or cols(F) == 0:
            return F
        _native.call("chfsi_project_out", self.h, rows(F), cols(F), ptr(F), ld(F), ptr(L), ld(L),
                     cols(L))
        return F

    def residual_norms(self, HY, Y, lam):
        n, k = rows(Y), cols(Y)
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        res = np.empty(k, dtype=np.float64)
        if k == 0:
            return res
        _native.call("chfsi_residual_norms", self.h, n, k, ptr(HY), ld(HY), ptr(Y), ld(Y),
                     lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                     res.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        return res

    def hermitian_norms(self, A):
        out = (ctypes.c_double * 2)()
        _native.call("chfsi_hermitian_norms", self.h, rows(A), ptr(A), ld(A), out)
        return float(out[0]), float(out[1])

    def hermitize(self, A):
        _native.call("chfsi_hermitize", self.h, rows(A), ptr(A), ld(A))
        return A

    def cholesky(self, A):
        """In-place lower Cholesky; raises NotPositiveDefinite(pivot)."""
        info = ctypes.c_int(0)
        _native.call("chfsi_cholesky", self.h, rows(A), ptr(A), ld(A), ctypes.byref(info))
        if info.value > 0:
            raise NotPositiveDefinite(info.value)
        if info.value < 0:
            raise ContractViolation(f"zpotrf: illegal argument {-info.value}")
        return A

    def cholesky_inverse(self, G, Li, shift=0.0):
        """Symmetrise G (+ shift I), factor G = L L^H in place and write Li = L^-1
        (chfsi_cholesky_inverse). Returns (diag(L), trace(G), zpotrf info)."""
        k = rows(G)
        diag = np.empty(k, dtype=np.float64)
        tr = ctypes.c_double(0.0)
        info = ctypes.c_int(0)
        _native.call("chfsi_cholesky_inverse", self.h, k, ptr(G), ld(G), float(shift), ptr(Li),
                     ld(Li), diag.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                     ctypes.byref(tr), ctypes.byref(info))
        return diag, float(tr.value), int(info.value)

    def reduce_to_standard(self, A, Linv, W, H):
        """H = Linv A Linv^H (chfsi_reduce_to_standard); W is an n x n work block."""
        n = rows(A)
        _native.call("chfsi_reduce_to_standard", self.h, n, ptr(A), ld(A), ptr(Linv), ld(Linv),
                     ptr(W), ld(W), ptr(H), ld(H))
        return H

    def trtri_lower(self, L, X):
        _native.call("chfsi_trtri_lower", self.h, rows(L), ptr(L), ld(L), ptr(X), ld(X))
        return X

    def heevd(self, A):
        n = rows(A)
        w = np.empty(n, dtype=np.float64)
        _native.call("chfsi_heevd", self.h, n, ptr(A), ld(A),
                     w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        return w

    def axpby(self, alpha, X, beta, Y):
        alpha = complex(alpha)
        beta = complex(beta)
        _native.call("chfsi_axpby", self.h, rows(Y), cols(Y), alpha.real, alpha.imag,
                     ptr(X), ld(X) if X is not None else 0, beta.real, beta.imag, ptr(Y), ld(Y))
        return Y


def peak_dmma_tflops(device=0, iters=20000):
    v = ctypes.c_double(0.0)
    _native.call("chfsi_peak_dmma", int(device), int(iters), ctypes.byref(v))
    return float(v.value)


def peak_dfma_tflops(device=0, iters=20000):
    v = ctypes.c_double(0.0)
    _native.call("chfsi_peak_dfma", int(device), int(iters), ctypes.byref(v))
    return float(v.value)
