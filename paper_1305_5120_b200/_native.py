"""ctypes binding of libchfsi_b200.so (include/chfsi_b200.h).

This is the only way the package reaches the GPU. There is no fallback: if
the shared library is missing or cannot be loaded the import of this module
raises, and every solver entry point fails loudly.
"""

import ctypes
import os

from .errors import ChfsiError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CHFSI_LIB") or os.path.join(_HERE, "_lib", "libchfsi_b200.so")

# status codes (include/chfsi_b200.h)
ERR_ARG = -1
ERR_CUDA = -2
ERR_CUSOLVER = -3
ERR_NOT_PD = -4
ERR_RANK = -5
ERR_NOMEM = -6

_c_void_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double
_pdbl = ctypes.POINTER(ctypes.c_double)
_pint = ctypes.POINTER(ctypes.c_int)
_pi64 = ctypes.POINTER(ctypes.c_int64)

# name -> (restype, argtypes); the complete exported surface of the header
SIGNATURES = {
    "chfsi_abi_version": (_int, []),
    "chfsi_last_error": (ctypes.c_char_p, []),
    "chfsi_create": (_int, [_int, _c_void_p, ctypes.POINTER(_c_void_p)]),
    "chfsi_destroy": (_int, [_c_void_p]),
    "chfsi_set_stream": (_int, [_c_void_p, _c_void_p]),
    "chfsi_synchronize": (_int, [_c_void_p]),
    "chfsi_launch_count": (ctypes.c_longlong, [_c_void_p, _int]),
    "chfsi_zgemm": (_int, [_c_void_p, _int, _int, _i64, _i64, _i64, _dbl, _dbl, _c_void_p, _i64,
                            _c_void_p, _i64, _dbl, _dbl, _c_void_p, _i64]),
    "chfsi_zgemm_tri": (_int, [_c_void_p, _int, _int, _i64, _i64, _i64, _dbl, _dbl, _c_void_p,
                                _i64, _c_void_p, _i64, _dbl, _dbl, _c_void_p, _i64, _int, _i64]),
    "chfsi_filter": (_int, [_c_void_p, _i64, _i64, _int, _dbl, _dbl, _dbl, _c_void_p, _i64,
                             _c_void_p, _i64, _c_void_p, _i64, _pint]),
    "chfsi_filter_streamed": (_int, [_c_void_p, _i64, _i64, _int, _dbl, _dbl, _dbl, _c_void_p,
                                      _i64, _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _i64,
                                      _int, _pint]),
    "chfsi_filter_streamed_to_host": (_int, [_c_void_p, _i64, _i64, _int, _dbl, _dbl, _dbl,
                                              _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _i64,
                                              _c_void_p, _i64, _int, _c_void_p, _i64, _pint]),
    "chfsi_filter_step": (_int, [_c_void_p, _i64, _i64, _c_void_p, _i64, _c_void_p, _i64, _dbl,
                                  _dbl, _c_void_p, _i64, _dbl, _c_void_p, _i64]),
    "chfsi_lanczos_bound": (_int, [_c_void_p, _i64, _int, _c_void_p, _i64, _c_void_p, _pdbl,
                                    _pdbl, _pint, _pdbl]),
    "chfsi_orthonormalize": (_int, [_c_void_p, _i64, _i64, _c_void_p, _i64, _c_void_p, _i64,
                                     _i64, _c_void_p, _i64, _c_void_p, _i64, _dbl, _pi64, _pdbl]),
    "chfsi_rayleigh_ritz": (_int, [_c_void_p, _i64, _i64, _c_void_p, _i64, _c_void_p, _i64,
                                    _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _i64, _pdbl,
                                    _pdbl]),
    "chfsi_rayleigh_ritz_from_hq": (_int, [_c_void_p, _i64, _i64, _c_void_p, _i64, _c_void_p,
                                            _i64, _c_void_p, _i64, _c_void_p, _i64, _pdbl,
                                            _pdbl]),
    "chfsi_project_out": (_int, [_c_void_p, _i64, _i64, _c_void_p, _i64, _c_void_p, _i64,
                                  _i64]),
    "chfsi_residual_norms": (_int, [_c_void_p, _i64, _i64, _c_void_p, _i64, _c_void_p, _i64,
                                     _pdbl, _pdbl]),
    "chfsi_hermitian_norms": (_int, [_c_void_p, _i64, _c_void_p, _i64, _pdbl]),
    "chfsi_hermitize": (_int, [_c_void_p, _i64, _c_void_p, _i64]),
    "chfsi_cholesky": (_int, [_c_void_p, _i64, _c_void_p, _i64, _pint]),
    "chfsi_cholesky_inverse": (_int, [_c_void_p, _i64, _c_void_p, _i64, _dbl, _c_void_p, _i64,
                                       _pdbl, _pdbl, _pint]),
    "chfsi_reduce_to_standard": (_int, [_c_void_p, _i64, _c_void_p, _i64, _c_void_p, _i64,
                                         _c_void_p, _i64, _c_void_p, _i64]),
    "chfsi_trtri_lower": (_int, [_c_void_p, _i64, _c_void_p, _i64, _c_void_p, _i64]),
    "chfsi_heevd": (_int, [_c_void_p, _i64, _c_void_p, _i64, _pdbl]),
    "chfsi_axpby": (_int, [_c_void_p, _i64, _i64, _dbl, _dbl, _c_void_p, _i64, _dbl, _dbl,
                            _c_void_p, _i64]),
    "chfsi_gemm_override": (_int, [_int, _int]),
    "chfsi_set_complex_mul": (_int, [_int]),
    "chfsi_get_complex_mul": (_int, []),
    "chfsi_declare_operator": (_int, [_c_void_p, _i64, _c_void_p, _i64]),
    "chfsi_apply_operator": (_int, [_c_void_p, _i64, _i64, _c_void_p, _i64, _c_void_p, _i64,
                                     _c_void_p, _i64]),
    "chfsi_gemm_plan": (_int, [_c_void_p, _int, _int, _int, _i64, _i64, _i64, _pint, _pint]),
    "chfsi_peak_dmma": (_int, [_int, _int, _pdbl]),
    "chfsi_peak_dfma": (_int, [_int, _int, _pdbl]),
    "chfsi_upload": (_int, [_c_void_p, _c_void_p, _i64, _i64, _i64, _c_void_p, _i64]),
    "chfsi_comm_available": (_int, [_pint]),
    "chfsi_comm_init_all": (_int, [_int, _pint, ctypes.POINTER(_c_void_p)]),
    "chfsi_comm_destroy": (_int, [_c_void_p]),
    "chfsi_comm_abort": (_int, [_c_void_p]),
    "chfsi_comm_allgather": (_int, [_c_void_p, _c_void_p, _c_void_p, ctypes.c_size_t, _c_void_p]),
    "chfsi_comm_broadcast": (_int, [_c_void_p, _c_void_p, ctypes.c_size_t, _int, _c_void_p]),
}


class NativeError(ChfsiError):
    """A call into libchfsi_b200.so failed (CUDA / cuSOLVER / allocation)."""

    def __init__(self, fn, status, message):
        self.fn = fn
        self.status = int(status)
        super().__init__(f"{fn} failed with status {status}: {message}")


_lib = None


def load():
    """Load the native library once; raises if it is absent (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libchfsi_b200.so not found at {LIB_PATH}; build it with "
            f"`python -c 'import __graft_entry__ as g; g.build()'` or "
            f"`make -C paper_1305_5120_b200/csrc`"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.chfsi_abi_version() != 1:
        raise ImportError("libchfsi_b200.so ABI version mismatch")
    _lib = lib
    return lib


def last_error():
    return load().chfsi_last_error().decode("utf-8", "replace")


def check(fn_name, status):
    if status != 0:
        raise NativeError(fn_name, status, last_error())
    return status


def call(fn_name, *args):
    """Call an exported function and raise NativeError on a nonzero status."""
    return check(fn_name, getattr(load(), fn_name)(*args))
