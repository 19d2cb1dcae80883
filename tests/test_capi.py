"""The C-ABI library loads without a GPU and exports exactly what include/chfsi_b200.h
declares; the ctypes signature table covers every declared entry point. No compute
calls (CPU box)."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "chfsi_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(chfsi_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_solver_surface():
    names = declared_functions()
    for must in ("chfsi_create", "chfsi_zgemm", "chfsi_filter", "chfsi_filter_step",
                 "chfsi_lanczos_bound", "chfsi_orthonormalize", "chfsi_rayleigh_ritz",
                 "chfsi_residual_norms", "chfsi_cholesky", "chfsi_trtri_lower", "chfsi_heevd",
                 "chfsi_hermitian_norms", "chfsi_hermitize"):
        assert must in names


def test_library_loads_and_exports_every_symbol():
    from paper_1305_5120_b200 import _native
    lib = _native.load()
    assert lib.chfsi_abi_version() == 1
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)


def test_ctypes_table_matches_header():
    from paper_1305_5120_b200 import _native
    assert sorted(_native.SIGNATURES) == declared_functions()


def test_null_handle_is_a_contract_error():
    from paper_1305_5120_b200 import _native
    lib = _native.load()
    st = lib.chfsi_zgemm(None, 0, 0, 1, 1, 1, 1.0, 0.0, None, 1, None, 1, 0.0, 0.0, None, 1)
    assert st == _native.ERR_ARG
    assert "null" in _native.last_error()


def test_no_cpu_fallback_when_library_missing(tmp_path, monkeypatch):
    import pytest
    from paper_1305_5120_b200 import _native
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        _native.load()
