"""Shared test setup: the `gpu` marker, import paths and seeded generators.

`-m "not gpu"` tests run on the CPU-only build box (oracle vs golden vectors,
host logic, C-ABI symbol table, gloo multi-process plumbing). `-m gpu` tests
are the parity tests proper: they call the CUDA path through the C ABI and
compare with the oracle (oracle/chfsi_oracle.py), which only tests may import.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the native kernels)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def rand_hermitian(rng, n, scale=1.0):
    g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return ((g + g.conj().T) / 2.0) * (scale / np.sqrt(n))


def spectrum_matrix(rng, evals):
    evals = np.asarray(evals, dtype=np.float64)
    n = evals.size
    q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    return (q * evals) @ q.conj().T


def rand_spd(rng, n, shift=None):
    m = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    b = m.conj().T @ m + (n if shift is None else shift) * np.eye(n)
    return (b + b.conj().T) / 2.0


def gapped_matrix(seed, n, nev, lo=4.0, hi_lo=6.0, hi=10.0):
    rng = np.random.default_rng(seed)
    evals = np.concatenate([np.sort(rng.uniform(0.0, lo, nev)),
                            np.sort(rng.uniform(hi_lo, hi, n - nev))])
    return spectrum_matrix(rng, evals), evals
