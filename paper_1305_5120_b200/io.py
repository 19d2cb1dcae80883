"""CHFSI-MAT1 matrix interchange (reference pkg/src/chfsi/io.py:46-127), GPU-bound.

File layout (little endian): 10-byte magic ``CHFSI-MAT1``, 1 kind byte (H =
hermitian, S = spd, B = block), uint64 rows, uint64 cols, then the column-major
complex128 payload -- exactly the numpy F-order / device block layout, so a
read is one file read into pinned host memory and one DMA to HBM; the
Hermitian check and symmetrisation run on the GPU (hermitian_norms /
hermitize kernels). Files are byte-compatible with the reference's
write_matrix/read_matrix (tests/golden/*.chfsi were written by the reference).
"""

import os
import struct

import numpy as np

from .errors import BadMagic, ContractViolation, MatrixFileError, SymmetryViolation, TruncatedPayload

__all__ = ["MAGIC", "write_matrix", "read_matrix", "read_header", "read_payload",
           "normalize_phase"]

MAGIC = b"CHFSI-MAT1"
KIND_BYTES = {"hermitian": b"H", "spd": b"S", "block": b"B"}
BYTE_KINDS = {v: k for k, v in KIND_BYTES.items()}
HEADER = struct.Struct("<10scQQ")  # 27 bytes


def read_header(path):
    """(kind, rows, cols) of a CHFSI-MAT1 file; validates magic, kind and payload size."""
    spath = str(path)
    size = os.path.getsize(spath)
    with open(spath, "rb") as fh:
        head = fh.read(HEADER.size)
    if len(head) < HEADER.size or head[: len(MAGIC)] != MAGIC:
        raise BadMagic(f"{spath}: expected magic {MAGIC!r} at offset 0")
    _, kind_byte, n, s = HEADER.unpack(head)
    if kind_byte not in BYTE_KINDS:
        raise MatrixFileError(f"{spath}: unknown kind byte {kind_byte!r}")
    expected = 16 * n * s
    actual = size - HEADER.size
    if actual != expected:
        raise TruncatedPayload(expected, actual, HEADER.size)
    return BYTE_KINDS[kind_byte], int(n), int(s)


def read_payload(path, out=None):
    """Payload as an F-order (rows, cols) complex128 array. ``out`` may be a
    preallocated (e.g. pinned) buffer of the right size, filled in place."""
    kind, n, s = read_header(path)
    if out is None:
        out = np.empty((n, s), dtype=np.complex128, order="F")
    flat = out.reshape(-1, order="F") if out.flags.f_contiguous else None
    if flat is None or flat.size != n * s:
        raise ContractViolation("payload buffer must be an F-contiguous (rows, cols) complex128 array")
    with open(str(path), "rb") as fh:
        fh.seek(HEADER.size)
        view = memoryview(flat.view(np.uint8))
        got = fh.readinto(view)
    if got != 16 * n * s:
        raise TruncatedPayload(16 * n * s, got, HEADER.size)
    if not np.little_endian:  # pragma: no cover
        out.byteswap(inplace=True)
    return kind, out


def write_matrix(path, m, kind=None):
    """Write a matrix or block (reference io.py:52-70 semantics)."""
    from .linalg import HermitianDenseMatrix, LowerTriangularFactor, VectorBlock
    if isinstance(m, (HermitianDenseMatrix, VectorBlock, LowerTriangularFactor)):
        arr = m.entries
    else:
        arr = np.asarray(m, dtype=np.complex128)
    if arr.ndim != 2:
        raise ContractViolation("only 2-d matrices/blocks can be written")
    if kind is None:
        kind = "block" if isinstance(m, VectorBlock) else "hermitian"
    if kind not in KIND_BYTES:
        raise ContractViolation(f"unknown matrix kind {kind!r}")
    if kind in ("hermitian", "spd") and arr.shape[0] != arr.shape[1]:
        raise ContractViolation(f"kind {kind!r} requires a square matrix")
    n, s = arr.shape
    with open(str(path), "wb") as fh:
        fh.write(HEADER.pack(MAGIC, KIND_BYTES[kind], n, s))
        fh.write(np.asarray(arr, dtype="<c16").tobytes(order="F"))


def read_matrix(path, device=None):
    """Read a CHFSI-MAT1 file (or Matrix-Market text for .mtx/.mm) onto the GPU.

    hermitian/spd -> HermitianDenseMatrix (deviation > 1e-10 relative raises
    SymmetryViolation), block -> VectorBlock (reference io.py:73-127).
    """
    import torch

    from . import device as dev
    from .linalg import HermitianDenseMatrix, VectorBlock, default_device, engine
    spath = str(path)
    device = device if device is not None else default_device()
    if spath.endswith(".mtx") or spath.endswith(".mm"):
        import scipy.io
        m = scipy.io.mmread(spath)
        arr = np.asarray(m.todense() if hasattr(m, "todense") else m, dtype=np.complex128)
        if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
            raise MatrixFileError(f"{spath}: expected a square matrix")
        kind = "hermitian"
        block = dev.to_device(arr, device)
    else:
        kind, n, s = read_header(spath)
        if kind != "block" and n != s:
            raise MatrixFileError(f"{spath}: kind {kind!r} payload is not square")
        # pinned staging buffer (s, n) whose numpy view is the F-order (n, s) payload
        pinned = torch.empty((s, n), dtype=torch.complex128, pin_memory=True)
        read_payload(spath, pinned.numpy().T)
        block = torch.empty((s, n), dtype=torch.complex128, device=device)
        block.copy_(pinned, non_blocking=True)
        torch.cuda.current_stream(device).synchronize()
        if kind == "block":
            return VectorBlock(block)
    scale, devn = engine(block.device).hermitian_norms(block)
    if scale > 0 and devn > 1e-10 * scale:
        raise SymmetryViolation(f"{spath}: Hermitian deviation {devn:.3e} exceeds 1e-10 * ||M||")
    return HermitianDenseMatrix(block, rtol=np.inf)


def normalize_phase(block):
    """Rotate each column so its largest-magnitude entry is real positive
    (reference io.py:130-144); host arrays, used for reproducible output files."""
    from .linalg import VectorBlock
    arr = np.array(block.entries if isinstance(block, VectorBlock) else block,
                   dtype=np.complex128, order="F")
    arr2 = arr if arr.ndim == 2 else arr.reshape(-1, 1)
    for j in range(arr2.shape[1]):
        i = int(np.argmax(np.abs(arr2[:, j])))
        pivot = arr2[i, j]
        mag = abs(pivot)
        if mag > 0:
            arr2[:, j] *= np.conj(pivot) / mag
            arr2[i, j] = mag  # exactly real
    return arr2 if arr.ndim == 2 else arr2[:, 0]
