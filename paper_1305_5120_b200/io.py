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
           "normalize_phase", "save_sequence", "load_sequence"]

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


# ----------------------------------------------------------------------
# sequence manifests (reference io.py:300-368): one CHFSI-MAT1 file per cycle matrix
# plus a text manifest with the SequenceSpec fields and the cycle -> file map; the same
# file names and manifest text as the reference, so either side reads the other's.

_SPEC_TYPES = {"n": int, "N": int, "nev": int, "delta0": float, "rho": float, "seed": int,
               "kind": str, "vary_b": bool, "band_max": float, "gap": float, "spread": float}


def save_sequence(seq, directory, stem="cycle"):
    """Write every cycle of a ProblemSequence (<stem>_0001_A.mat, + _B.mat for generalized
    problems) and <stem>_manifest.txt; returns the manifest path. A matrix shared by
    consecutive cycles (a fixed B) is written once per cycle, as by the reference."""
    from dataclasses import fields
    os.makedirs(directory, exist_ok=True)
    spec = seq.spec
    lines = ["# chfsi sequence manifest"]
    for f in fields(spec):
        lines.append(f"{f.name} = {getattr(spec, f.name)}")
    for ell, (a_mat, b_mat) in enumerate(seq.problems, start=1):
        a_name = f"{stem}_{ell:04d}_A.mat"
        write_matrix(os.path.join(directory, a_name), a_mat, kind="hermitian")
        if b_mat is None:
            lines.append(f"cycle {ell}: {a_name}")
        else:
            b_name = f"{stem}_{ell:04d}_B.mat"
            write_matrix(os.path.join(directory, b_name), b_mat, kind="spd")
            lines.append(f"cycle {ell}: {a_name} {b_name}")
    manifest = os.path.join(directory, f"{stem}_manifest.txt")
    with open(manifest, "w", encoding="utf-8") as fh:
        fh.write("\n".join(lines) + "\n")
    return manifest


def load_sequence(manifest_path, device=None):
    """Rebuild a ProblemSequence from a manifest: every matrix goes straight from its file
    into pinned memory and HBM (read_matrix); B files with identical bytes (a fixed
    metric) become ONE device matrix, so its Cholesky factor is computed once for the
    whole sequence (solve_generalized caches it on the object)."""
    import hashlib

    from .errors import ConfigError
    from .sequence import ProblemSequence, SequenceSpec
    base = os.path.dirname(os.path.abspath(manifest_path))
    spec_vals, cycles = {}, []
    with open(manifest_path, "r", encoding="utf-8") as fh:
        for line in fh:
            body = line.split("#", 1)[0].strip()
            if not body:
                continue
            if body.startswith("cycle "):
                idx, names = body[len("cycle "):].split(":", 1)
                cycles.append((int(idx), names.split()))
            elif "=" in body:
                key, raw = (t.strip() for t in body.split("=", 1))
                if key not in _SPEC_TYPES:
                    raise ConfigError(f"manifest: unknown spec key {key!r}")
                typ = _SPEC_TYPES[key]
                spec_vals[key] = raw.lower() in ("true", "yes", "1") if typ is bool else typ(raw)
    spec = SequenceSpec(**spec_vals)
    cycles.sort()
    problems, shared = [], {}
    for _, names in cycles:
        a_mat = read_matrix(os.path.join(base, names[0]), device=device)
        b_mat = None
        if len(names) > 1:
            path = os.path.join(base, names[1])
            h = hashlib.sha256()
            with open(path, "rb") as fb:
                for chunk in iter(lambda: fb.read(1 << 24), b""):
                    h.update(chunk)
            key = h.hexdigest()
            if key not in shared:
                shared[key] = read_matrix(path, device=device)
            b_mat = shared[key]
        problems.append((a_mat, b_mat))
    if len(problems) != spec.N:
        raise ConfigError(f"manifest lists {len(problems)} cycles but spec says N = {spec.N}")
    return ProblemSequence(spec=spec, problems=problems)
