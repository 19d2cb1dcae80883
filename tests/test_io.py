"""CHFSI-MAT1 interchange (reference io.py:46-144) against files written by the
reference itself (tests/golden/*.chfsi, scripts/make_golden.py::gen_io)."""

import os

import numpy as np
import pytest

from paper_1305_5120_b200 import io as cio
from paper_1305_5120_b200.errors import BadMagic, ContractViolation, MatrixFileError, \
    SymmetryViolation, TruncatedPayload

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def meta():
    return np.load(os.path.join(GOLD, "io_meta.npz"))


@pytest.mark.parametrize("name,kind,key", [("herm7.chfsi", "hermitian", "herm"),
                                           ("block9x3.chfsi", "block", "block"),
                                           ("spd5.chfsi", "spd", "spd")])
def test_reads_reference_files_bit_exact(name, kind, key):
    k, arr = cio.read_payload(os.path.join(GOLD, name))
    assert k == kind
    assert arr.flags.f_contiguous
    assert np.array_equal(arr, meta()[key])


@pytest.mark.parametrize("name,kind,key", [("herm7.chfsi", "hermitian", "herm"),
                                           ("block9x3.chfsi", "block", "block"),
                                           ("spd5.chfsi", "spd", "spd")])
def test_writer_is_byte_identical_to_reference(tmp_path, name, kind, key):
    p = tmp_path / name
    cio.write_matrix(p, meta()[key], kind=kind)
    assert p.read_bytes() == open(os.path.join(GOLD, name), "rb").read()


def test_header_errors(tmp_path):
    bad = tmp_path / "bad.chfsi"
    bad.write_bytes(b"NOT-A-MATRIX-FILE-AT-ALL-xxxxxxxx")
    with pytest.raises(BadMagic):
        cio.read_header(bad)
    good = open(os.path.join(GOLD, "herm7.chfsi"), "rb").read()
    trunc = tmp_path / "trunc.chfsi"
    trunc.write_bytes(good[:-16])
    with pytest.raises(TruncatedPayload) as exc:
        cio.read_header(trunc)
    assert exc.value.expected == 16 * 49 and exc.value.actual == 16 * 48 and exc.value.offset == 27
    kindless = tmp_path / "kind.chfsi"
    kindless.write_bytes(good[:10] + b"X" + good[11:])
    with pytest.raises(MatrixFileError):
        cio.read_header(kindless)
    with pytest.raises(ContractViolation):
        cio.write_matrix(tmp_path / "x.chfsi", np.ones((2, 3), dtype=complex), kind="hermitian")
    with pytest.raises(ContractViolation):
        cio.write_matrix(tmp_path / "x.chfsi", np.ones(3, dtype=complex))


def test_payload_into_preallocated_buffer():
    buf = np.empty((9, 3), dtype=np.complex128, order="F")
    kind, out = cio.read_payload(os.path.join(GOLD, "block9x3.chfsi"), out=buf)
    assert out is buf and np.array_equal(buf, meta()["block"])


def test_normalize_phase_matches_reference():
    got = cio.normalize_phase(meta()["block"])
    assert np.array_equal(got, meta()["block_phase"])


@pytest.mark.gpu
def test_read_matrix_onto_device(tmp_path):
    import paper_1305_5120_b200 as G
    h = cio.read_matrix(os.path.join(GOLD, "herm7.chfsi"))
    assert isinstance(h, G.HermitianDenseMatrix) and h.n == 7
    ref = meta()["herm"]
    assert np.array_equal(h.entries, ref)  # already exactly Hermitian: symmetrising is exact
    b = cio.read_matrix(os.path.join(GOLD, "block9x3.chfsi"))
    assert isinstance(b, G.VectorBlock) and (b.n, b.s) == (9, 3)
    assert np.array_equal(b.entries, meta()["block"])
    skew = np.array(ref)
    skew[0, 1] += 1.0
    p = tmp_path / "skew.chfsi"
    cio.write_matrix(p, skew)
    with pytest.raises(SymmetryViolation):
        cio.read_matrix(p)
