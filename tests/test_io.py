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


def _manifest_dir():
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "manifest")


def test_save_sequence_byte_identical_to_reference(tmp_path):
    """save_sequence writes the same per-cycle CHFSI-MAT1 files and manifest text as the
    reference's save_sequence (io.py:300-333; tests/golden/manifest was written by it)."""
    from paper_1305_5120_b200.io import read_payload, save_sequence
    from paper_1305_5120_b200.sequence import ProblemSequence, SequenceSpec
    ref = _manifest_dir()
    probs = []
    for ell in range(1, 4):
        a = read_payload(os.path.join(ref, f"gen_{ell:04d}_A.mat"))[1]
        b = read_payload(os.path.join(ref, f"gen_{ell:04d}_B.mat"))[1]
        probs.append((a, b))
    seq = ProblemSequence(spec=SequenceSpec(n=12, N=3, nev=3, seed=4, kind="generalized"),
                          problems=probs)
    manifest = save_sequence(seq, str(tmp_path), stem="gen")
    assert os.path.basename(manifest) == "gen_manifest.txt"
    for name in sorted(os.listdir(ref)):
        with open(os.path.join(ref, name), "rb") as f1, open(tmp_path / name, "rb") as f2:
            assert f1.read() == f2.read(), name


def test_manifest_parse_errors(tmp_path):
    from paper_1305_5120_b200.errors import ConfigError
    from paper_1305_5120_b200.io import load_sequence
    bad = tmp_path / "m.txt"
    bad.write_text("# chfsi sequence manifest\nn = 12\nbogus = 3\n")
    with pytest.raises(ConfigError, match="unknown spec key"):
        load_sequence(str(bad))


@pytest.mark.gpu
def test_load_sequence_reference_manifest_to_device():
    """load_sequence reads the reference's manifest onto the GPU; the fixed metric B of a
    generalized sequence becomes one device matrix shared by every cycle."""
    from paper_1305_5120_b200.io import load_sequence, read_payload
    seq = load_sequence(os.path.join(_manifest_dir(), "gen_manifest.txt"))
    assert seq.spec.kind == "generalized" and seq.spec.N == 3 and len(seq.problems) == 3
    bs = [b for _, b in seq.problems]
    assert bs[0] is bs[1] is bs[2]
    for ell, (a, b) in enumerate(seq.problems, start=1):
        ra = read_payload(os.path.join(_manifest_dir(), f"gen_{ell:04d}_A.mat"))[1]
        assert np.max(np.abs(a.entries - (ra + ra.conj().T) / 2)) <= 1e-15 * np.max(np.abs(ra))
