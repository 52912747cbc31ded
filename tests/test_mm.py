"""Matrix Market exchange (matrix_market.hpp:11-19), host-side
in libairg_b200.so: byte-identical files and bit-identical matrices against
the reference's own read_matrix_market / write_matrix_market (oracle/_ref),
including duplicate entries (summed in the order SparseMatrix::from_triplets
sums them), comments, blank lines and the reference's error messages."""
import os

import numpy as np
import pytest

import refpy
from backends import same_bits
from paper_2408_08262_b200 import airg, problems


@pytest.fixture(scope="module")
def ref():
    r = refpy.ref()
    if r is None:
        pytest.skip("reference build (oracle/_ref) not available")
    return r


def _sm(p):
    return airg.SparseMatrix.from_arrays(p.n, p.n, p.row_offsets, p.cols, p.vals)


def _same(a, rp, ci, v):
    assert np.array_equal(a.row_offsets, rp) and np.array_equal(a.col_indices, ci)
    assert same_bits(a.values, v)


def test_write_byte_identical_and_round_trip(ref, tmp_path):
    p = problems.make(0)
    ours, theirs = tmp_path / "ours.mtx", tmp_path / "theirs.mtx"
    airg.write_matrix_market(_sm(p), ours)
    ref.mm_write(ref.mat_from_problem(p), str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()
    back = airg.read_matrix_market(ours)
    _same(back, p.row_offsets, p.cols, p.vals)  # %.17g: exact round trip


def test_read_matches_reference_with_duplicates(ref, tmp_path):
    rng = np.random.default_rng(3)
    n, m, k = 50, 40, 900  # many duplicates, unsorted, mixed magnitudes
    rows = rng.integers(1, n + 1, k)
    cols = rng.integers(1, m + 1, k)
    vals = rng.standard_normal(k) * 10.0 ** rng.integers(-8, 8, k)
    f = tmp_path / "dup.mtx"
    with open(f, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate REAL general\n% a comment\n\n%another\n")
        fh.write(f"{n} {m} {k}\n")
        for r, c, v in zip(rows, cols, vals):
            fh.write(f"{r}  {c}\t{float(v)!r}\n")
    a = airg.read_matrix_market(f)
    rn, rm, rp, ci, v = ref.mm_read(str(f))
    assert (a.nrows, a.ncols) == (n, m) == (rn, rm)
    _same(a, rp, ci, v)


@pytest.mark.parametrize("body,msg", [
    ("", "empty file"),
    ("%%MatrixMarket vector coordinate real general\n1 1 0\n", "malformed header"),
    ("%%MatrixMarket matrix array real general\n1 1\n1.0\n", "unsupported format"),
    ("%%MatrixMarket matrix coordinate real general\n2 2\n", "malformed size line"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "truncated entry list"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "index out of bounds at entry 1"),
])
def test_errors_match_reference(ref, tmp_path, body, msg):
    f = tmp_path / "bad.mtx"
    f.write_text(body)
    with pytest.raises(airg.AirgRuntimeError, match=msg) as ours:
        airg.read_matrix_market(f)
    with pytest.raises(refpy.OracleError) as theirs:
        ref.mm_read(str(f))
    assert str(ours.value) == str(theirs.value)


def test_missing_file(tmp_path):
    with pytest.raises(airg.AirgRuntimeError, match="cannot open for reading"):
        airg.read_matrix_market(tmp_path / "nope.mtx")
