"""CPU tier for problem setup (matio.py:104-217): the
native Matrix Market parser and the Jacobi scaling against the reference's
own outputs on synthetic files (tests/golden/mm, oracle/make_golden.py
gen_matio) -- bit for bit -- and the reference's parser tests
(test_matio.py) restated."""

import os

import numpy as np
import pytest

from conftest import ROOT, golden
from paper_1908_04081_b200 import SparseMatrix
from paper_1908_04081_b200.matio import (DegenerateMatrixError, MatrixMarketError, build_rhs,
                                         jacobi_precondition, read_matrix_market)

MM = os.path.join(ROOT, "tests", "golden", "mm")


def _files():
    g = golden("matio")
    return [(int(k), str(g[f"f{k}_name"])) for k in range(int(g["nfiles"]))]


@pytest.mark.parametrize("k,name", _files())
def test_parse_and_scale_match_reference(k, name):
    g = golden("matio")
    a = read_matrix_market(os.path.join(MM, name))
    np.testing.assert_array_equal(a.row_ptr, g[f"f{k}_row_ptr"])
    np.testing.assert_array_equal(a.col_idx, g[f"f{k}_col_idx"])
    np.testing.assert_array_equal(a.values, g[f"f{k}_values"])
    ah, dinv = jacobi_precondition(a)
    np.testing.assert_array_equal(ah.values, g[f"f{k}_jvalues"])
    np.testing.assert_array_equal(dinv, g[f"f{k}_dinv"])
    d = ah.to_dense()
    assert np.max(np.abs(d - d.T)) == 0.0  # bitwise symmetric


@pytest.mark.parametrize("name,gold", [("nos1", "problem_nos1"), ("494_bus", "problem_494bus")])
def test_acceptance_matrices_match_reference(name, gold):
    """The reference's own acceptance matrices, when its tree is mounted (this
    container); the scaled CSR equals its load_problem output bit for bit."""
    path = f"/root/reference/pkg/data/matrices/{name}.mtx"
    if not os.path.exists(path):
        pytest.skip("reference matrices not mounted")
    ah, _ = jacobi_precondition(read_matrix_market(path))
    g = golden(gold)
    np.testing.assert_array_equal(ah.row_ptr, g["row_ptr"])
    np.testing.assert_array_equal(ah.col_idx, g["col_idx"])
    np.testing.assert_array_equal(ah.values, g["values"])


def test_identity_general_duplicates(tmp_path):
    p = tmp_path / "id.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n1 1 1\n2 2 1\n3 3 1\n")
    a = read_matrix_market(str(p))
    assert (a.n, a.nnz, a.n_a) == (3, 3, 1)
    np.testing.assert_array_equal(a.to_dense(), np.eye(3))
    p = tmp_path / "gen.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n"
                 "2 2 4\n1 1 2.0\n1 2 1.0\n2 1 1.0\n2 2 3.0\n")
    np.testing.assert_array_equal(read_matrix_market(str(p)).to_dense(), [[2.0, 1.0], [1.0, 3.0]])
    p = tmp_path / "dup.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 1.0\n1 1 2.0\n2 2 1.0\n")
    assert read_matrix_market(str(p)).to_dense()[0, 0] == 3.0
    p = tmp_path / "asym.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 2.0\n1 2 1.0\n2 2 3.0\n")
    with pytest.raises(MatrixMarketError):
        read_matrix_market(str(p))


@pytest.mark.parametrize("content,line", [
    ("%%NotMatrixMarket\n2 2 1\n1 1 1.0\n", 1),
    ("%%MatrixMarket matrix coordinate complex symmetric\n2 2 1\n1 1 1.0 0.0\n", 1),
    ("%%MatrixMarket matrix coordinate pattern symmetric\n2 2 1\n1 1\n", 1),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1.0\n", 2),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1.0\nbroken line\n", 4),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1.0\n3 1 1.0\n", 4),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 1.0\n2 2 1.0\n", 4),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 1.0\n", 3),
    ("%%MatrixMarket matrix coordinate real symmetric\n% only comments\n", 2),
])
def test_parse_errors_carry_line_numbers(tmp_path, content, line):
    p = tmp_path / "bad.mtx"
    p.write_text(content)
    with pytest.raises(MatrixMarketError) as exc:
        read_matrix_market(str(p))
    assert exc.value.line_no == line
    assert f"(line {line})" in str(exc.value)


def test_jacobi_known_answers():
    def sparse(m):
        import scipy.sparse as sp
        c = sp.csr_matrix(np.asarray(m, dtype=float))
        return SparseMatrix(n=c.shape[0], row_ptr=c.indptr.astype(np.int64),
                            col_idx=c.indices.astype(np.int32), values=c.data,
                            n_a=int(np.diff(c.indptr).max()))
    ah, dinv = jacobi_precondition(sparse(np.diag([4.0, 9.0, 0.25])))
    np.testing.assert_array_equal(ah.to_dense(), np.eye(3))
    np.testing.assert_allclose(dinv, [0.5, 1 / 3, 2.0])
    ah, _ = jacobi_precondition(sparse([[4.0, 1.0], [1.0, 2.0]]))
    off = 1.0 / (2 * np.sqrt(2))
    np.testing.assert_allclose(ah.to_dense(), [[1.0, off], [off, 1.0]], rtol=1e-15)
    with pytest.raises(DegenerateMatrixError):
        jacobi_precondition(sparse([[-1.0, 0.0], [0.0, 2.0]]))


def test_build_rhs():
    np.testing.assert_array_equal(build_rhs(4), [0.5, 0.5, 0.5, 0.5])
    assert abs(np.linalg.norm(build_rhs(494)) - 1.0) <= 8 * np.finfo(float).eps
    with pytest.raises(ValueError):
        build_rhs(0)
