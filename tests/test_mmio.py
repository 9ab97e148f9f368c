"""Matrix Market ingest of the Python API (paper_2106_16064_b200.mmio), the
reference's test_io.cpp cases (the same KATs the C++ drop-in runs in
tests/cpp/test_dropin.cpp), plus csr_from_coo (csr.hpp:123-164)."""
import io

import numpy as np
import pytest

import paper_2106_16064_b200 as spmk


def rd(text):
    return spmk.read_matrix_market(io.StringIO(text))


def test_general_symmetric_pattern_integer():  # test_io.cpp:11-103
    a = rd("%%MatrixMarket matrix coordinate real general\n% a comment\n\n2 2 2\n1 1 1.0\n2 2 4.0\n")
    assert (a.num_rows, a.num_cols) == (2, 2)
    assert a.row_ptr.tolist() == [0, 1, 2] and a.col_idx.tolist() == [0, 1] and a.values.tolist() == [1.0, 4.0]
    s = rd("%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n2 1 5.0\n3 3 1.0\n3 1 2.0\n")
    assert s.nnz() == 5
    assert s.row_ptr.tolist() == [0, 2, 3, 5]
    assert s.col_idx.tolist() == [1, 2, 0, 0, 2] and s.values.tolist() == [5.0, 2.0, 5.0, 2.0, 1.0]
    p = rd("%%MatrixMarket matrix coordinate pattern general\n2 3 2\n1 3\n2 1\n")
    assert p.values.tolist() == [1.0, 1.0] and p.col_idx.tolist() == [2, 0]
    assert rd("%%MatrixMarket matrix coordinate integer general\n1 1 1\n1 1 7\n").values.tolist() == [7.0]


@pytest.mark.parametrize("banner", [
    "%%MatrixMarket matrix coordinate complex general", "%%MatrixMarket matrix coordinate real skew-symmetric",
    "%%MatrixMarket matrix coordinate real hermitian", "%%MatrixMarket matrix array real general",
    "%%MatrixMarket vector coordinate real general", "MatrixMarket matrix coordinate real general"])
def test_rejected_headers(banner):  # test_io.cpp:104-150
    with pytest.raises(spmk.Error):
        rd(banner + "\n1 1 0\n")


def test_located_errors():
    with pytest.raises(spmk.Error, match="line 3.*bounds"):
        rd("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    with pytest.raises(spmk.Error, match="truncated"):
        rd("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n")
    with pytest.raises(spmk.Error, match="line 3.*malformed"):
        rd("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 oops 1.0\n")
    with pytest.raises(spmk.Error, match="line 1.*empty"):
        rd("")
    with pytest.raises(spmk.Error, match="size line"):
        rd("%%MatrixMarket matrix coordinate real general\n2 2\n")


def test_writer_format_and_round_trip(tmp_path):  # test_io.cpp:152-198
    a = spmk.csr_from_coo([0, 1], [0, 1], [1.0, 4.0], 2, 2)
    out = io.StringIO()
    spmk.write_matrix_market(a, out)
    assert out.getvalue() == "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 2 4\n"
    e = io.StringIO()
    spmk.write_matrix_market(spmk.csr_from_coo([], [], [], 3, 3), e)
    assert e.getvalue() == "%%MatrixMarket matrix coordinate real general\n3 3 0\n"
    r, c, v = [], [], []
    for i in range(50):
        for j in range(0, 50, 1 + i % 7):
            r.append(i), c.append(j), v.append(np.float32(1.0) / np.float32(1 + i + j))
    b = spmk.csr_from_coo(r, c, v, 50, 50)
    path = tmp_path / "b.mtx"
    spmk.write_matrix_market(b, path)
    b2 = spmk.read_matrix_market(path)
    assert np.array_equal(b2.row_ptr, b.row_ptr) and np.array_equal(b2.col_idx, b.col_idx)
    assert np.array_equal(b2.values.view(np.uint32), b.values.view(np.uint32))


def test_csr_from_coo_sorts_sums_and_checks():  # csr.hpp:123-164
    a = spmk.csr_from_coo([1, 0, 1, 1], [2, 1, 0, 2], [1.0, 2.0, 3.0, 0.5], 3, 3)
    assert a.row_ptr.tolist() == [0, 1, 3, 3]
    assert a.col_idx.tolist() == [1, 0, 2] and a.values.tolist() == [2.0, 3.0, 1.5]
    with pytest.raises(spmk.Error, match="out of range"):
        spmk.csr_from_coo([3], [0], [1.0], 3, 3)
    with pytest.raises(spmk.Error):
        spmk.csr_from_coo([], [], [], -1, 3)


def test_matches_oracle_csr_from_coo(orc):
    rng = np.random.default_rng(3)
    r = rng.integers(0, 40, 500)
    c = rng.integers(0, 30, 500)
    v = rng.standard_normal(500).astype(np.float32)
    key = r * 30 + c
    _, first = np.unique(key, return_index=True)  # no duplicates: the sum order cannot matter
    r, c, v = r[first], c[first], v[first]
    perm = rng.permutation(r.size)
    a = spmk.csr_from_coo(r[perm], c[perm], v[perm], 40, 30)
    o = orc.csr_from_coo(40, 30, r[perm], c[perm], v[perm])
    assert np.array_equal(a.row_ptr, o.row_ptr) and np.array_equal(a.col_idx, o.col_idx)
    assert np.array_equal(a.values, o.val)
