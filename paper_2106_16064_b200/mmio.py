"""Matrix Market ingest for the Python API, the same
contract as the C++ drop-in `include/spmk/io.hpp`, which restates the
reference's proj/include/spmk/io.hpp:75-173:

  * `coordinate` format only, field real | integer | pattern, symmetry
    general | symmetric; comments (`%`) and blank lines skipped;
  * 1-based indices checked against the declared size, pattern entries read
    as 1, symmetric off-diagonal entries mirrored;
  * duplicates summed and rows sorted by `csr_from_coo` (csr.hpp:123-164);
  * every malformed input raises `Error("matrix market, line <n>: ...")`;
  * the writer emits "coordinate real general" in row-major order with
    max_digits10 (9 significant digits for fp32, the C++ stream format), so
    read(write(a)) == a and the text equals the C++ writer's.

Host-side ingest: the result is a `CsrMatrix` ready for `DeviceCsr.from_host`
(real-matrix validation, e.g. SuiteSparse inputs for `tools/sweep.py --mtx`).
"""
from __future__ import annotations

import io
import os
from dataclasses import dataclass
from typing import List, TextIO, Union

import numpy as np

from .spmk import CsrMatrix, Error

__all__ = ["MatrixMarketHeader", "csr_from_coo", "read_matrix_market", "write_matrix_market"]


@dataclass(frozen=True)
class MatrixMarketHeader:
    field: str = "real"         # real | integer | pattern
    symmetry: str = "general"   # general | symmetric


def csr_from_coo(rows, cols, vals, num_rows: int, num_cols: int) -> CsrMatrix:
    """csr.hpp:123-164: canonical CSR from coordinate triples (range-checked,
    sorted by (row, col), duplicates summed).  The sort is stable, so
    duplicates are summed in input order (the reference's std::sort leaves
    that order unspecified; without duplicates both are identical)."""
    if num_rows < 0 or num_cols < 0:
        raise Error("negative dimension")
    r = np.asarray(rows, dtype=np.int64).reshape(-1)
    c = np.asarray(cols, dtype=np.int64).reshape(-1)
    v = np.asarray(vals, dtype=np.float32).reshape(-1)
    if not (r.shape == c.shape == v.shape):
        raise Error("coordinate arrays differ in length")
    bad = (r < 0) | (r >= num_rows) | (c < 0) | (c >= num_cols)
    if bad.any():
        i = int(np.argmax(bad))
        raise Error(f"coordinate out of range: ({r[i]}, {c[i]}, {float(v[i])}) for {num_rows}x{num_cols}")
    order = np.lexsort((c, r))  # stable: by row, then column
    r, c, v = r[order], c[order], v[order]
    if r.size:
        new = np.ones(r.size, dtype=bool)
        new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        starts = np.flatnonzero(new)
        if starts.size != r.size:  # sum runs left to right in fp32, as `sum += value`
            out = v[starts].copy()
            ends = np.append(starts[1:], r.size)
            for k in np.flatnonzero(ends - starts > 1):
                acc = np.float32(v[starts[k]])
                for j in range(starts[k] + 1, ends[k]):
                    acc = np.float32(acc + v[j])
                out[k] = acc
            v = out
        r, c = r[starts], c[starts]
    row_ptr = np.zeros(num_rows + 1, dtype=np.int64)
    np.add.at(row_ptr, r + 1, 1)
    np.cumsum(row_ptr, out=row_ptr)
    return CsrMatrix(num_rows, num_cols, row_ptr, c, v)


class _Lines:
    def __init__(self, f: TextIO):
        self.f, self.n, self.text = f, 0, ""

    def next(self):
        t = self.f.readline()
        if t == "":
            return None
        self.n += 1
        self.text = t.rstrip("\n")
        return self.text.split()

    def fail(self, msg: str, at: int = 0):
        raise Error(f"matrix market, line {at or self.n}: {msg}")


def _read_banner(ln: _Lines) -> MatrixMarketHeader:
    w = ln.next()
    if w is None:
        ln.fail("empty input", 1)
    if len(w) != 5 or w[0].lower() != "%%matrixmarket":
        ln.fail("malformed banner, expected '%%MatrixMarket matrix coordinate <field> <symmetry>'")
    if w[1].lower() != "matrix":
        ln.fail(f"unsupported object '{w[1]}'")
    if w[2].lower() != "coordinate":
        ln.fail(f"unsupported format '{w[2]}' (only coordinate)")
    field, sym = w[3].lower(), w[4].lower()
    if field not in ("real", "integer", "pattern"):
        ln.fail(f"unsupported field '{w[3]}'")
    if sym not in ("general", "symmetric"):
        ln.fail(f"unsupported symmetry '{w[4]}'")
    return MatrixMarketHeader(field, sym)


def _parse_int(s: str):
    try:
        return int(s)
    except ValueError:
        return None


def read_matrix_market(src: Union[str, os.PathLike, TextIO]) -> CsrMatrix:
    """io.hpp:75-160: read a coordinate Matrix Market file (path or text stream)."""
    if isinstance(src, (str, os.PathLike)):
        try:
            f = open(src, "r")
        except OSError:
            raise Error(f"cannot open {os.fspath(src)}") from None
        with f:
            return read_matrix_market(f)
    ln = _Lines(src)
    h = _read_banner(ln)
    while True:  # size line after comments / blank lines
        w = ln.next()
        if w is None:
            ln.fail("missing size line", ln.n + 1)
        if not w or w[0].startswith("%"):
            continue
        vals = [_parse_int(x) for x in w] if len(w) == 3 else [None]
        if len(w) != 3 or any(x is None for x in vals):
            ln.fail("size line must be 'rows cols nnz'")
        rows, cols, declared = vals
        if rows < 0 or cols < 0 or declared < 0:
            ln.fail("negative size field")
        break
    fields = 2 if h.field == "pattern" else 3
    ri: List[int] = []
    ci: List[int] = []
    vi: List[float] = []
    got = 0
    while got < declared:
        w = ln.next()
        if w is None:
            ln.fail(f"truncated entry list: got {got} of {declared}", ln.n + 1)
        if not w:
            continue
        if len(w) != fields:
            ln.fail(f"entry must have {fields} fields")
        i, j = _parse_int(w[0]), _parse_int(w[1])
        v = 1.0
        ok = i is not None and j is not None
        if ok and h.field != "pattern":
            try:
                v = float(w[2])
            except ValueError:
                ok = False
        if not ok:
            ln.fail(f"malformed entry '{ln.text}'")
        if i < 1 or i > rows or j < 1 or j > cols:
            ln.fail(f"index ({i}, {j}) outside declared bounds")
        ri.append(i - 1)
        ci.append(j - 1)
        vi.append(v)
        if h.symmetry == "symmetric" and i != j:
            ri.append(j - 1)
            ci.append(i - 1)
            vi.append(v)
        got += 1
    return csr_from_coo(ri, ci, np.asarray(vi, dtype=np.float64).astype(np.float32), rows, cols)


def write_matrix_market(a: CsrMatrix, dst: Union[str, os.PathLike, TextIO]) -> None:
    """io.hpp:162-173: "coordinate real general", row-major, round-trip digits."""
    if isinstance(dst, (str, os.PathLike)):
        try:
            f = open(dst, "w")
        except OSError:
            raise Error(f"cannot open {os.fspath(dst)} for writing") from None
        with f:
            return write_matrix_market(a, f)
    out = io.StringIO()
    out.write("%%MatrixMarket matrix coordinate real general\n")
    out.write(f"{a.num_rows} {a.num_cols} {a.nnz()}\n")
    rp, ci, va = a.row_ptr, a.col_idx, a.values
    for r in range(a.num_rows):
        for e in range(int(rp[r]), int(rp[r + 1])):
            out.write(f"{r + 1} {int(ci[e]) + 1} {format(float(va[e]), '.9g')}\n")  # max_digits10
    dst.write(out.getvalue())
