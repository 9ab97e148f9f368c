"""The selection harness on the device (bench.hpp:103-189 semantics):
5 records per cell, the auto record is the rule's kernel, every variant agrees
within the north-star bound, GFLOP/s follows 2*nnz*n/t, CSV round trip, and
the banded generator's structure."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200 import inputs, selection  # noqa: E402

pytestmark = pytest.mark.gpu


def test_run_benchmark_records_and_loss():
    corpus = [("heavy-s10", inputs.rmat(10, 8, "heavy", 3)), ("banded-s10", inputs.banded(1 << 10, 8))]
    recs = selection.run_benchmark(corpus, [1, 8], repeats=3, warmup=1)
    assert len(recs) == 2 * 2 * 5
    for name, a in corpus:
        f = a.features()
        for n in (1, 8):
            cell = [r for r in recs if r.matrix_name == name and r.n == n]
            assert len(cell) == 5 and sum(r.selected_by_rule for r in cell) == 1
            auto = next(r for r in cell if r.selected_by_rule)
            assert auto.kernel == spmk.kernel_name(spmk.select_kernel(f, n))
    for r in recs:
        assert r.correct, r
        assert r.gflops == pytest.approx(2.0 * r.nnz * r.n / r.time_seconds / 1e9, rel=1e-9)
    s = selection.summarize_selection_loss(recs)
    assert set(s.per_n_loss) == {1, 8} and all(0.0 <= v <= 1.0 for v in s.per_n_loss.values())
    back = selection.read_csv(selection.emit_csv(recs, s))
    assert [(r.matrix_name, r.n, r.kernel, r.selected_by_rule) for r in back] == \
        [(r.matrix_name, r.n, r.kernel, r.selected_by_rule) for r in recs]


def test_banded_structure():
    m, half = 1000, 8
    h = inputs.banded(m, half).download()
    lens = np.diff(h.row_ptr)
    assert lens[0] == half + 1 and lens[m // 2] == 2 * half + 1 and lens[-1] == half + 1
    r = m // 2
    assert list(h.col_idx[h.row_ptr[r]:h.row_ptr[r + 1]]) == list(range(r - half, r + half + 1))
    assert np.all(h.values == 1.0)
