"""Selection harness host logic (paper_2106_16064_b200/selection.py) against
the reference's own KATs: test_bench.cpp:87-191 (selection loss, CSV) and
test_selector.cpp:93-165 (calibrate_thresholds)."""
import random

import pytest

import paper_2106_16064_b200 as spmk
from paper_2106_16064_b200 import selection as sel

K = spmk.kAllKernels


def feats(avg, cv, rows=1000):
    return spmk.MatrixFeatures(avg, avg * cv, cv, rows, int(avg * rows))


def add_cell(records, matrix, n, g, chosen):
    for k in range(4):
        records.append(sel.BenchRecord(matrix, nnz=100, n=n, kernel=spmk.kernel_name(K[k]), gflops=g[k],
                                       time_seconds=2.0 * 100 * n / g[k] / 1e9))
    records.append(sel.BenchRecord(matrix, nnz=100, n=n, kernel=spmk.kernel_name(chosen),
                                   gflops=g[chosen.index], time_seconds=2.0 * 100 * n / g[chosen.index] / 1e9,
                                   selected_by_rule=True))


def test_auto_matching_best_gives_zero_loss():  # test_bench.cpp:87-95
    r = []
    add_cell(r, "m1", 1, [1, 2, 3, 4], spmk.kSeqBalanced)
    add_cell(r, "m1", 8, [5, 2, 3, 4], spmk.kParRowSplit)
    s = sel.summarize_selection_loss(r)
    assert s.per_n_loss[1] == pytest.approx(0.0)
    assert s.per_n_loss[8] == pytest.approx(0.0)
    assert s.single_kernel_loss["seq-ws"] == pytest.approx(0.1)


def test_auto_at_half_best():  # test_bench.cpp:97-103
    r = []
    add_cell(r, "m1", 4, [2, 4, 1, 1], spmk.kParRowSplit)
    add_cell(r, "m2", 4, [3, 6, 1, 1], spmk.kParRowSplit)
    assert sel.summarize_selection_loss(r).per_n_loss[4] == pytest.approx(0.5)


def test_rule_beats_every_fixed_kernel():  # test_bench.cpp:105-122
    r = []
    for m in range(4):
        add_cell(r, f"m{m}", 1, [10, 9, 2, 2], spmk.kParRowSplit)
        add_cell(r, f"m{m}", 4, [9, 10, 2, 2], spmk.kParBalanced)
        add_cell(r, f"m{m}", 32, [2, 2, 10, 9], spmk.kSeqRowSplit)
        add_cell(r, f"m{m}", 128, [2, 2, 9, 10], spmk.kSeqBalanced)
    s = sel.summarize_selection_loss(r)
    auto = sel.mean_per_n_loss(s)
    assert all(auto < l for l in s.single_kernel_loss.values())
    assert sel.min_single_kernel_loss(s) > 0.0


def test_single_kernel_loss_zero_iff_always_best():  # test_bench.cpp:124-131
    r = []
    add_cell(r, "m1", 2, [5, 1, 1, 1], spmk.kParRowSplit)
    add_cell(r, "m1", 16, [5, 1, 1, 1], spmk.kSeqRowSplit)
    s = sel.summarize_selection_loss(r)
    assert s.single_kernel_loss["par-rs"] == 0.0 and s.single_kernel_loss["par-ws"] > 0.0


def test_incomplete_records_raise():  # test_bench.cpp:133-143
    r = []
    add_cell(r, "m1", 1, [1, 2, 3, 4], spmk.kSeqBalanced)
    with pytest.raises(spmk.Error):
        sel.summarize_selection_loss(r[:-1])
    with pytest.raises(spmk.Error):
        sel.summarize_selection_loss(r[1:])


def test_emit_csv_shapes_and_round_trip():  # test_bench.cpp:145-191
    assert sel.emit_csv([], sel.SelectionLossSummary()) == (
        "matrix_name,num_rows,num_cols,nnz,n,kernel,time_seconds,gflops,correct,selected_by_rule\n")
    r = []
    add_cell(r, "m1", 1, [1, 2, 3, 4], spmk.kSeqBalanced)
    text = sel.emit_csv(r, sel.summarize_selection_loss(r))
    lines = text.splitlines()[1:]
    assert sum(1 for l in lines if l.startswith("#")) == 5
    assert sum(1 for l in lines if not l.startswith("#")) == 5
    for rec in sel.read_csv(text):
        assert rec.gflops == pytest.approx(2.0 * rec.nnz * rec.n / rec.time_seconds / 1e9, rel=1e-4)


def cal_cell(records, f, n, g):
    for k in range(4):
        records.append(sel.CalibrationRecord(f, n, K[k], g[k]))


def test_calibration_degenerate_corpus():  # test_selector.cpp:93-104
    r = []
    for i, cv in enumerate((0.3, 0.7, 1.5, 3.0)):
        cal_cell(r, feats(40 + i, cv), 32, [1.0, 1.0, 1.0, 10.0])
    t = sel.calibrate_thresholds(r)
    assert t.t_cv == 0.25 and t.t_parallel_avg == 32.0


def test_calibration_zero_loss_returns_defaults():  # test_selector.cpp:106-116
    r = []
    cal_cell(r, feats(50, 0.2), 32, [1, 1, 10, 2])
    cal_cell(r, feats(50, 2.5), 32, [1, 1, 2, 10])
    cal_cell(r, feats(5, 1.0), 2, [2, 10, 1, 1])
    cal_cell(r, feats(64, 1.0), 2, [10, 2, 1, 1])
    assert sel.calibrate_thresholds(r) == spmk.SelectorThresholds()


def test_calibration_crossover():  # test_selector.cpp:118-129
    r = []
    for i, cv in enumerate((0.4, 0.8, 1.2, 1.4)):
        cal_cell(r, feats(30 + i, cv), 16, [1, 1, 10, 5])
    for i, cv in enumerate((1.6, 1.9, 2.5, 3.5)):
        cal_cell(r, feats(34 + i, cv), 16, [1, 1, 5, 10])
    assert sel.calibrate_thresholds(r).t_cv in (1.0, 2.0)


def test_calibration_never_loses_to_defaults():  # test_selector.cpp:131-158
    rng = random.Random(9)
    r = []
    for cell in range(30):
        g = [0.5 + rng.random() * 9.5 for _ in range(4)]
        cal_cell(r, feats(rng.random() * 200.0, rng.random() * 4.0, 1 + rng.randrange(10000)),
                 1 + rng.randrange(128), g)
    t = sel.calibrate_thresholds(r)

    def loss(th):
        tot = 0.0
        for i in range(0, len(r), 4):
            best = max(x.gflops for x in r[i:i + 4])
            kid = spmk.select_kernel(r[i].features, r[i].n, th)
            tot += 1.0 - r[i + kid.index].gflops / best
        return tot / (len(r) // 4)

    assert loss(t) <= loss(spmk.SelectorThresholds()) + 1e-12


def test_calibration_validation():  # test_selector.cpp:160-165
    with pytest.raises(spmk.Error):
        sel.calibrate_thresholds([])
    with pytest.raises(spmk.Error):
        sel.calibrate_thresholds([sel.CalibrationRecord(feats(10, 1.0), 8, spmk.kSeqRowSplit, 1.0)])


# ---- extension: n_parallel_max in the grid, held-out split
def test_extended_calibration_keeps_defaults_when_they_are_optimal():
    r = []
    cal_cell(r, feats(50, 0.2), 32, [1, 1, 10, 2])
    cal_cell(r, feats(5, 1.0), 2, [2, 10, 1, 1])
    assert sel.calibrate_thresholds_extended(r) == spmk.SelectorThresholds()


def test_extended_calibration_moves_the_parallel_crossover():
    # parallel-reduction variants win up to N = 8 on these cells: the reference
    # grid (n_parallel_max fixed at 4) cannot express that, the extension can
    r = []
    for i, n in enumerate((1, 2, 4, 8)):
        cal_cell(r, feats(5 + i, 0.5), n, [1, 10, 2, 2])
    for i, n in enumerate((16, 32, 64)):
        cal_cell(r, feats(5 + i, 0.5), n, [1, 2, 10, 2])
    base = sel.calibrate_thresholds(r)
    ext = sel.calibrate_thresholds_extended(r)
    assert base.n_parallel_max == 4
    assert ext.n_parallel_max == 8
    assert sel.calibration_loss(r, ext) == 0.0 < sel.calibration_loss(r, base)


def test_holdout_calibration_reports_both_splits():
    train, test = [], []
    for i, n in enumerate((1, 2, 4, 8, 16)):
        cal_cell(train, feats(5 + i, 0.5), n, [1, 10, 2, 2] if n <= 8 else [1, 2, 10, 2])
        cal_cell(test, feats(6 + i, 0.6), n, [1, 10, 2, 2] if n <= 8 else [1, 2, 10, 2])
    h = sel.holdout_calibration(train, test)
    assert h["thresholds"]["n_parallel_max"] == 8
    assert h["test_loss_calibrated"] == 0.0 < h["test_loss_default"]
    assert h["train_loss_calibrated"] <= h["train_loss_default"]
