"""Hub rows of the row-split variants (hub_kernels.cuh): rows with >= L
nonzeros are skipped by the main par-rs / seq-rs kernels and computed by the
hub kernels on the side stream, in the reference's order (kernels.hpp:157-224
per-lane chains + tree; kernels.hpp:339-376 one ordered chain).  Bit-exact
against the oracle for every lane width, column counts that are not multiples
of the 32-column tile, and the tile-splitting edge cases (hub rows first,
last, adjacent, filling a whole row-split tile, next to empty rows).
"""
from contextlib import contextmanager

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200.inputs import SKEWS  # noqa: E402
from oracle.oracle import Csr  # noqa: E402

pytestmark = pytest.mark.gpu


def to_host(a: Csr):
    return spmk.CsrMatrix(a.m, a.k, a.row_ptr, a.col_idx, a.val)


def run(dev, kid, x_np, **cfg):
    xd = torch.from_numpy(np.ascontiguousarray(x_np)).cuda()
    y = dev.spmm(kid, xd, cfg=spmk.KernelConfig(**cfg) if cfg else None)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def assert_bits(y, want, ctx):
    if not np.array_equal(y.view(np.uint32), want.view(np.uint32)):
        bad = np.argwhere(y.view(np.uint32) != want.view(np.uint32))
        i = tuple(bad[0])
        raise AssertionError(f"{ctx}: {len(bad)} elements differ, first {i}: got {y[i]!r} want {want[i]!r}")


def hub_matrix(orc, seed=5):
    """Rows 0, 1 (adjacent), 40..47 (whole seq-rs tiles), 90 and
    the last row are hubs; rows 2, 60 and 91 are empty."""
    rng = np.random.default_rng(seed)
    m, k = 128, 3000
    lens = rng.integers(1, 12, m)
    for r in (0, 1, *range(40, 48), 90, m - 1):
        lens[r] = rng.integers(200, 2500)
    for r in (2, 60, 91):
        lens[r] = 0
    rows, cols = [], []
    for r in range(m):
        c = rng.choice(k, size=lens[r], replace=False)
        rows += [r] * len(c)
        cols += list(c)
    vals = rng.standard_normal(len(rows)).astype(np.float32)
    a = orc.csr_from_coo(m, k, np.array(rows), np.array(cols), vals)
    a.name = "hubs"
    return a


@contextmanager
def knobs(handles, **kv):
    """Per-handle tuning knobs (spmk_csr_set_tuning), restored afterwards."""
    old = [{k: d.get_tuning(k) for k in kv} for d in handles]
    for d in handles:
        for k, v in kv.items():
            d.set_tuning(k, v)
    try:
        yield
    finally:
        for d, o in zip(handles, old):
            for k, v in o.items():
                d.set_tuning(k, v)


@pytest.fixture(scope="module")
def cases(orc, corpus):
    sel = [a for a in corpus if a.max_row_nnz() >= 16][:4] + [hub_matrix(orc)]
    return [(a, spmk.DeviceCsr.from_host(to_host(a))) for a in sel]


@pytest.mark.parametrize("L", [16, 100, 1000])
def test_seq_rs_hub_rows_bit_exact(orc, cases, L):
    with knobs([d for _, d in cases], hub_nnz=L):
        for a, d in cases:
            for n in (1, 3, 32, 33, 64, 100):
                x = orc.make_dense(a.k, n, 17 * n + L)
                assert_bits(run(d, spmk.kSeqRowSplit, x), orc.spmm(a, 2, x), f"{a.name} n={n} L={L}")


@pytest.mark.parametrize("W", [2, 4, 8, 16, 32, 64])
def test_par_rs_hub_rows_bit_exact(orc, cases, W):
    for L in (16, 300):
        with knobs([d for _, d in cases], hub_nnz=L):
            for a, d in cases:
                for n in (1, 5, 32, 40):
                    x = orc.make_dense(a.k, n, 13 * n + W + L)
                    y = run(d, spmk.kParRowSplit, x, lane_width=W)
                    assert_bits(y, orc.spmm(a, 0, x, lane_width=W), f"{a.name} n={n} W={W} L={L}")


def test_hub_rows_seq_rs_tile_sizes(orc, cases):
    """Different row-split tile sizes (rows per tile) cut differently around hubs."""
    a, d = cases[-1]
    x = orc.make_dense(a.k, 8, 3)
    want = orc.spmm(a, 2, x)
    for tile in (16, 64, 256, 4096):
        with knobs([d], hub_nnz=150, seq_tile_nnz=tile):
            assert_bits(run(d, spmk.kSeqRowSplit, x), want, f"tile={tile}")


def test_hub_path_disabled_matches(orc, cases):
    a, d = cases[-1]
    x = orc.make_dense(a.k, 32, 9)
    with knobs([d], hub_nnz=0):
        y0 = run(d, spmk.kSeqRowSplit, x)
    with knobs([d], hub_nnz=64):
        y1 = run(d, spmk.kSeqRowSplit, x)
    assert_bits(y1, y0, "seq-rs hub on/off")
    assert_bits(y1, orc.spmm(a, 2, x), "seq-rs vs oracle")


def test_hub_rows_rmat_heavy(orc):
    """Default threshold on a device R-MAT heavy graph (rows up to ~4K nonzeros)."""
    d = spmk.DeviceCsr.generate_rmat(16, 16, SKEWS["heavy"], 1)
    h = d.download()
    a = Csr(h.num_rows, h.num_cols, np.asarray(h.row_ptr), np.asarray(h.col_idx), np.asarray(h.values), "rmat16")
    assert a.max_row_nnz() >= 1024
    for n in (1, 32):
        x = orc.make_dense(a.k, n, n)
        assert_bits(run(d, spmk.kSeqRowSplit, x), orc.spmm(a, 2, x), f"seq-rs n={n}")
        assert_bits(run(d, spmk.kParRowSplit, x), orc.spmm(a, 0, x), f"par-rs n={n}")


@pytest.mark.parametrize("kidx", [0, 2])
def test_hub_path_full_corpus(orc, corpus, kidx):
    """Every corpus matrix with almost every row on the hub path (L = 16)."""
    for a in corpus:
        d = spmk.DeviceCsr.from_host(to_host(a))
        d.set_tuning("hub_nnz", 16)
        for n in (1, 4, 32):
            x = orc.make_dense(a.k, n, 5 * n + kidx)
            assert_bits(run(d, spmk.KernelId(kidx), x), orc.spmm(a, kidx, x), f"{a.name} n={n} k={kidx}")


@pytest.mark.slow
def test_cfg5_hub_slice_bit_exact(orc):
    """BASELINE cfg5 graph (R-MAT s25 e16 heavy seed 1), slice 0 of the 8-way
    equal-nnz partition: 66M nonzeros, 51.7M of them in the 11,104 rows >= 1024 (max
    373,191), the slice the per-slice rule sends to par-rs at N=1.  The
    two-pass hub path is bit-exact against the reference order."""
    full = spmk.DeviceCsr.generate_rmat(25, 16, SKEWS["heavy"], 1)
    b = full.row_slices(8)
    d = full.slice(int(b[0]), int(b[1]))
    del full
    torch.cuda.empty_cache()
    assert d.select(1) == spmk.kParRowSplit
    h = d.download()
    a = Csr(h.num_rows, h.num_cols, np.asarray(h.row_ptr), np.asarray(h.col_idx), np.asarray(h.values), "cfg5s0")
    assert a.max_row_nnz() == 373191
    x = orc.make_dense(a.k, 1, 0x00D5EED + 1)
    assert_bits(run(d, spmk.kParRowSplit, x), orc.spmm(a, 0, x), "cfg5 slice 0 par-rs")


def test_seq_rs_two_pass_fold(orc, cases):
    """seq-rs through the products + streamed-fold path (one chain per column,
    hub_two_pass=1; off by default because the producer/folder kernel is
    faster for seq-rs) gives the same bits."""
    with knobs([d for _, d in cases], hub_nnz=16, hub_two_pass=1):
        for a, d in cases:
            for n in (1, 3, 32, 100):
                x = orc.make_dense(a.k, n, 11 * n)
                assert_bits(run(d, spmk.kSeqRowSplit, x), orc.spmm(a, 2, x), f"{a.name} n={n}")
