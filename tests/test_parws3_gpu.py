"""GPU tests of par_ws3 (par_ws3.cuh: SpMV par-ws on plans without long rows)
against the CPU oracle of spmm_par_balanced (kernels.hpp:232-330): bit-exact
in the reference's order, with and without empty rows (compact-row lookup or
identity), every tile size, and the par_ws2 fallback when the plan has long
rows."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2106_16064_b200 as spmk  # noqa: E402

pytestmark = pytest.mark.gpu


def host(m, k, rp, ci, va):
    return spmk.CsrMatrix(m, k, np.asarray(rp, np.int64), np.asarray(ci, np.int64), np.asarray(va, np.float32))


def csr_of(a):
    from oracle.oracle import Csr

    return Csr(a.num_rows, a.num_cols, np.asarray(a.row_ptr), np.asarray(a.col_idx), np.asarray(a.values))


def rows_matrix(rng, m, k, lens):
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    ci = np.concatenate([np.sort(rng.choice(k, int(L), replace=False)) for L in lens]).astype(np.int64)
    va = rng.uniform(-1, 1, int(rp[-1])).astype(np.float32)
    return host(m, k, rp, ci, va)


def run(d, x, **tune):
    for kk, v in tune.items():
        d.set_tuning(kk, v)
    y = torch.full((d.num_rows, x.shape[1]), float("nan"), device="cuda")
    d.spmm(spmk.kParBalanced, torch.from_numpy(x).cuda(), y)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def same_bits(y, want):
    yn, wn = np.isnan(y), np.isnan(want)
    assert np.array_equal(yn, wn)
    assert np.array_equal(y[~yn].view(np.uint32), want[~wn].view(np.uint32))


@pytest.mark.parametrize("n", [1, 2, 3, 4])
@pytest.mark.parametrize("empty_rows", [False, True])
@pytest.mark.parametrize("cpt", [0, 4, 8, 64])
def test_bit_exact(orc, empty_rows, cpt, n):
    rng = np.random.default_rng(3 + cpt)
    m, k = 5000, 4000
    lens = rng.integers(1, 60, m)  # rows of 1..59: many cross 32-nonzero chunks
    if empty_rows:
        lens[rng.integers(0, m, 500)] = 0
    a = rows_matrix(rng, m, k, lens)
    d = spmk.DeviceCsr.from_host(a)
    x = orc.make_dense(k, n, 17 + cpt)
    x[5, 0] = -0.0
    want = orc.spmm(csr_of(a), 1, x)
    same_bits(run(d, x, parws3=1, parws_cpt=cpt), want)
    same_bits(run(d, x, parws3=0, parws_cpt=cpt), want)
    if empty_rows:
        e = lens == 0
        y = run(d, x, parws3=1, parws_cpt=cpt)
        assert np.all(y[e] == 0) and not np.any(np.signbit(y[e]))


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_long_rows(orc, n):
    """Rows longer than a tile make the plan carry long rows (per-chunk H
    partials, owner prefixes in T, fix-up): bit-exact through par_ws3's long
    mode and through par_ws2 / the tile kernel."""
    rng = np.random.default_rng(9)
    m, k = 3000, 9000
    lens = rng.integers(0, 40, m)
    lens[7] = 8000
    lens[100] = 700
    lens[101] = 300
    a = rows_matrix(rng, m, k, lens)
    d = spmk.DeviceCsr.from_host(a)
    x = orc.make_dense(k, n, 4)
    want = orc.spmm(csr_of(a), 1, x)
    for cpt in (4, 8, 0):
        same_bits(run(d, x, parws3=1, parws_cpt=cpt), want)  # par_ws2 / tile kernel
        same_bits(run(d, x, parws3=2, parws_cpt=cpt), want)  # par_ws3 with H / T partials


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_inf_nan_in_x(orc, n):
    """Dead lanes gather X row 0 and live runs never read them: inf / NaN in
    X (row 0 too) give the reference's bits."""
    rng = np.random.default_rng(21)
    m, k = 2000, 1500
    a = rows_matrix(rng, m, k, rng.integers(1, 45, m))
    d = spmk.DeviceCsr.from_host(a)
    x = orc.make_dense(k, n, 8)
    x[0, 0] = np.inf
    x[3, 0] = np.nan
    x[4, 0] = -np.inf
    same_bits(run(d, x, parws3=1, parws_cpt=0), orc.spmm(csr_of(a), 1, x))


@pytest.mark.parametrize("n", [2, 3, 4])
def test_unaligned_operands(orc, n):
    """X / Y views 4 bytes off a 16-byte boundary: scalar loads and stores,
    same bits."""
    rng = np.random.default_rng(2)
    m, k = 1500, 1200
    a = rows_matrix(rng, m, k, rng.integers(1, 40, m))
    d = spmk.DeviceCsr.from_host(a)
    x = orc.make_dense(k, n, 31)
    d.set_tuning("parws3", 1)
    d.set_tuning("parws_cpt", 0)
    xb = torch.zeros(k * n + 1, device="cuda")
    xb[1:] = torch.from_numpy(x).cuda().view(-1)
    yb = torch.full((m * n + 1,), float("nan"), device="cuda")
    d.spmm(spmk.kParBalanced, xb[1:].view(k, n), yb[1:].view(m, n))
    torch.cuda.synchronize()
    same_bits(yb[1:].view(m, n).cpu().numpy(), orc.spmm(csr_of(a), 1, x))
