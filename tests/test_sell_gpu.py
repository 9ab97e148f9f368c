"""GPU tests of the lane-per-job seq-ws path (sell_kernels.cuh: segment-sliced
layout, dynamic work queue, fold pass) against the CPU oracle of
spmm_seq_balanced (kernels.hpp:384-455): bit-exact in the reference's order.

Covers what the corpus-wide parity tests do not single out: path selection,
the fold pass's two tiers (rows of <= 8 / > 8 / > 64 slots), padding lanes
next to inf / NaN in X, empty rows, repeated calls and CUDA-graph replays
(the work-queue counters reset themselves), every sweep shape, and the
multi-tile variant (seq_impl 3).
"""
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


def run(d, x, n_cfg=None, **tune):
    for k, v in tune.items():
        d.set_tuning(k, v)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    y = torch.full((d.num_rows, x.shape[1]), float("nan"), device="cuda")
    d.spmm(spmk.kSeqBalanced, xd, y, cfg=n_cfg)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def same_bits(y, want):
    """Bit equality; NaNs compare by position (payloads may differ)."""
    yn, wn = np.isnan(y), np.isnan(want)
    assert np.array_equal(yn, wn)
    assert np.array_equal(y[~yn].view(np.uint32), want[~wn].view(np.uint32))


def mixed_matrix(rng, m=3000, k=20000, chunk=256):
    """Rows of 0 .. 39 nonzeros, empty rows, and long rows of 9 and 65
    segments (fold pass, CTA tier, one and two staging rounds) and of 7 / 2
    segments (warp tier); columns strictly increasing per row."""
    lens = rng.integers(0, 40, m)
    lens[rng.integers(0, m, 300)] = 0
    lens[5] = 8 * chunk + 3          # 9 segments: fold pass, CTA tier
    lens[17] = 64 * chunk + 10       # > 64 slots: several staging rounds
    lens[33] = 7 * chunk             # <= 8 slots: warp tier
    lens[900] = 2 * chunk - 1
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    ci = np.concatenate([np.sort(rng.choice(k, int(min(L, k)), replace=False)) if L <= k else
                         np.sort(rng.integers(0, k, int(L))) for L in lens]).astype(np.int64)
    va = rng.uniform(-1, 1, int(rp[-1])).astype(np.float32)
    return host(m, k, rp, ci, va)


@pytest.fixture(scope="module")
def mixed():
    a = mixed_matrix(np.random.default_rng(5))
    return a, spmk.DeviceCsr.from_host(a)


def test_path_selection(mixed):
    a, d = mixed
    d.set_tuning("seq_impl", 2)
    assert d.spmm_path(spmk.kSeqBalanced, 32) == "sell"
    assert d.spmm_path(spmk.kSeqBalanced, 64) == "tile"  # N = 8 / 16 / 32 by default (measured)
    assert d.spmm_path(spmk.kSeqBalanced, 16) == "sell"
    assert d.spmm_path(spmk.kSeqBalanced, 8) == "sell"
    assert d.spmm_path(spmk.kSeqBalanced, 4) == "tile"
    assert d.spmm_path(spmk.kSeqBalanced, 33) == "tile"
    assert d.spmm_path(spmk.kSeqBalanced, 32, spmk.KernelConfig(seq_chunk=1000)) == "tile"
    assert d.spmm_path(spmk.kSeqRowSplit, 32) == "sell"
    assert d.spmm_path(spmk.kSeqRowSplit, 8) == "sell"
    assert d.spmm_path(spmk.kSeqRowSplit, 12) == "tile"
    for kid in (spmk.kParRowSplit, spmk.kParBalanced):
        assert d.spmm_path(kid, 32) == "tile"
    d.set_tuning("seq_impl", 3)
    assert d.spmm_path(spmk.kSeqBalanced, 64) == "sell"
    d.set_tuning("seq_impl", 1)
    assert d.spmm_path(spmk.kSeqBalanced, 32) == "tile"
    d.set_tuning("seq_impl", 2)


@pytest.mark.parametrize("n", [8, 16, 32])
@pytest.mark.parametrize("chunk", [1, 7, 256, 512])
def test_bit_exact_mixed_rows(orc, mixed, chunk, n):
    a, d = mixed
    x = orc.make_dense(a.num_cols, n, 77 + chunk)
    cfg = spmk.KernelConfig(seq_chunk=chunk)
    y = run(d, x, cfg, seq_impl=2)
    same_bits(y, orc.spmm(csr_of(a), 3, x, seq_chunk=chunk))
    empty = np.diff(np.asarray(a.row_ptr)) == 0
    assert np.all(y[empty] == 0) and not np.any(np.signbit(y[empty]))


@pytest.mark.parametrize("n", [8, 16, 32])
@pytest.mark.parametrize("shape", [0, 1, 2, 3])
def test_every_sweep_shape(orc, mixed, shape, n):
    a, d = mixed
    x = orc.make_dense(a.num_cols, n, 91)
    y = run(d, x, None, seq_impl=2, sell_cfg=shape)
    d.set_tuning("sell_cfg", 0)
    same_bits(y, orc.spmm(csr_of(a), 3, x))


@pytest.mark.parametrize("n", [64, 96, 128])
def test_multi_tile_variant(orc, mixed, n):
    a, d = mixed
    x = orc.make_dense(a.num_cols, n, 13 + n)
    y = run(d, x, None, seq_impl=3)
    d.set_tuning("seq_impl", 2)
    same_bits(y, orc.spmm(csr_of(a), 3, x))


@pytest.mark.parametrize("n", [8, 16, 32])
def test_padding_lanes_ignore_inf_nan(orc, mixed, n):
    """Padding positions gather X row 0; with inf / NaN there they must add
    nothing (the reference never touches them)."""
    a, d = mixed
    x = orc.make_dense(a.num_cols, n, 5)
    x[0, : n // 4] = np.inf
    x[0, n // 4: n // 2] = -np.inf
    x[0, n // 2:] = np.nan
    x[7, 3] = np.nan
    y = run(d, x, None, seq_impl=2)
    same_bits(y, orc.spmm(csr_of(a), 3, x))


def test_repeated_calls_and_graph_replay(orc, mixed):
    """The work-queue counters reset at the end of every sweep: back-to-back
    calls, a second stream and CUDA-graph replays give the same bits."""
    a, d = mixed
    d.set_tuning("seq_impl", 2)
    x = torch.from_numpy(orc.make_dense(a.num_cols, 32, 3)).cuda()
    want = orc.spmm(csr_of(a), 3, x.cpu().numpy())
    y = torch.empty((a.num_rows, 32), device="cuda")
    for _ in range(5):
        d.spmm(spmk.kSeqBalanced, x, y)
    torch.cuda.synchronize()
    same_bits(y.cpu().numpy(), want)
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        y2 = torch.empty_like(y)
        d.spmm(spmk.kSeqBalanced, x, y2, stream=s2)
    torch.cuda.synchronize()
    same_bits(y2.cpu().numpy(), want)
    g = torch.cuda.CUDAGraph()
    yg = torch.full_like(y, float("nan"))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        d.spmm(spmk.kSeqBalanced, x, yg, stream=s)  # warm-up outside capture (plan built)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            d.spmm(spmk.kSeqBalanced, x, yg, stream=s)
    for _ in range(4):
        yg.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        same_bits(yg.cpu().numpy(), want)


def test_degenerate_matrices(orc):
    cases = [
        host(5, 4, [0, 0, 0, 0, 0, 0], [], []),                          # all rows empty
        host(1, 3, [0, 3], [0, 1, 2], [1.0, -2.0, 3.0]),                 # one row
        host(4, 600, [0, 0, 600, 600, 600], np.arange(600), np.linspace(-1, 1, 600)),  # one long row
        host(33, 40, np.arange(34), np.arange(33) % 40, np.ones(33)),   # 33 one-nonzero rows (2 slices)
    ]
    for a in cases:
        d = spmk.DeviceCsr.from_host(a)
        for chunk in (1, 3, 256):
            for n in (8, 16, 32):
                x = orc.make_dense(a.num_cols, n, chunk)
                y = run(d, x, spmk.KernelConfig(seq_chunk=chunk), seq_impl=2)
                same_bits(y, orc.spmm(csr_of(a), 3, x, seq_chunk=chunk))


@pytest.mark.parametrize("n", [8, 16, 32])
@pytest.mark.parametrize("hub", [-1, 0, 8, 300])
def test_seq_rowsplit_through_the_sweep(orc, mixed, hub, n):
    """seq-rs (kernels.hpp:339-376) at N = 8 / 16 / 32: one job per row, rows
    of >= hub_nnz nonzeros on the hub kernel (-1: default, 0: none)."""
    a, d = mixed
    x = orc.make_dense(a.num_cols, n, 101)
    for k, v in (("seq_impl", 2), ("hub_nnz", hub)):
        d.set_tuning(k, v)
    xd = torch.from_numpy(x).cuda()
    y = torch.full((a.num_rows, n), float("nan"), device="cuda")
    d.spmm(spmk.kSeqRowSplit, xd, y)
    torch.cuda.synchronize()
    d.set_tuning("hub_nnz", -1)
    same_bits(y.cpu().numpy(), orc.spmm(csr_of(a), 2, x))


@pytest.mark.parametrize("n", [8, 32])
def test_fold_reads_this_calls_partials(orc, n):
    """The fold pass starts while the sweep drains (programmatic dependent
    launch) and must read the H slots this call wrote: a fresh handle's first
    call (H uninitialised) and then calls with other X (H holding the previous
    call's partials) are all bit-exact."""
    a = mixed_matrix(np.random.default_rng(11), m=2000)
    d = spmk.DeviceCsr.from_host(a)
    for chunk in (1, 7, 256):
        cfg = spmk.KernelConfig(seq_chunk=chunk)
        for seed in (1, 2, 3):
            x = orc.make_dense(a.num_cols, n, 1000 * chunk + seed)
            y = run(d, x, cfg, seq_impl=2)
            same_bits(y, orc.spmm(csr_of(a), 3, x, seq_chunk=chunk))
