"""GPU parity tests: the sm_100a path through the C ABI vs the CPU oracle and
the reference's golden digests.

Contract (north_star):
  * indices / partition boundaries / variant choices: bit-exact;
  * Y: bit-identical to the reference's fp32 kernel of the same KernelId at
    the same lane_width / seq_chunk (same partials, same summation order), and
    |y - y64| <= 1e-5 * sum_j |a_ij x_jc| against the fp64 oracle (the
    north_star tolerance, written here).
"""
import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2106_16064_b200 as spmk  # noqa: E402
from oracle.oracle import Csr  # noqa: E402

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
TOL = 1e-5  # north_star: |Δ| ≤ 1e-5·Σ|a_ij·x_j|
NS = (1, 2, 3, 4, 5, 8, 16, 32, 64, 128)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def to_host(a: Csr):
    return spmk.CsrMatrix(a.m, a.k, a.row_ptr, a.col_idx, a.val)


@pytest.fixture(scope="module")
def dev_corpus(corpus):
    return [(a, spmk.DeviceCsr.from_host(to_host(a))) for a in corpus]


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


def assert_tol(y, y64, bound, ctx):
    err = np.abs(y.astype(np.float64) - y64)
    ok = err <= TOL * bound
    assert ok.all(), f"{ctx}: max err/bound {np.max(err / np.maximum(bound, 1e-300))}"


# ------------------------------------------------------------------ inputs
def test_device_rmat_bit_identical_to_reference():
    for g in GOLDEN["rmat"]:
        d = spmk.DeviceCsr.generate_rmat(g["scale"], g["edge_factor"], tuple(g["skew"]), g["seed"])
        h = d.download()
        assert d.nnz == g["nnz"]
        assert sha(h.row_ptr) == g["row_ptr"] and sha(h.col_idx) == g["col_idx"]
        assert np.all(h.values == 1.0)


def test_device_make_dense_bit_identical_to_reference():
    for g in GOLDEN["dense"]:
        x = spmk.make_dense_device(g["rows"], g["cols"], g["seed"])
        torch.cuda.synchronize()
        assert sha(x.cpu().numpy()) == g["sha"]


def test_upload_roundtrip(dev_corpus):
    for a, d in dev_corpus:
        h = d.download()
        assert np.array_equal(h.row_ptr, a.row_ptr) and np.array_equal(h.col_idx, a.col_idx)
        assert np.array_equal(h.values.view(np.uint32), a.val.view(np.uint32))
        assert d.max_row_nnz == a.max_row_nnz()


# ------------------------------------------------------------------ selection
def test_features_and_selection_bit_exact(orc, dev_corpus):
    for (a, d), g in zip(dev_corpus, GOLDEN["corpus"]):
        f = d.features()
        want = g["features"]
        assert f.avg_row == want[0], a.name  # bit-exact by construction
        assert f.stdv_row == pytest.approx(want[1], rel=1e-12, abs=1e-300)
        assert f.cv == pytest.approx(want[2], rel=1e-12, abs=1e-300)
        for n in range(1, 130):
            assert d.select(n).index == GOLDEN["select"][a.name][str(n)], (a.name, n)


def test_plan_partition_bit_exact(orc, dev_corpus):
    for a, d in dev_corpus:
        for ch, g in GOLDEN["plan"][a.name].items():
            cf, nch = d.plan(int(ch))
            assert nch == g["num_chunks"] and sha(cf) == g["chunk_first_row"], (a.name, ch)
        assert sha(d.elem_row()) == GOLDEN["plan"][a.name]["1"]["elem_row"]
        for parts in (1, 2, 3, 8):
            assert np.array_equal(d.row_slices(parts), orc.row_slices(a, parts)), (a.name, parts)


# ------------------------------------------------------------------ kernels
def test_kernels_match_reference_digests(orc, dev_corpus):
    by = {a.name: (a, d) for a, d in dev_corpus}
    for g in GOLDEN["spmm"]:
        a, d = by[g["matrix"]]
        x = orc.make_dense(a.k, g["n"], g["x_seed"])
        y = run(d, spmk.KernelId(g["kernel"]), x, lane_width=g["lane_width"], seq_chunk=g["seq_chunk"])
        assert sha(y) == g["y"], g


@pytest.mark.parametrize("kidx", [0, 1, 2, 3])
def test_kernels_bit_exact_full_corpus(orc, dev_corpus, kidx):
    """acceptance.cpp:46-77 (criterion 1), fp32, N in {1..128}: bit-exact vs the
    reference order and within the north_star bound of the fp64 oracle."""
    kid = spmk.KernelId(kidx)
    for a, d in dev_corpus:
        for n in NS:
            x = orc.make_dense(a.k, n, 1000 + n)
            y = run(d, kid, x)
            assert_bits(y, orc.spmm(a, kidx, x), f"{a.name} n={n} {kid.name}")
            y64, bound = orc.oracle_rows(a, x)
            assert_tol(y, y64, bound, f"{a.name} n={n} {kid.name}")
            tol = orc.kernel_tolerance(a.max_row_nnz())  # the reference's own rule
            assert np.all(np.abs(y - y64) <= tol * np.maximum(1.0, np.abs(y64)))


@pytest.mark.parametrize("W", [2, 4, 8, 16, 32, 64])
def test_lane_width_variants(orc, dev_corpus, W):
    for a, d in dev_corpus[::2]:
        for n in (1, 3, 4, 8, 32):
            x = orc.make_dense(a.k, n, 31 * n + W)
            for kidx in (0, 1):  # par-ws at W=64: par_ws64.cuh (two virtual lanes per lane)
                y = run(d, spmk.KernelId(kidx), x, lane_width=W)
                assert_bits(y, orc.spmm(a, kidx, x, lane_width=W), f"{a.name} n={n} k={kidx} W={W}")


@pytest.mark.parametrize("S", [1, 2, 7, 16, 100, 256, 1000, 5000])
def test_seq_chunk_variants(orc, dev_corpus, S):
    for a, d in dev_corpus[::2]:
        for n in (1, 5, 32, 64):
            x = orc.make_dense(a.k, n, 7 * n + S)
            y = run(d, spmk.kSeqBalanced, x, seq_chunk=S)
            assert_bits(y, orc.spmm(a, 3, x, seq_chunk=S), f"{a.name} n={n} S={S}")


def test_reference_kats_on_device():
    """test_kernels.cpp KATs re-instantiated in fp32 through the device path."""
    a = spmk.CsrMatrix(2, 2, [0, 1, 3], [0, 0, 1], [1.0, 2.0, 3.0])
    x = np.array([[10.0], [20.0]], np.float32)
    for kid in spmk.kAllKernels:  # :60-69
        assert list(spmk.spmm(kid, a, x)[:, 0]) == [10.0, 80.0]
    x2 = np.array([[10.0, 1.0], [20.0, 2.0]], np.float32)  # :71-87
    assert spmk.spmm(spmk.kSeqRowSplit, a, x2).tolist() == [[10.0, 1.0], [80.0, 8.0]]
    assert list(spmk.spmm(spmk.kSeqBalanced, a, x, spmk.KernelConfig(seq_chunk=2))[:, 0]) == [10.0, 80.0]
    # identity passes X through (:89-99)
    eye = spmk.CsrMatrix(4, 4, [0, 1, 2, 3, 4], [0, 1, 2, 3], [1.0] * 4)
    xe = np.random.default_rng(17).uniform(-1, 1, (4, 8)).astype(np.float32)
    for kid in spmk.kAllKernels:
        assert np.array_equal(spmk.spmm(kid, eye, xe), xe)
    # single 100-nnz row across chunks (:101-111)
    long_row = spmk.CsrMatrix(1, 100, [0, 100], list(range(100)), [1.0] * 100)
    ones = np.ones((100, 1), np.float32)
    assert spmk.spmm(spmk.kParBalanced, long_row, ones)[0, 0] == 100.0
    assert spmk.spmm(spmk.kSeqBalanced, long_row, ones, spmk.KernelConfig(seq_chunk=16))[0, 0] == 100.0
    # errors (:231-246)
    with pytest.raises(spmk.Error):
        spmk.spmm(spmk.kParRowSplit, a, np.zeros((3, 1), np.float32))
    for bad in (dict(lane_width=3), dict(lane_width=128), dict(vdl_group=3), dict(seq_chunk=0)):
        with pytest.raises(spmk.Error):
            spmk.spmm(spmk.kParRowSplit, a, x, spmk.KernelConfig(**bad))
    with pytest.raises(spmk.UnsupportedError):
        spmk.spmm(spmk.kSeqRowSplit, a, x.astype(np.float64))


def test_empty_and_degenerate_shapes():
    z = spmk.CsrMatrix(64, 64, np.zeros(65, np.int64), [], [])
    x = np.ones((64, 3), np.float32)
    for kid in spmk.kAllKernels:
        assert np.all(spmk.spmm(kid, z, x) == 0)
    a = spmk.CsrMatrix(2, 2, [0, 1, 3], [0, 0, 1], [1.0, 2.0, 3.0])
    for kid in spmk.kAllKernels:
        assert spmk.spmm(kid, a, np.zeros((2, 0), np.float32)).shape == (2, 0)
    # Y fully overwritten, including empty rows (garbage in, zeros out)
    d = spmk.DeviceCsr.from_host(spmk.CsrMatrix(3, 2, [0, 1, 1, 2], [0, 1], [2.0, 3.0]))
    xd = torch.ones((2, 4), device="cuda")
    for kid in spmk.kAllKernels:
        y = torch.full((3, 4), float("nan"), device="cuda")
        d.spmm(kid, xd, y)
        torch.cuda.synchronize()
        assert y.cpu().tolist() == [[2.0] * 4, [0.0] * 4, [3.0] * 4]


def test_invalid_csr_rejected(orc):
    with pytest.raises(spmk.Error):  # column out of range
        spmk.DeviceCsr.from_host(spmk.CsrMatrix(1, 2, [0, 1], [5], [1.0]))
    with pytest.raises(spmk.Error):  # row_ptr not monotone
        spmk.DeviceCsr.from_host(spmk.CsrMatrix(2, 2, [0, 2, 1], [0], [1.0]))
    # Unsorted / duplicate columns: validate() rejects them (csr.hpp:95-119),
    # spmm computes in position order like the reference's spmm_* (which never
    # call validate), so the result equals the reference kernels' on the same arrays.
    rp, ci = [0, 3, 5], [2, 1, 1, 0, 0]
    va = np.array([1.5, -2.0, 0.25, 3.0, -1.0], np.float32)
    d = spmk.DeviceCsr.from_host(spmk.CsrMatrix(2, 4, rp, ci, va))
    with pytest.raises(spmk.Error):
        d.validate()
    a = Csr(2, 4, np.array(rp, np.int64), np.array(ci, np.int64), va, "unsorted")
    for n in (1, 4):
        x = orc.make_dense(4, n, 3 + n)
        for kid in spmk.kAllKernels:
            assert_bits(run(d, kid, x), orc.spmm(a, kid.index, x), f"unsorted {kid.name} n={n}")
    spmk.DeviceCsr.from_host(spmk.CsrMatrix(1, 4, [0, 2], [1, 2], [1.0, 1.0])).validate()


def test_determinism_and_stats(orc, dev_corpus):
    """test_kernels.cpp:207-229 (bit-identical reruns) and :248-272 (counters)."""
    for a, d in dev_corpus[::4]:
        x = orc.make_dense(a.k, 5, 42)
        for kid in spmk.kAllKernels:
            assert np.array_equal(run(d, kid, x), run(d, kid, x))
            for W in (4, 32):
                got = d.kernel_stats(kid, 5, spmk.KernelConfig(lane_width=W))
                assert got == orc.kernel_stats(a, kid.index, 5, lane_width=W)


def test_host_api_matches_device_api(orc, dev_corpus):
    a, d = dev_corpus[20]
    x = orc.make_dense(a.k, 8, 3)
    for kid in spmk.kAllKernels:
        assert np.array_equal(d.spmm_host(kid, x), run(d, kid, x))
        assert np.array_equal(spmk.spmm(kid, to_host(a), x), run(d, kid, x))


def test_row_slices_parity(orc):
    """Multi-GPU contract on one device: each equal-nnz slice, run standalone,
    reproduces its rows of the full product bit-exactly (§8e)."""
    a = orc.generate_rmat(12, 8, (0.57, 0.19, 0.19, 0.05), 5)
    d = spmk.DeviceCsr.from_host(to_host(a))
    x = orc.make_dense(a.k, 4, 11)
    b = d.row_slices(4)
    assert np.array_equal(b, orc.row_slices(a, 4))
    for kid in (spmk.kSeqRowSplit, spmk.kParRowSplit):
        full = run(d, kid, x)
        for g in range(4):
            s = d.slice(int(b[g]), int(b[g + 1]))
            assert np.array_equal(run(s, kid, x), full[b[g]:b[g + 1]])
    for kid in (spmk.kSeqBalanced, spmk.kParBalanced):  # chunking restarts at the slice origin
        for g in range(4):
            s = d.slice(int(b[g]), int(b[g + 1]))
            sh = s.download()
            sa = Csr(sh.num_rows, sh.num_cols, sh.row_ptr, sh.col_idx, sh.values)
            assert_bits(run(s, kid, x), orc.spmm(sa, kid.index, x), f"slice {g} {kid.name}")


@pytest.mark.slow
def test_cfg2_full_size(orc):
    """BASELINE cfg2 at full size: R-MAT s20 e16 heavy seed 1, N=32.
    All four variants bit-exact vs the reference order (the row-split ones
    with their 1,351 hub rows on the hub path; par-rs also at N=1, where the
    hub rows take the two-pass products + streamed-fold path) and within the
    north_star bound on a row sample incl. the hub rows."""
    d = spmk.DeviceCsr.generate_rmat(20, 16, (0.57, 0.19, 0.19, 0.05), 1)
    assert d.nnz == 16083729
    assert d.select(32) == spmk.kSeqBalanced
    h = d.download()
    a = Csr(h.num_rows, h.num_cols, h.row_ptr, h.col_idx, h.values)
    x = spmk.make_dense_device(a.k, 32, 0x00D5EED + 32)
    torch.cuda.synchronize()
    xh = x.cpu().numpy()
    lens = np.diff(a.row_ptr)
    rows = np.unique(np.concatenate([np.argsort(lens)[-64:], np.random.default_rng(1).integers(0, a.m, 4000)]))
    y64, bound = orc.oracle_rows(a, xh, rows=rows)
    for kid in spmk.kAllKernels:
        y = d.spmm(kid, x)
        torch.cuda.synchronize()
        yh = y.cpu().numpy()
        assert_tol(yh[rows], y64, bound, f"cfg2 {kid.name}")
        assert_bits(yh, orc.spmm(a, kid.index, xh), f"cfg2 {kid.name}")
    x1 = spmk.make_dense_device(a.k, 1, 0x00D5EED + 1)
    torch.cuda.synchronize()
    x1h = x1.cpu().numpy()
    for kid in (spmk.kParRowSplit, spmk.kSeqRowSplit):
        y = d.spmm(kid, x1)
        torch.cuda.synchronize()
        assert_bits(y.cpu().numpy(), orc.spmm(a, kid.index, x1h), f"cfg2 N=1 {kid.name}")


@pytest.mark.parametrize("vl", [1, 4, 8])
def test_par_rs_virtual_lanes(orc, dev_corpus, vl):
    """par-rs at lane_width 32 with VL virtual lanes per physical lane (the
    tree levels inside a lane in registers): the same bits for every VL."""
    for a, d in dev_corpus:
        old = d.get_tuning("parrs_vl")
        d.set_tuning("parrs_vl", vl)
        try:
            for n in (1, 2, 3, 4):
                x = orc.make_dense(a.k, n, 97 * n + vl)
                assert_bits(run(d, spmk.kParRowSplit, x), orc.spmm(a, 0, x), f"{a.name} n={n} vl={vl}")
        finally:
            d.set_tuning("parrs_vl", old)
