"""CPU tests: the C oracle (oracle/spmk_oracle.c) pinned against the reference.

Pinning, in order of strength:
  1. against the reference's own outputs, recorded as digests in
     tests/golden/golden.json by tests/golden/make_golden.py (always runs);
  2. against the reference library itself (oracle/_ref/libspmk_ref.so) when
     it was built here (skipped elsewhere);
  3. the reference's known-answer tests restated (proj/tests/*.cpp).
"""
import hashlib
import json
import os

import numpy as np
import pytest

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
PAD = np.iinfo(np.int64).max


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------- golden digests
def test_corpus_matches_reference_digests(corpus):
    assert [a.name for a in corpus] == [g["name"] for g in GOLDEN["corpus"]]
    for a, g in zip(corpus, GOLDEN["corpus"]):
        assert (a.m, a.k, a.nnz, a.max_row_nnz()) == (g["m"], g["k"], g["nnz"], g["max_row"]), a.name
        assert sha(a.row_ptr) == g["row_ptr"] and sha(a.col_idx) == g["col_idx"], a.name
        assert sha(a.val) == g["values"], a.name


def test_features_and_selector_match_reference(orc, corpus):
    for a, g in zip(corpus, GOLDEN["corpus"]):
        f = orc.extract_features(a)
        assert list(f) == g["features"], a.name  # bit-exact doubles
        sel = GOLDEN["select"][a.name]
        for n in range(1, 130):
            assert orc.select_kernel(f[0], f[2], n) == sel[str(n)], (a.name, n)


def test_plan_matches_reference(orc, corpus):
    for a in corpus:
        for ch, g in GOLDEN["plan"][a.name].items():
            er, nch, cf = orc.plan_balanced(a, int(ch))
            assert nch == g["num_chunks"]
            assert sha(er) == g["elem_row"]
            assert sha(cf.astype(np.int64)) == g["chunk_first_row"]


def test_kernels_match_reference_digests(orc, corpus):
    by = {a.name: a for a in corpus}
    xs = {}
    for g in GOLDEN["spmm"]:
        a = by[g["matrix"]]
        key = (a.name, g["n"])
        if key not in xs:
            xs[key] = orc.make_dense(a.k, g["n"], g["x_seed"])
        y = orc.spmm(a, g["kernel"], xs[key], lane_width=g["lane_width"], seq_chunk=g["seq_chunk"])
        assert sha(y) == g["y"], g


def test_rmat_and_dense_streams_match_reference(orc):
    for g in GOLDEN["rmat"]:
        a = orc.generate_rmat(g["scale"], g["edge_factor"], tuple(g["skew"]), g["seed"])
        assert a.nnz == g["nnz"] and sha(a.row_ptr) == g["row_ptr"] and sha(a.col_idx) == g["col_idx"]
    for g in GOLDEN["dense"]:
        assert sha(orc.make_dense(g["rows"], g["cols"], g["seed"])) == g["sha"]


# ---------------------------------------------------------------- live reference
def test_randomized_chunks_against_reference(orc, ref):
    """acceptance.cpp:81-119 style: random lane chunks, C in {1,2,4}, W 2..64."""
    rng = np.random.default_rng(0xACCE)
    for _ in range(2000):
        w = int(rng.choice([2, 4, 8, 16, 32, 64]))
        c = int(rng.choice([1, 2, 4]))
        rows = np.cumsum(rng.random(w) < 0.35) + int(rng.integers(0, 4))
        rows = rows.astype(np.int64)
        npad = int(rng.integers(0, w // 2 + 1))
        if npad:
            rows[w - npad:] = PAD
        vals = (rng.standard_normal(w * c)).astype(np.float32)
        assert np.array_equal(orc.conditional_scan(rows, vals, c).view(np.uint32),
                              ref.conditional_scan(rows, vals, c).view(np.uint32))


def test_kernels_bit_exact_against_reference(orc, ref, corpus):
    for a in corpus[::3]:
        h = ref.handle(a)
        for n in (1, 4, 7, 33):
            x = orc.make_dense(a.k, n, 77 + n)
            for kidx in range(4):
                for W, S in ((32, 256), (8, 3)):
                    yo = orc.spmm(a, kidx, x, lane_width=W, seq_chunk=S)
                    yr = h.spmm(kidx, x, lane_width=W, seq_chunk=S)
                    assert np.array_equal(yo.view(np.uint32), yr.view(np.uint32)), (a.name, n, kidx, W, S)


def test_kernel_stats_against_reference(orc, ref, corpus):
    for a in corpus[::4]:
        h = ref.handle(a)
        for n in (1, 3, 8):
            x = orc.make_dense(a.k, n, 5)
            for kidx in (0, 1):
                for W in (4, 32):
                    assert orc.kernel_stats(a, kidx, n, lane_width=W) == h.kernel_stats(kidx, x, lane_width=W)


def test_partition_and_slices_against_reference(orc, ref, corpus):
    for items in (0, 1, 7, 1000, 16083729):
        for parts in (1, 2, 3, 8):
            for w in range(parts):
                assert orc.partition(items, parts, w) == ref.partition(items, parts, w)
    for a in corpus:
        for parts in (1, 2, 4, 8):
            b = orc.row_slices(a, parts)
            assert b[0] == 0 and b[-1] == a.m and np.all(np.diff(b) >= 0)
            for g in range(1, parts):
                lo, _ = ref.partition(a.nnz, parts, g)
                assert b[g] == np.searchsorted(a.row_ptr, lo, side="left")


def test_fp64_oracle_matches_reference(orc, ref, corpus):
    for a in corpus[::5]:
        h = ref.handle(a)
        x = orc.make_dense(a.k, 5, 9)
        y, bound = orc.oracle_rows(a, x, threads=3)
        assert np.array_equal(y, h.oracle_spmm(x))
        assert np.all(bound >= np.abs(y))


# ---------------------------------------------------------------- reference KATs
def test_reference_kats_core(orc):
    # test_core.cpp:59-93
    a = orc.csr_from_coo(4, 2, [0, 0, 1, 1, 2, 2, 3, 3], [0, 1] * 4, [1] * 8)
    assert orc.extract_features(a) == (2.0, 0.0, 0.0)
    rows = [0] + [1] * 3 + [3] * 4
    cols = [0] + [0, 1, 2] + [0, 1, 2, 3]
    a = orc.csr_from_coo(4, 4, rows, cols, [1.0] * 8)
    f = orc.extract_features(a)
    assert f[0] == 2.0 and f[1] == pytest.approx(1.5811388300841898) and f[2] == pytest.approx(0.7905694150420949)
    a = orc.csr_from_coo(3, 3, [], [], [])
    assert orc.extract_features(a) == (0.0, 0.0, 0.0)
    with pytest.raises(ValueError):
        orc.extract_features(orc.csr_from_coo(0, 3, [], [], []))


def test_reference_kats_scan(orc):
    # test_reduction.cpp:62-76
    assert list(orc.conditional_scan([0, 0, 1, 1], [1, 2, 3, 4])) == [1, 3, 3, 7]
    assert list(orc.conditional_scan([5, 5, 5, 5], [1, 1, 1, 1])) == [1, 2, 3, 4]
    assert list(orc.conditional_scan([0, 1, 2, 3], [9, 8, 7, 6])) == [9, 8, 7, 6]


def test_reference_kats_kernels(orc):
    # test_kernels.cpp:37-69, 101-111, 132-138
    a = orc.csr_from_coo(2, 2, [0, 1, 1], [0, 0, 1], [1, 1, 1])
    er, nch, _ = orc.plan_balanced(a, 2)
    assert list(er) == [0, 1, 1] and nch == 2
    a = orc.csr_from_coo(2, 2, [0, 1, 1], [0, 0, 1], [1.0, 2.0, 3.0])
    x = np.array([[10.0], [20.0]], np.float32)
    for k in range(4):
        assert list(orc.spmm(a, k, x)[:, 0]) == [10.0, 80.0]
    assert list(orc.spmm(a, 3, x, seq_chunk=2)[:, 0]) == [10.0, 80.0]
    a = orc.csr_from_coo(1, 100, [0] * 100, list(range(100)), [1.0] * 100)
    x = np.ones((100, 1), np.float32)
    assert orc.spmm(a, 1, x)[0, 0] == 100.0 and orc.spmm(a, 3, x, seq_chunk=16)[0, 0] == 100.0
    # invalid configs (test_kernels.cpp:239-246)
    assert not orc.check_config(lane_width=3) and not orc.check_config(lane_width=128)
    assert not orc.check_config(vdl_group=3) and not orc.check_config(seq_chunk=0)


def test_reference_kats_selector(orc):
    # test_selector.cpp:28-38
    assert orc.select_kernel(5, 2.0, 1) == 1
    assert orc.select_kernel(100, 0.1, 128) == 2
    assert orc.select_kernel(10, 3.0, 32) == 3
    assert orc.select_kernel(64, 0.5, 2) == 0
    assert orc.select_kernel(32.0, 0.5, 1) == 0  # ties favor row-split
    assert orc.select_kernel(10.0, 1.0, 32) == 2


# ---------------------------------------------------------------- row-subset mode
def test_row_subset_oracle_matches_full_kernels(orc, corpus):
    """so_spmm_rows32 (used at full BASELINE size, where the whole-matrix
    restatement is too slow) reproduces so_spmm row for row: every variant,
    lane widths 2..64, seq_chunk 1..4096, rows in shuffled order."""
    from oracle.oracle import oracle_rows32, spmm_rows

    rng = np.random.default_rng(3)
    for a in corpus[::2]:
        rows = rng.permutation(a.m)[: max(1, a.m // 2)]
        col32 = a.col_idx.astype(np.int32)
        for n in (1, 3, 8):
            x = orc.make_dense(a.k, n, 11 + n)
            for kidx in range(4):
                for W, S in ((32, 256), (2, 1), (64, 7), (8, 4096), (16, 33)):
                    full = orc.spmm(a, kidx, x, lane_width=W, seq_chunk=S)[rows]
                    sub = spmm_rows(orc, a.row_ptr, col32, a.val, kidx, x, rows, lane_width=W, seq_chunk=S,
                                    threads=3)
                    assert np.array_equal(full.view(np.uint32), sub.view(np.uint32)), (a.name, n, kidx, W, S)
        y, b = oracle_rows32(orc, a.row_ptr, col32, a.val, x, rows, threads=2)
        y2, b2 = orc.oracle_rows(a, x, rows=rows, threads=2)
        assert np.array_equal(y, y2) and np.array_equal(b, b2)


def test_row_subset_oracle_against_reference(orc, ref, corpus):
    from oracle.oracle import spmm_rows

    for a in corpus[1::5]:
        h = ref.handle(a)
        rows = np.arange(a.m)[::-3]
        x = orc.make_dense(a.k, 5, 21)
        for kidx in range(4):
            yr = h.spmm(kidx, x, lane_width=16, seq_chunk=100)[rows]
            ys = spmm_rows(orc, a.row_ptr, a.col_idx.astype(np.int32), a.val, kidx, x, rows, lane_width=16,
                           seq_chunk=100)
            assert np.array_equal(yr.view(np.uint32), ys.view(np.uint32)), (a.name, kidx)
