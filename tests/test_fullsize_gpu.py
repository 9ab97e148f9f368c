"""Full BASELINE-size parity (cfg4, cfg5) and the cfg3 sweep cells against the
reference order.

cfg4 (SpMM N=64, R-MAT 2^24 e32, 520.8M nonzeros, X byte offsets above 2^32)
and cfg5 (SpMV on R-MAT 2^25 e16, 528.7M nonzeros, rows of 400K nonzeros;
generated values and the column-stochastic values PageRank uses) are checked
three ways:
  * against digests the REFERENCE ITSELF produced at these sizes
    (tests/golden/fullsize.json, tests/golden/make_fullsize.py): the CSR, X,
    the rule's choice, the WHOLE Y of the rule's kernel and Y on a row sample
    (every row >= 1024 nonzeros + 4096 random rows) for all four kernels;
  * bit for bit against the C oracle's row-subset mode (so_spmm_rows32: the
    reference's order with the global chunk boundaries) on that sample;
  * within the north-star bound |y - y64| <= 1e-5 * sum_j |a_ij x_j| of the
    fp64 oracle on the sample.
The sweep cells (uniform / banded / heavy x 2^18..2^22) run all four kernels
against the oracle's row-subset mode on a sample as well.
"""
import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200.inputs import SKEWS, banded, rmat  # noqa: E402
from paper_2106_16064_b200.pagerank import column_counts, make_column_stochastic  # noqa: E402
from oracle.oracle import oracle_rows32, spmm_rows  # noqa: E402

pytestmark = pytest.mark.gpu

GOLD_PATH = os.path.join(os.path.dirname(__file__), "golden", "fullsize.json")
GOLD = json.load(open(GOLD_PATH)) if os.path.exists(GOLD_PATH) else {}
DENSE_SEED = 0x00D5EED


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class _DevArray:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def host_arrays(d: spmk.DeviceCsr):
    """(row_ptr int64, col_idx int32, values fp32) of a handle, on the host."""
    rp, ci, va = d.device_arrays()
    row_ptr = torch.as_tensor(_DevArray(rp, d.num_rows + 1, "<i4"), device="cuda").cpu().numpy().astype(np.int64)
    col = torch.as_tensor(_DevArray(ci, d.nnz, "<i4"), device="cuda").cpu().numpy()
    val = torch.as_tensor(_DevArray(va, d.nnz, "<f4"), device="cuda").cpu().numpy()
    return row_ptr, col, val


def sample_rows(row_ptr, m, long_nnz=1024, count=4096, seed=0):
    lens = np.diff(row_ptr)
    rnd = np.random.default_rng(seed).choice(m, size=min(count, m), replace=False)
    return np.unique(np.concatenate([np.flatnonzero(lens >= long_nnz), rnd])).astype(np.int64)


def check_rows(orc, name, kidx, y_rows, rp, ci, va, xh, rows, bound=True):
    want = spmm_rows(orc, rp, ci, va, kidx, xh, rows)
    if not np.array_equal(y_rows.view(np.uint32), want.view(np.uint32)):
        bad = np.argwhere(y_rows.view(np.uint32) != want.view(np.uint32))
        i = tuple(bad[0])
        raise AssertionError(f"{name} kernel {kidx}: {len(bad)} elements differ from the reference order, "
                             f"first at sample {i} (row {rows[i[0]]}): {y_rows[i]!r} vs {want[i]!r}")
    if bound:
        y64, b = oracle_rows32(orc, rp, ci, va, xh, rows)
        assert np.all(np.abs(y_rows.astype(np.float64) - y64) <= 1e-5 * b + 1e-30), f"{name} kernel {kidx}: bound"


def _full_case(orc, name, stochastic_keys):
    g = GOLD.get(name)
    if g is None:
        pytest.skip(f"tests/golden/fullsize.json has no {name} (run tests/golden/make_fullsize.py)")
    d = spmk.DeviceCsr.generate_rmat(g["scale"], g["ef"], tuple(g["skew"]), g["seed"])
    assert (d.num_rows, d.num_cols, d.nnz, d.max_row_nnz) == (g["m"], g["k"], g["nnz"], g["max_row"])
    rp, ci, va = host_arrays(d)
    assert sha(rp) == g["row_ptr"] and sha(ci) == g["col_idx_i32"], "device R-MAT differs from the reference"
    n = g["n"]
    x = spmk.make_dense_device(d.num_cols, n, DENSE_SEED + n)
    xh = x.cpu().numpy()
    assert sha(xh) == g["x"], "device make_dense differs from the reference"
    rows = sample_rows(rp, d.num_rows)
    assert len(rows) == g["sample_rows"] and sha(rows) == g["sample_rows_sha"]
    rows_d = torch.from_numpy(rows).cuda()
    y = torch.empty((d.num_rows, n), dtype=torch.float32, device="cuda")
    for key in stochastic_keys:
        gv = g["values"][key]
        if key == "stochastic":
            make_column_stochastic(d, column_counts(d))
            torch.cuda.synchronize()
            va = host_arrays(d)[2]
        assert sha(va) == gv["values"]
        kid = d.select(n)
        assert kid.index == gv["rule"], f"{name}/{key}: rule picked {kid.name}, reference {gv['rule']}"
        for kidx in [kid.index] + [k for k in range(4) if k != kid.index]:
            d.spmm(spmk.KernelId(kidx), x, y)
            torch.cuda.synchronize()
            if kidx == kid.index:
                assert sha(y.cpu().numpy()) == gv["y_full"], f"{name}/{key}: whole Y differs from the reference"
            ys = y[rows_d].cpu().numpy()
            assert sha(ys) == gv["y_sample"][str(kidx)], f"{name}/{key} kernel {kidx}: sample differs"
            if kidx == kid.index:
                check_rows(orc, f"{name}/{key}", kidx, ys, rp, ci, va, xh, rows)
    return d


@pytest.mark.slow
def test_cfg4_full_size(orc):
    """cfg4: the rule's seq-ws bit-identical to the reference on the whole Y
    (4.3 GB), every kernel on the sample."""
    d = _full_case(orc, "cfg4", ("generated",))
    assert d.select(64) == spmk.kSeqBalanced


@pytest.mark.slow
def test_cfg5_full_size(orc):
    """cfg5: the rule's par-ws (both value sets) bit-identical to the
    reference on the whole Y, every kernel on the sample."""
    _full_case(orc, "cfg5", ("generated", "stochastic"))


SWEEP_N = {18: 1, 19: 4, 20: 32, 21: 128, 22: 8}


@pytest.mark.slow
@pytest.mark.parametrize("family", ["uniform", "banded", "heavy"])
def test_sweep_cells_against_oracle(orc, family):
    """One cell per (family, scale) of the cfg3 sweep: all four kernels
    bit-exact against the reference order (oracle row-subset mode) on every
    row >= 256 nonzeros plus 2048 random rows, and within the fp64 bound."""
    for s, n in SWEEP_N.items():
        d = banded(1 << s, 8) if family == "banded" else rmat(s, 16, family, 1)
        rp, ci, va = host_arrays(d)
        rows = sample_rows(rp, d.num_rows, long_nnz=256, count=2048, seed=s)
        x = spmk.make_dense_device(d.num_cols, n, DENSE_SEED + n)
        xh = x.cpu().numpy()
        rows_d = torch.from_numpy(rows).cuda()
        for kidx in range(4):
            y = d.spmm(spmk.KernelId(kidx), x)
            torch.cuda.synchronize()
            check_rows(orc, f"{family}-s{s} n={n}", kidx, y[rows_d].cpu().numpy(), rp, ci, va, xh, rows,
                       bound=(kidx == 0))
        del d, x
        torch.cuda.empty_cache()
