"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front end for the two CPU checkers.

* ``Oracle``   — the plain-C restatement (oracle/spmk_oracle.c), always built.
* ``RefLib``   — the UNMODIFIED reference headers behind oracle/ref_shim.cpp
                 (oracle/_ref/libspmk_ref.so), present wherever build() ran with
                 /root/reference mounted (the .so then travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
ORACLE_SO = os.path.join(REF_DIR, "libspmk_oracle.so")
REF_SO = os.path.join(REF_DIR, "libspmk_ref.so")

i64, u64, f64, f32, i32 = C.c_int64, C.c_uint64, C.c_double, C.c_float, C.c_int32
P = C.POINTER

KERNEL_NAMES = ("par-rs", "par-ws", "seq-rs", "seq-ws")  # kernels.hpp:40-50


def _ptr(a, ct):
    return a.ctypes.data_as(P(ct))


@dataclass
class Csr:
    """Host CSR in the reference layout (csr.hpp:24-57): int64 indices, fp32."""

    m: int
    k: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    val: np.ndarray
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def max_row_nnz(self) -> int:
        return int(np.diff(self.row_ptr).max()) if self.m else 0


class _SoCsr(C.Structure):
    _fields_ = [("m", i64), ("k", i64), ("nnz", i64), ("row_ptr", P(i64)),
                ("col_idx", P(i64)), ("val", P(f32))]


def _so_to_csr(s: _SoCsr, name="") -> Csr:
    m, nnz = s.m, s.nnz
    rp = np.ctypeslib.as_array(s.row_ptr, shape=(m + 1,)).copy()
    ci = np.ctypeslib.as_array(s.col_idx, shape=(max(nnz, 1),))[:nnz].copy()
    va = np.ctypeslib.as_array(s.val, shape=(max(nnz, 1),))[:nnz].copy()
    return Csr(m, s.k, rp, ci, va, name)


class Oracle:
    """The C restatement.  Method names/arguments follow the reference."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle oracle`")
        L = self.lib = C.CDLL(path)
        L.so_csr_free.argtypes = [P(_SoCsr)]
        L.so_csr_from_coo.argtypes = [i64, i64, i64, P(i64), P(i64), P(f32), P(_SoCsr)]
        L.so_generate_rmat.argtypes = [C.c_uint32, u64, f64, f64, f64, f64, u64, P(_SoCsr)]
        L.so_full_corpus.argtypes = [u64, P(_SoCsr), C.c_void_p]
        L.so_make_dense.argtypes = [i64, i64, u64, P(f32)]
        L.so_extract_features.argtypes = [P(i64), i64, P(f64)]
        L.so_select_kernel.argtypes = [f64, f64, u64, u64, f64, f64]
        L.so_plan_balanced.argtypes = [P(i64), i64, i64, i64, P(i64), P(i64)]
        L.so_plan_balanced.restype = i64
        L.so_partition.argtypes = [i64, i64, i64, P(i64), P(i64)]
        L.so_row_slices.argtypes = [P(i64), i64, i64, i64, P(i64)]
        L.so_conditional_scan.argtypes = [i64, i64, P(i64), P(f32)]
        L.so_check_config.argtypes = [i64, i64, i64]
        L.so_spmm.argtypes = [P(_SoCsr), C.c_int, i64, i64, i64, P(f32), i64, P(f32)]
        L.so_kernel_stats.argtypes = [P(_SoCsr), C.c_int, i64, i64, i64, P(u64), P(u64)]
        L.so_kernel_tolerance.argtypes = [i64]
        L.so_kernel_tolerance.restype = f64
        L.so_oracle_rows.argtypes = [P(_SoCsr), P(f32), i64, P(i64), i64, P(f64), P(f64), C.c_int]
        L.so_spmm_rows32.argtypes = [P(i64), P(i32), P(f32), C.c_int, i64, i64, P(f32), i64, P(i64), i64,
                                     P(f32), C.c_int]
        L.so_oracle_rows32.argtypes = [P(i64), P(i32), P(f32), P(f32), i64, P(i64), i64, P(f64), P(f64),
                                       C.c_int]

    # -- helpers
    @staticmethod
    def _view(a: Csr):
        rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(a.col_idx, dtype=np.int64)
        va = np.ascontiguousarray(a.val, dtype=np.float32)
        s = _SoCsr(a.m, a.k, a.nnz, _ptr(rp, i64), _ptr(ci, i64), _ptr(va, f32))
        return s, (rp, ci, va)

    def _take(self, s: _SoCsr, name="") -> Csr:
        out = _so_to_csr(s, name)
        self.lib.so_csr_free(C.byref(s))
        return out

    # -- inputs (rmat.hpp / corpus.hpp / csr.hpp)
    def csr_from_coo(self, m, k, rows, cols, vals) -> Csr:
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float32)
        s = _SoCsr()
        if self.lib.so_csr_from_coo(m, k, len(rows), _ptr(rows, i64), _ptr(cols, i64),
                                    _ptr(vals, f32), C.byref(s)) != 0:
            raise ValueError("coordinate out of range")
        return self._take(s)

    def generate_rmat(self, scale, edge_factor, skew=(0.57, 0.19, 0.19, 0.05), seed=1) -> Csr:
        s = _SoCsr()
        if self.lib.so_generate_rmat(scale, edge_factor, *skew, seed, C.byref(s)) != 0:
            raise ValueError("bad rmat params")
        return self._take(s)

    def full_corpus(self, seed=42):
        arr = (_SoCsr * 32)()
        names = C.create_string_buffer(64 * 32)
        n = self.lib.so_full_corpus(seed, arr, names)
        out = []
        for i in range(n):
            nm = names.raw[64 * i: 64 * (i + 1)].split(b"\0")[0].decode()
            out.append(self._take(arr[i], nm))
        return out

    def make_dense(self, rows, cols, seed) -> np.ndarray:
        out = np.empty((rows, cols), np.float32)
        self.lib.so_make_dense(rows, cols, seed, _ptr(out, f32))
        return out

    # -- hot path
    def extract_features(self, a: Csr):
        out = np.zeros(3, np.float64)
        rp = np.ascontiguousarray(a.row_ptr, np.int64)
        if self.lib.so_extract_features(_ptr(rp, i64), a.m, _ptr(out, f64)) != 0:
            raise ValueError("extract_features requires num_rows >= 1")
        return tuple(float(v) for v in out)

    def select_kernel(self, avg_row, cv, n, n_parallel_max=4, t_parallel_avg=32.0, t_cv=1.0) -> int:
        return self.lib.so_select_kernel(avg_row, cv, n, n_parallel_max, t_parallel_avg, t_cv)

    def plan_balanced(self, a: Csr, chunk):
        rp = np.ascontiguousarray(a.row_ptr, np.int64)
        er = np.empty(max(a.nnz, 1), np.int64)
        nch = (a.nnz + chunk - 1) // chunk if chunk >= 1 else 0
        cf = np.empty(max(nch, 1), np.int64)
        r = self.lib.so_plan_balanced(_ptr(rp, i64), a.m, a.nnz, chunk, _ptr(er, i64), _ptr(cf, i64))
        if r < 0:
            raise ValueError("chunk_size must be >= 1")
        return er[: a.nnz], int(r), cf[:r]

    def partition(self, items, parts, w):
        lo, hi = i64(), i64()
        self.lib.so_partition(items, parts, w, C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def row_slices(self, a: Csr, parts):
        rp = np.ascontiguousarray(a.row_ptr, np.int64)
        b = np.empty(parts + 1, np.int64)
        self.lib.so_row_slices(_ptr(rp, i64), a.m, a.nnz, parts, _ptr(b, i64))
        return b

    def conditional_scan(self, rows, vals, comps=1):
        rows = np.ascontiguousarray(rows, np.int64)
        vals = np.ascontiguousarray(vals, np.float32).copy()
        self.lib.so_conditional_scan(len(rows), comps, _ptr(rows, i64), _ptr(vals, f32))
        return vals

    def check_config(self, lane_width=32, vdl_group=0, seq_chunk=256) -> bool:
        return self.lib.so_check_config(lane_width, vdl_group, seq_chunk) == 0

    def spmm(self, a: Csr, kernel: int, x: np.ndarray, lane_width=32, vdl_group=0, seq_chunk=256):
        x = np.ascontiguousarray(x, np.float32)
        n = x.shape[1]
        y = np.empty((a.m, n), np.float32)
        s, keep = self._view(a)
        if self.lib.so_spmm(C.byref(s), kernel, lane_width, vdl_group, seq_chunk,
                            _ptr(x, f32), n, _ptr(y, f32)) != 0:
            raise ValueError("invalid kernel config")
        return y

    def kernel_stats(self, a: Csr, kernel, n, lane_width=32, vdl_group=0):
        s, keep = self._view(a)
        m, sc = u64(), u64()
        self.lib.so_kernel_stats(C.byref(s), kernel, lane_width, vdl_group, n, C.byref(m), C.byref(sc))
        return m.value, sc.value

    def kernel_tolerance(self, max_row_nnz):
        return self.lib.so_kernel_tolerance(max_row_nnz)

    def oracle_rows(self, a: Csr, x: np.ndarray, rows=None, threads=None):
        """fp64 ground truth (csr.hpp:185-205) + Σ|a·x| bound, optionally on a row sample."""
        x = np.ascontiguousarray(x, np.float32)
        n = x.shape[1]
        s, keep = self._view(a)
        if rows is None:
            cnt, rp = a.m, None
        else:
            rows = np.ascontiguousarray(rows, np.int64)
            cnt, rp = len(rows), _ptr(rows, i64)
        y = np.empty((cnt, n), np.float64)
        b = np.empty((cnt, n), np.float64)
        self.lib.so_oracle_rows(C.byref(s), _ptr(x, f32), n, rp, cnt, _ptr(y, f64), _ptr(b, f64),
                                threads or os.cpu_count() or 1)
        return y, b


class RefLib:
    """The reference itself (unmodified headers), via oracle/ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_generate_rmat.argtypes = [C.c_uint32, u64, f64, f64, f64, f64, u64]
        L.ref_generate_rmat.restype = vp
        L.ref_csr_from_coo.argtypes = [i64, i64, i64, P(i64), P(i64), P(f32)]
        L.ref_csr_from_coo.restype = vp
        L.ref_csr_from_arrays.argtypes = [i64, i64, i64, P(i64), P(i64), P(f32), C.c_int]
        L.ref_csr_from_arrays.restype = vp
        L.ref_csr_from_arrays32.argtypes = [i64, i64, i64, P(i32), P(i32), P(f32)]
        L.ref_csr_from_arrays32.restype = vp
        for fn in ("ref_csr_rows", "ref_csr_cols", "ref_csr_nnz", "ref_csr_max_row"):
            getattr(L, fn).argtypes = [vp]
            getattr(L, fn).restype = i64
        L.ref_csr_free.argtypes = [vp]
        L.ref_csr_name.argtypes = [vp]
        L.ref_csr_name.restype = C.c_char_p
        L.ref_csr_copy.argtypes = [vp, P(i64), P(i64), P(f32)]
        L.ref_full_corpus.argtypes = [u64]
        L.ref_full_corpus.restype = i64
        L.ref_corpus_get.argtypes = [i64]
        L.ref_corpus_get.restype = vp
        L.ref_make_dense.argtypes = [i64, i64, u64, P(f32)]
        L.ref_spmm.argtypes = [vp, C.c_int, i64, i64, i64, i64, P(f32), i64, P(f32)]
        L.ref_time_spmm.argtypes = [vp, C.c_int, P(f32), i64, i64, i64, i64]
        L.ref_time_spmm.restype = f64
        L.ref_oracle_spmm.argtypes = [vp, P(f32), i64, P(f64)]
        L.ref_extract_features.argtypes = [vp, P(f64)]
        L.ref_select_kernel.argtypes = [f64, f64, f64, i64, i64, u64, u64, f64, f64]
        L.ref_plan_balanced.argtypes = [vp, i64, P(i64)]
        L.ref_plan_balanced.restype = i64
        L.ref_partition.argtypes = [i64, i64, i64, P(i64), P(i64)]
        L.ref_conditional_scan.argtypes = [i64, i64, P(i64), P(f32)]
        L.ref_kernel_stats.argtypes = [vp, C.c_int, i64, i64, P(f32), i64, P(u64), P(u64)]
        L.ref_kernel_tolerance.argtypes = [i64]
        L.ref_kernel_tolerance.restype = f64
        L.ref_hardware_concurrency.restype = i64

    def err(self):
        return self.lib.ref_last_error().decode()

    # handles <-> Csr
    def to_csr(self, h, name=None) -> Csr:
        L = self.lib
        m, k, nnz = L.ref_csr_rows(h), L.ref_csr_cols(h), L.ref_csr_nnz(h)
        rp = np.empty(m + 1, np.int64)
        ci = np.empty(max(nnz, 1), np.int64)
        va = np.empty(max(nnz, 1), np.float32)
        L.ref_csr_copy(h, _ptr(rp, i64), _ptr(ci, i64), _ptr(va, f32))
        nm = name if name is not None else L.ref_csr_name(h).decode()
        return Csr(m, k, rp, ci[:nnz], va[:nnz], nm)

    def handle(self, a: Csr, validate=False):
        rp = np.ascontiguousarray(a.row_ptr, np.int64)
        ci = np.ascontiguousarray(a.col_idx, np.int64)
        va = np.ascontiguousarray(a.val, np.float32)
        h = self.lib.ref_csr_from_arrays(a.m, a.k, a.nnz, _ptr(rp, i64), _ptr(ci, i64), _ptr(va, f32),
                                         int(validate))
        if not h:
            raise ValueError(self.err())
        return _RefHandle(self, h)

    def handle32(self, m, k, row_ptr32, col32, val):
        rp = np.ascontiguousarray(row_ptr32, np.int32)
        ci = np.ascontiguousarray(col32, np.int32)
        va = np.ascontiguousarray(val, np.float32)
        h = self.lib.ref_csr_from_arrays32(m, k, len(ci), _ptr(rp, i32), _ptr(ci, i32), _ptr(va, f32))
        return _RefHandle(self, h)

    def generate_rmat(self, scale, edge_factor, skew=(0.57, 0.19, 0.19, 0.05), seed=1) -> Csr:
        h = self.lib.ref_generate_rmat(scale, edge_factor, *skew, seed)
        if not h:
            raise ValueError(self.err())
        out = self.to_csr(h, "")
        self.lib.ref_csr_free(h)
        return out

    def csr_from_coo(self, m, k, rows, cols, vals) -> Csr:
        rows = np.ascontiguousarray(rows, np.int64)
        cols = np.ascontiguousarray(cols, np.int64)
        vals = np.ascontiguousarray(vals, np.float32)
        h = self.lib.ref_csr_from_coo(m, k, len(rows), _ptr(rows, i64), _ptr(cols, i64), _ptr(vals, f32))
        if not h:
            raise ValueError(self.err())
        out = self.to_csr(h, "")
        self.lib.ref_csr_free(h)
        return out

    def full_corpus(self, seed=42):
        n = self.lib.ref_full_corpus(seed)
        return [self.to_csr(self.lib.ref_corpus_get(i)) for i in range(n)]

    def make_dense(self, rows, cols, seed):
        out = np.empty((rows, cols), np.float32)
        self.lib.ref_make_dense(rows, cols, seed, _ptr(out, f32))
        return out

    def select_kernel(self, avg_row, cv, n, n_parallel_max=4, t_parallel_avg=32.0, t_cv=1.0, stdv=0.0,
                      num_rows=1, nnz=0):
        return self.lib.ref_select_kernel(avg_row, stdv, cv, num_rows, nnz, n, n_parallel_max,
                                          t_parallel_avg, t_cv)

    def partition(self, items, parts, w):
        lo, hi = i64(), i64()
        self.lib.ref_partition(items, parts, w, C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def conditional_scan(self, rows, vals, comps=1):
        rows = np.ascontiguousarray(rows, np.int64)
        vals = np.ascontiguousarray(vals, np.float32).copy()
        if self.lib.ref_conditional_scan(len(rows), comps, _ptr(rows, i64), _ptr(vals, f32)) != 0:
            raise ValueError(self.err())
        return vals

    def kernel_tolerance(self, max_row_nnz):
        return self.lib.ref_kernel_tolerance(max_row_nnz)

    def hardware_concurrency(self):
        return self.lib.ref_hardware_concurrency()


class _RefHandle:
    def __init__(self, ref: RefLib, h):
        self.ref, self.h, self.L = ref, h, ref.lib

    def __del__(self):
        try:
            self.L.ref_csr_free(self.h)
        except Exception:
            pass

    @property
    def m(self):
        return self.L.ref_csr_rows(self.h)

    def spmm(self, kernel, x, lane_width=32, vdl_group=0, seq_chunk=256, worker_count=0):
        x = np.ascontiguousarray(x, np.float32)
        n = x.shape[1]
        y = np.empty((self.m, n), np.float32)
        if self.L.ref_spmm(self.h, kernel, lane_width, vdl_group, seq_chunk, worker_count,
                           _ptr(x, f32), n, _ptr(y, f32)) != 0:
            raise ValueError(self.ref.err())
        return y

    def time_spmm(self, kernel, x, repeats=7, warmup=2, worker_count=0):
        x = np.ascontiguousarray(x, np.float32)
        return self.L.ref_time_spmm(self.h, kernel, _ptr(x, f32), x.shape[1], repeats, warmup, worker_count)

    def oracle_spmm(self, x):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty((self.m, x.shape[1]), np.float64)
        if self.L.ref_oracle_spmm(self.h, _ptr(x, f32), x.shape[1], _ptr(y, f64)) != 0:
            raise ValueError(self.ref.err())
        return y

    def extract_features(self):
        out = np.zeros(3, np.float64)
        if self.L.ref_extract_features(self.h, _ptr(out, f64)) != 0:
            raise ValueError(self.ref.err())
        return tuple(float(v) for v in out)

    def plan_balanced(self, chunk):
        nnz = self.L.ref_csr_nnz(self.h)
        er = np.empty(max(nnz, 1), np.int64)
        r = self.L.ref_plan_balanced(self.h, chunk, _ptr(er, i64))
        if r < 0:
            raise ValueError(self.ref.err())
        return er[:nnz], int(r)

    def kernel_stats(self, kernel, x, lane_width=32, vdl_group=0):
        x = np.ascontiguousarray(x, np.float32)
        m, s = u64(), u64()
        if self.L.ref_kernel_stats(self.h, kernel, lane_width, vdl_group, _ptr(x, f32), x.shape[1],
                                   C.byref(m), C.byref(s)) != 0:
            raise ValueError(self.ref.err())
        return m.value, s.value


def load_oracle():
    return Oracle()


def load_ref():
    """The reference library, or None when it was not built (no /root/reference)."""
    try:
        return RefLib()
    except (FileNotFoundError, OSError):
        return None


# ----------------------------------------------------------------- iterative SpMV
def pagerank_step64(orc: Oracle, a: Csr, x: np.ndarray, counts: np.ndarray, alpha: float):
    """One PageRank step in fp64 on the column-stochastic A (a.val already
    1/outdeg(col)): x' = alpha*A x + (1-alpha)/M + alpha*dangling(x)/M.
    No reference counterpart (the reference has no iterative driver); this is
    the checker for paper_2106_16064_b200/pagerank.py.  Returns (x'64, bound)
    with bound = alpha * sum_j |a_ij x_j| per row."""
    m = a.m
    y64, b = orc.oracle_rows(a, x.reshape(m, 1).astype(np.float32))
    dang = float(np.sum(x.reshape(-1).astype(np.float64)[counts == 0]))
    base = (1.0 - alpha) / m + alpha * dang / m
    return alpha * y64[:, 0] + base, alpha * b[:, 0]


def pagerank64(orc: Oracle, a: Csr, counts: np.ndarray, alpha: float, iters: int):
    """fp64 power iteration from x0 = 1/M (free-running reference)."""
    m = a.m
    x = np.full(m, 1.0 / m)
    rows = np.repeat(np.arange(m), np.diff(a.row_ptr))
    vals = a.val.astype(np.float64)
    for _ in range(iters):
        y = np.bincount(rows, weights=vals * x[a.col_idx], minlength=m)
        dang = x[counts == 0].sum()
        x = alpha * y + (1.0 - alpha) / m + alpha * dang / m
    return x


def _threads(threads):
    return threads or min(64, os.cpu_count() or 1)


def spmm_rows(orc: "Oracle", row_ptr, col_idx32, val, kernel: int, x: np.ndarray, rows,
              lane_width=32, seq_chunk=256, threads=None) -> np.ndarray:
    """The reference's fp32 kernel `kernel` evaluated for the listed rows only
    (so_spmm_rows32: same order and global chunk boundaries as the full
    kernel).  col_idx32 is the int32 device layout; returns (len(rows), n)."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx32, np.int32)
    va = np.ascontiguousarray(val, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    rows = np.ascontiguousarray(rows, np.int64)
    n = x.shape[1]
    y = np.empty((len(rows), n), np.float32)
    if orc.lib.so_spmm_rows32(_ptr(rp, i64), _ptr(ci, i32), _ptr(va, f32), kernel, lane_width, seq_chunk,
                              _ptr(x, f32), n, _ptr(rows, i64), len(rows), _ptr(y, f32),
                              _threads(threads)) != 0:
        raise ValueError("invalid kernel config")
    return y


def oracle_rows32(orc: "Oracle", row_ptr, col_idx32, val, x: np.ndarray, rows, threads=None):
    """fp64 ground truth and Σ|a·x| bound (csr.hpp:185-205) for listed rows, int32 columns."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx32, np.int32)
    va = np.ascontiguousarray(val, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    rows = np.ascontiguousarray(rows, np.int64)
    n = x.shape[1]
    y = np.empty((len(rows), n), np.float64)
    b = np.empty((len(rows), n), np.float64)
    orc.lib.so_oracle_rows32(_ptr(rp, i64), _ptr(ci, i32), _ptr(va, f32), _ptr(x, f32), n, _ptr(rows, i64),
                             len(rows), _ptr(y, f64), _ptr(b, f64), _threads(threads))
    return y, b
