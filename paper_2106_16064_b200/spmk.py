"""Python front end of the B200-native spmk engine (ctypes over the C ABI).

Mirrors the reference interface of the hot path (proj/include/spmk):
``KernelId`` constants and ``kernel_name/kernel_index/parse_kernel``
(kernels.hpp:17-57), ``KernelConfig`` (kernels.hpp:81-87),
``SelectorThresholds``/``select_kernel`` (selector.hpp:16-34),
``MatrixFeatures``/``extract_features`` (csr.hpp:86-92,166-181),
``plan_balanced`` (kernels.hpp:133-149) and ``spmm`` (kernels.hpp:457-464).
Errors raise ``Error`` (error.hpp:10-13).

Two ways to call it:
* ``DeviceCsr`` — a resident handle; ``spmm`` takes device pointers (e.g. the
  ``data_ptr()`` of torch CUDA tensors) and a stream: the hot path.
* ``spmm(id, a, x, cfg)`` on host ``CsrMatrix``/numpy operands — the
  reference's value-returning call shape (uploads, runs, downloads).

There is NO CPU fallback: importing this module loads libspmk_b200.so and
every compute call runs the sm_100a kernels; without the library it raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspmk_b200.so")


class Error(RuntimeError):
    """spmk::Error (error.hpp:10-13)."""


class UnsupportedError(Error):
    """Valid for the reference but not on the device path (e.g. T=double)."""


# --------------------------------------------------------------------- ctypes
i64, u64, f64, f32, i32, vp = C.c_int64, C.c_uint64, C.c_double, C.c_float, C.c_int32, C.c_void_p
P = C.POINTER


class _Cfg(C.Structure):
    _fields_ = [("lane_width", u64), ("vdl_group", u64), ("seq_chunk", u64), ("worker_count", u64)]


class _Thr(C.Structure):
    _fields_ = [("n_parallel_max", u64), ("t_parallel_avg", f64), ("t_cv", f64)]


class _Feat(C.Structure):
    _fields_ = [("avg_row", f64), ("stdv_row", f64), ("cv", f64), ("num_rows", i64), ("nnz", i64)]


_SIGS = {
    "spmk_last_error": ([], C.c_char_p),
    "spmk_spmm_path": ([vp, C.c_int, P(_Cfg), i64, P(C.c_int)], C.c_int),
    "spmk_version": ([], C.c_int),
    "spmk_default_config": ([P(_Cfg)], None),
    "spmk_default_thresholds": ([P(_Thr)], None),
    "spmk_check_config": ([P(_Cfg)], C.c_int),
    "spmk_kernel_name": ([C.c_int], C.c_char_p),
    "spmk_parse_kernel": ([C.c_char_p, P(C.c_int)], C.c_int),
    "spmk_csr_create": ([i64, i64, i64, P(i64), P(i64), P(f32), C.c_int, P(vp)], C.c_int),
    "spmk_csr_create_device": ([i64, i64, i64, vp, vp, vp, C.c_int, P(vp)], C.c_int),
    "spmk_csr_slice": ([vp, i64, i64, C.c_int, P(vp)], C.c_int),
    "spmk_csr_abs_copy": ([vp, P(vp)], C.c_int),
    "spmk_csr_destroy": ([vp], C.c_int),
    "spmk_csr_validate": ([vp], C.c_int),
    "spmk_csr_set_tuning": ([vp, C.c_char_p, i64], C.c_int),
    "spmk_csr_get_tuning": ([vp, C.c_char_p, P(i64)], C.c_int),
    "spmk_csr_info": ([vp, P(i64), P(i64), P(i64), P(i64), P(i64)], C.c_int),
    "spmk_csr_device_arrays": ([vp, P(vp), P(vp), P(vp)], C.c_int),
    "spmk_csr_download": ([vp, P(i64), P(i64), P(f32)], C.c_int),
    "spmk_features_compute": ([vp, P(_Feat)], C.c_int),
    "spmk_features_host": ([i64, P(i64), P(_Feat)], C.c_int),
    "spmk_select": ([P(_Feat), u64, P(_Thr)], C.c_int),
    "spmk_select_for": ([vp, u64, P(_Thr), P(C.c_int)], C.c_int),
    "spmk_plan": ([vp, i64, P(i64), P(i64)], C.c_int),
    "spmk_plan_elem_row": ([vp, P(i64)], C.c_int),
    "spmk_partition": ([i64, i64, i64, P(i64), P(i64)], None),
    "spmk_row_slices": ([vp, i64, P(i64)], C.c_int),
    "spmk_spmm": ([vp, C.c_int, P(_Cfg), vp, i64, vp, vp], C.c_int),
    "spmk_spmm_auto": ([vp, P(_Thr), P(_Cfg), vp, i64, vp, vp, P(C.c_int)], C.c_int),
    "spmk_spmm_host": ([vp, C.c_int, P(_Cfg), P(f32), i64, P(f32), vp], C.c_int),
    "spmk_spmm_host_async": ([vp, C.c_int, P(_Cfg), P(f32), i64, P(f32), vp], C.c_int),
    "spmk_spmm_csr_host": ([i64, i64, i64, P(i64), P(i64), P(f32), C.c_int, P(_Cfg), P(f32), i64,
                            P(f32), C.c_int], C.c_int),
    "spmk_kernel_stats": ([vp, C.c_int, P(_Cfg), i64, P(u64), P(u64)], C.c_int),
    "spmk_kernel_tolerance": ([i64], f64),
    "spmk_l2_persist_x": ([vp, vp, C.c_size_t], C.c_int),
    "spmk_launch_count": ([], u64),
    "spmk_timing_enable": ([C.c_int], C.c_int),
    "spmk_timing_last": ([P(f32), P(f32)], C.c_int),
    "spmk_timing_summary": ([P(f32), P(f32), P(C.c_int)], C.c_int),
    "spmk_mg_available": ([P(C.c_int)], C.c_int),
    "spmk_mg_unique_id": ([vp], C.c_int),
    "spmk_mg_init": ([vp, C.c_int, C.c_int, C.c_int, P(vp)], C.c_int),
    "spmk_mg_destroy": ([vp], C.c_int),
    "spmk_mg_info": ([vp, P(C.c_int), P(C.c_int), P(C.c_int)], C.c_int),
    "spmk_mg_slice": ([vp, vp, P(vp), P(i64), P(i64)], C.c_int),
    "spmk_mg_broadcast": ([vp, vp, i64, C.c_int, vp], C.c_int),
    "spmk_mg_allgather_x": ([vp, vp, i64, vp], C.c_int),
    "spmk_mg_allgather_rows": ([vp, vp, P(i64), i64, vp], C.c_int),
    "spmk_mg_allreduce_f64": ([vp, vp, i64, vp], C.c_int),
    "spmk_mg_allreduce_i32": ([vp, vp, i64, vp], C.c_int),
    "spmk_mg_barrier": ([vp, vp], C.c_int),
    "spmk_mg_spmm": ([vp, vp, P(_Thr), P(_Cfg), vp, i64, vp, vp, P(C.c_int)], C.c_int),
    "spmk_generate_rmat": ([C.c_uint32, u64, f64, f64, f64, f64, u64, C.c_int, P(vp)], C.c_int),
    "spmk_make_dense": ([i64, i64, u64, vp, vp], C.c_int),
    "spmk_make_dense_host": ([i64, i64, u64, P(f32), C.c_int], C.c_int),
    "spmk_measure_kernel": ([vp, C.c_int, P(_Cfg), i64, u64, i64, i64, C.c_int, P(f64), P(C.c_int)], C.c_int),
    "spmk_column_counts": ([vp, vp, vp], C.c_int),
    "spmk_csr_values_inv_column_counts": ([vp, vp, vp], C.c_int),
    "spmk_pagerank_scratch_doubles": ([], i64),
    "spmk_pagerank_init": ([vp, vp, i64, i64, f64, vp, vp, vp], C.c_int),
    "spmk_pagerank_step": ([vp, vp, vp, i64, i64, f64, vp, vp, vp, C.c_int32, vp], C.c_int),
    "spmk_pagerank_step_p2p": ([vp, vp, P(vp), C.c_int32, vp, i64, i64, i64, f64, vp, vp, vp], C.c_int),
    "spmk_ipc_handle": ([vp, vp], C.c_int),
    "spmk_ipc_open": ([vp, P(vp)], C.c_int),
    "spmk_ipc_close": ([vp], C.c_int),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib: Optional[C.CDLL] = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libspmk_b200.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise Error(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


_STATUS = {1: "EINVAL", 2: "EDIM", 3: "ECUDA", 4: "ENOMEM", 5: "ENCCL", 6: "EUNSUPPORTED"}


def _check(st: int):
    if st != 0:
        msg = load_library().spmk_last_error().decode()
        cls = UnsupportedError if st == 6 else Error
        raise cls(f"spmk {_STATUS.get(st, st)}: {msg}")


def _ptr(a, ct):
    return a.ctypes.data_as(P(ct))


# --------------------------------------------------------------------- types
@dataclass(frozen=True)
class KernelId:
    """KernelId{Reduction, Balancing} (kernels.hpp:21-26); index = 2*seq + ws."""

    index: int

    @property
    def name(self) -> str:
        return kernel_name(self)


kParRowSplit = KernelId(0)
kParBalanced = KernelId(1)
kSeqRowSplit = KernelId(2)
kSeqBalanced = KernelId(3)
kAllKernels = (kParRowSplit, kParBalanced, kSeqRowSplit, kSeqBalanced)
_NAMES = ("par-rs", "par-ws", "seq-rs", "seq-ws")


def kernel_name(kid: KernelId) -> str:
    return _NAMES[kid.index]


def kernel_index(kid: KernelId) -> int:
    return kid.index


def parse_kernel(name: str) -> KernelId:
    if name not in _NAMES:
        raise Error(f"unknown kernel name: {name}")
    return KernelId(_NAMES.index(name))


@dataclass
class KernelConfig:
    """KernelConfig (kernels.hpp:81-87); worker_count is ignored on device."""

    lane_width: int = 32
    vdl_group: int = 0
    seq_chunk: int = 256
    worker_count: int = 0

    def _c(self) -> _Cfg:
        vals = (self.lane_width, self.vdl_group, self.seq_chunk, self.worker_count)
        if any(int(v) < 0 for v in vals):
            raise Error("KernelConfig fields must be non-negative")
        return _Cfg(*[int(v) for v in vals])


def check_config(cfg: KernelConfig) -> None:
    c = cfg._c()
    _check(load_library().spmk_check_config(C.byref(c)))


@dataclass
class SelectorThresholds:
    """SelectorThresholds (selector.hpp:16-22)."""

    n_parallel_max: int = 4
    t_parallel_avg: float = 32.0
    t_cv: float = 1.0

    def _c(self) -> _Thr:
        return _Thr(int(self.n_parallel_max), float(self.t_parallel_avg), float(self.t_cv))


@dataclass
class MatrixFeatures:
    """MatrixFeatures (csr.hpp:86-92)."""

    avg_row: float = 0.0
    stdv_row: float = 0.0
    cv: float = 0.0
    num_rows: int = 0
    nnz: int = 0

    def _c(self) -> _Feat:
        return _Feat(self.avg_row, self.stdv_row, self.cv, self.num_rows, self.nnz)

    @staticmethod
    def _from(f: _Feat) -> "MatrixFeatures":
        return MatrixFeatures(f.avg_row, f.stdv_row, f.cv, f.num_rows, f.nnz)


@dataclass
class CsrMatrix:
    """Host CSR in the reference layout (csr.hpp:24-57): int64 indices, fp32 values."""

    num_rows: int
    num_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int64)
        if isinstance(self.values, np.ndarray) and self.values.dtype == np.float64:
            raise UnsupportedError("T=double: the device path is fp32 only")
        self.values = np.ascontiguousarray(self.values, dtype=np.float32)

    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def max_row_nnz(self) -> int:
        return int(np.diff(self.row_ptr).max()) if self.num_rows else 0


def select_kernel(f: MatrixFeatures, n: int, t: SelectorThresholds = SelectorThresholds()) -> KernelId:
    """selector.hpp:28-34 (pure host function, evaluated in the library)."""
    fc, tc = f._c(), t._c()
    return KernelId(load_library().spmk_select(C.byref(fc), int(n), C.byref(tc)))


def extract_features(a: CsrMatrix) -> MatrixFeatures:
    """csr.hpp:166-181 on a host CSR (reference summation order)."""
    out = _Feat()
    _check(load_library().spmk_features_host(a.num_rows, _ptr(a.row_ptr, i64), C.byref(out)))
    return MatrixFeatures._from(out)


def kernel_tolerance(max_row_nnz: int) -> float:
    return load_library().spmk_kernel_tolerance(int(max_row_nnz))


def partition(items: int, parts: int, w: int):
    lo, hi = i64(), i64()
    load_library().spmk_partition(items, parts, w, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


# --------------------------------------------------------------------- handle
class DeviceCsr:
    """Resident A on one GPU (spmk_csr_t).  Construct with ``from_host``,
    ``from_device`` (int32 CUDA tensors) or ``generate_rmat``."""

    def __init__(self, handle, keepalive=None):
        self._h = C.c_void_p(handle)
        self._keep = keepalive
        self.lib = load_library()
        m, k, nnz, mx, ne = i64(), i64(), i64(), i64(), i64()
        _check(self.lib.spmk_csr_info(self._h, C.byref(m), C.byref(k), C.byref(nnz), C.byref(mx), C.byref(ne)))
        self.num_rows, self.num_cols, self.nnz = m.value, k.value, nnz.value
        self.max_row_nnz, self.empty_rows = mx.value, ne.value

    # constructors
    @classmethod
    def from_host(cls, a: CsrMatrix, device: int = 0) -> "DeviceCsr":
        lib = load_library()
        h = vp()
        _check(lib.spmk_csr_create(a.num_rows, a.num_cols, a.nnz(), _ptr(a.row_ptr, i64),
                                   _ptr(a.col_idx, i64), _ptr(a.values, f32), device, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_device(cls, num_rows, num_cols, row_ptr, col_idx, values, copy=True) -> "DeviceCsr":
        """int32 CUDA tensors (torch) already in HBM."""
        lib = load_library()
        h = vp()
        _check(lib.spmk_csr_create_device(num_rows, num_cols, int(col_idx.numel()), row_ptr.data_ptr(),
                                          col_idx.data_ptr(), values.data_ptr(), int(copy), C.byref(h)))
        return cls(h.value, None if copy else (row_ptr, col_idx, values))

    @classmethod
    def generate_rmat(cls, scale, edge_factor, skew=(0.57, 0.19, 0.19, 0.05), seed=1, device=0):
        """generate_rmat<float> (rmat.hpp:61-88) on the device, bit-exact."""
        lib = load_library()
        h = vp()
        _check(lib.spmk_generate_rmat(scale, edge_factor, *skew, seed, device, C.byref(h)))
        return cls(h.value)

    def slice(self, row_begin: int, row_end: int, device: int = 0) -> "DeviceCsr":
        h = vp()
        _check(self.lib.spmk_csr_slice(self._h, row_begin, row_end, device, C.byref(h)))
        return DeviceCsr(h.value)

    def abs_copy(self) -> "DeviceCsr":
        """|A| (same structure, |values|) as a new resident handle."""
        h = vp()
        _check(self.lib.spmk_csr_abs_copy(self._h, C.byref(h)))
        return DeviceCsr(h.value)

    def close(self):
        if self._h is not None and self._h.value:
            self.lib.spmk_csr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # queries
    def validate(self) -> None:
        """validate (csr.hpp:95-119): raises Error unless every row's columns
        are strictly increasing (bounds are checked at creation)."""
        _check(self.lib.spmk_csr_validate(self._h))

    def set_tuning(self, key: str, value: int) -> None:
        """Per-handle performance knob (never changes a result bit)."""
        _check(self.lib.spmk_csr_set_tuning(self._h, key.encode(), int(value)))

    def spmm_path(self, kid: KernelId, n: int, cfg: Optional[KernelConfig] = None) -> str:
        """'sell' when spmm(kid, X of width n) runs the lane-per-job seq-ws sweep
        (+ fold pass; empty rows written by the sweep), else 'tile'."""
        c = (cfg or KernelConfig())._c()
        out = C.c_int()
        _check(self.lib.spmk_spmm_path(self._h, kid.index, C.byref(c), int(n), C.byref(out)))
        return "sell" if out.value == 1 else "tile"

    def get_tuning(self, key: str) -> int:
        v = i64()
        _check(self.lib.spmk_csr_get_tuning(self._h, key.encode(), C.byref(v)))
        return v.value

    def download(self) -> CsrMatrix:
        rp = np.empty(self.num_rows + 1, np.int64)
        ci = np.empty(max(self.nnz, 1), np.int64)
        va = np.empty(max(self.nnz, 1), np.float32)
        _check(self.lib.spmk_csr_download(self._h, _ptr(rp, i64), _ptr(ci, i64), _ptr(va, f32)))
        return CsrMatrix(self.num_rows, self.num_cols, rp, ci[: self.nnz], va[: self.nnz])

    def device_arrays(self):
        a, b, c = vp(), vp(), vp()
        _check(self.lib.spmk_csr_device_arrays(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def features(self) -> MatrixFeatures:
        out = _Feat()
        _check(self.lib.spmk_features_compute(self._h, C.byref(out)))
        return MatrixFeatures._from(out)

    def select(self, n: int, t: SelectorThresholds = SelectorThresholds()) -> KernelId:
        out = C.c_int()
        tc = t._c()
        _check(self.lib.spmk_select_for(self._h, int(n), C.byref(tc), C.byref(out)))
        return KernelId(out.value)

    def plan(self, chunk: int):
        """plan_balanced: (chunk_first_row[num_chunks] = elem_row[q*chunk], num_chunks)."""
        nch = i64()
        _check(self.lib.spmk_plan(self._h, chunk, None, C.byref(nch)))
        out = np.empty(max(nch.value, 1), np.int64)
        _check(self.lib.spmk_plan(self._h, chunk, _ptr(out, i64), C.byref(nch)))
        return out[: nch.value], nch.value

    def elem_row(self) -> np.ndarray:
        out = np.empty(max(self.nnz, 1), np.int64)
        _check(self.lib.spmk_plan_elem_row(self._h, _ptr(out, i64)))
        return out[: self.nnz]

    def row_slices(self, parts: int) -> np.ndarray:
        out = np.empty(parts + 1, np.int64)
        _check(self.lib.spmk_row_slices(self._h, parts, _ptr(out, i64)))
        return out

    def kernel_stats(self, kid: KernelId, n: int, cfg: KernelConfig = KernelConfig()):
        m, s = u64(), u64()
        c = cfg._c()
        _check(self.lib.spmk_kernel_stats(self._h, kid.index, C.byref(c), n, C.byref(m), C.byref(s)))
        return m.value, s.value

    # compute
    def _check_out(self, y, n):
        if not (isinstance(y, np.ndarray) and y.dtype == np.float32 and y.flags.c_contiguous
                and y.shape == (self.num_rows, n)):
            raise Error(f"Y must be a C-contiguous float32 array of shape ({self.num_rows}, {n})")

    def spmm_ptr(self, kid: KernelId, d_x: int, n: int, d_y: int, stream: int = 0,
                 cfg: Optional[KernelConfig] = None) -> None:
        """Y = A*X on device pointers (asynchronous on `stream`)."""
        c = (cfg or KernelConfig())._c()
        _check(self.lib.spmk_spmm(self._h, kid.index, C.byref(c), C.c_void_p(d_x), n, C.c_void_p(d_y),
                                  C.c_void_p(stream)))

    def spmm(self, kid: KernelId, x, y=None, stream=None, cfg: Optional[KernelConfig] = None):
        """torch CUDA tensors in/out (fp32, row-major)."""
        import torch

        if not (x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.dim() in (1, 2)):
            raise Error("X must be a contiguous float32 CUDA tensor of 1 or 2 dimensions")
        n = x.shape[1] if x.dim() == 2 else 1
        if x.shape[0] != self.num_cols:
            raise Error(f"dimension mismatch: A is {self.num_rows}x{self.num_cols}, X has {x.shape[0]} rows")
        if y is None:
            y = torch.empty((self.num_rows, n), dtype=torch.float32, device=x.device)
        elif not (y.is_cuda and y.dtype == torch.float32 and y.is_contiguous() and y.device == x.device
                  and y.numel() == self.num_rows * n and (y.dim() == 2 and tuple(y.shape) == (self.num_rows, n)
                                                          or y.dim() == 1 and n == 1)):
            raise Error(f"Y must be a contiguous float32 CUDA tensor of shape ({self.num_rows}, {n}) "
                        f"on {x.device}")
        st = stream if stream is not None else torch.cuda.current_stream(x.device)
        self.spmm_ptr(kid, x.data_ptr(), n, y.data_ptr(), st.cuda_stream, cfg)
        return y

    def spmm_auto(self, x, y=None, stream=None, cfg=None, t: SelectorThresholds = SelectorThresholds()):
        kid = self.select(x.shape[1], t)
        return self.spmm(kid, x, y, stream, cfg), kid

    def spmm_host(self, kid: KernelId, x: np.ndarray, cfg: Optional[KernelConfig] = None,
                  stream: int = 0, out: Optional[np.ndarray] = None) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        if x.ndim != 2 or x.shape[0] != self.num_cols:
            raise Error(f"dimension mismatch: A is {self.num_rows}x{self.num_cols}, X has shape {x.shape}")
        n = x.shape[1]
        y = out if out is not None else np.empty((self.num_rows, n), np.float32)
        self._check_out(y, n)
        c = (cfg or KernelConfig())._c()
        _check(self.lib.spmk_spmm_host(self._h, kid.index, C.byref(c), _ptr(x, f32), n, _ptr(y, f32),
                                       C.c_void_p(stream)))
        return y

    def spmm_host_async(self, kid: KernelId, x: np.ndarray, out: np.ndarray, stream: int,
                        cfg: Optional[KernelConfig] = None) -> None:
        """Enqueue H2D(x) -> Y = A x -> D2H(out) on `stream` (no synchronize);
        x and out must be pinned and stay alive until the stream passes."""
        if not (isinstance(x, np.ndarray) and x.dtype == np.float32 and x.flags.c_contiguous and x.ndim == 2
                and x.shape[0] == self.num_cols):
            raise Error(f"X must be a C-contiguous float32 array of shape ({self.num_cols}, n)")
        self._check_out(out, x.shape[1])
        c = (cfg or KernelConfig())._c()
        _check(self.lib.spmk_spmm_host_async(self._h, kid.index, C.byref(c), _ptr(x, f32), x.shape[1],
                                             _ptr(out, f32), C.c_void_p(stream)))


def spmm(kid: KernelId, a: CsrMatrix, x: np.ndarray, cfg: KernelConfig = KernelConfig(),
         device: int = 0) -> np.ndarray:
    """spmm(KernelId, CsrMatrix, DenseMatrix, KernelConfig) -> DenseMatrix
    (kernels.hpp:457-464), host operands, computed on the GPU."""
    x = np.asarray(x)
    if x.dtype == np.float64:
        raise UnsupportedError("T=double: the device path is fp32 only")
    x = np.ascontiguousarray(x, np.float32)
    if x.ndim == 1:
        x = x[:, None]
    if a.num_cols != x.shape[0]:
        raise Error(f"dimension mismatch: A is {a.num_rows}x{a.num_cols}, X has {x.shape[0]} rows")
    check_config(cfg)
    n = x.shape[1]
    y = np.empty((a.num_rows, n), np.float32)
    c = cfg._c()
    _check(load_library().spmk_spmm_csr_host(a.num_rows, a.num_cols, a.nnz(), _ptr(a.row_ptr, i64),
                                             _ptr(a.col_idx, i64), _ptr(a.values, f32), kid.index,
                                             C.byref(c), _ptr(x, f32), n, _ptr(y, f32), device))
    return y


def make_dense_device(rows: int, cols: int, seed: int, device=None):
    """make_dense<float> (corpus.hpp:116-122) generated on the device."""
    import torch

    out = torch.empty((rows, cols), dtype=torch.float32, device=device or "cuda")
    st = torch.cuda.current_stream(out.device)
    _check(load_library().spmk_make_dense(rows, cols, seed, C.c_void_p(out.data_ptr()),
                                          C.c_void_p(st.cuda_stream)))
    return out


def l2_persist_x(stream, x, nbytes=None):
    """Access-policy window keeping X resident in L2 for kernels on `stream`."""
    ptr = x.data_ptr() if x is not None else None
    nb = 0 if x is None else (nbytes if nbytes is not None else x.numel() * 4)
    _check(load_library().spmk_l2_persist_x(C.c_void_p(stream.cuda_stream), C.c_void_p(ptr), nb))


def launch_count() -> int:
    """Kernel launches issued by libspmk_b200.so so far (all entry points)."""
    return int(load_library().spmk_launch_count())


def timing_enable(on: bool = True) -> None:
    _check(load_library().spmk_timing_enable(int(on)))


def timing_last():
    """(dominant-kernel ms, whole-call ms) of the last spmm on this thread."""
    a, b = f32(), f32()
    _check(load_library().spmk_timing_last(C.byref(a), C.byref(b)))
    return a.value, b.value


def timing_summary():
    """(total dominant-kernel ms, total whole-call ms, calls) over the spmm calls
    on this thread since timing_enable (the last 256 kept)."""
    a, b, n = f32(), f32(), C.c_int()
    _check(load_library().spmk_timing_summary(C.byref(a), C.byref(b), C.byref(n)))
    return a.value, b.value, n.value
