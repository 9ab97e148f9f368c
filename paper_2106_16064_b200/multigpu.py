"""Multi-GPU front end: one process per GPU, NCCL over NVLink /
NVSwitch through the library's own C ABI (spmk_mg_*, csrc/capi_mg.cu).

The row-partitioned configs cut A into equal-nnz row slices (the reference's
static partition, kernels.hpp:124-129, applied to nonzeros: spmk_row_slices),
replicate X once, and let every rank write its own Y slice with the per-slice
rule — there is no collective inside the SpMM.  The iterative driver
(pagerank.DistributedPageRank) exchanges Y slices with one grouped broadcast.

torch.distributed is used only to ship the 128-byte NCCL unique id from rank 0
(any backend); every collective on the data path is the library's.

Host bookkeeping shared by the CUDA path and the gloo tests:
  x_chunk(k, n, world)       floats per rank of the chunked X upload
  upload_range(k, n, world, g)   X elements rank g copies from the host
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

from .spmk import (DeviceCsr, Error, KernelConfig, KernelId, SelectorThresholds, _check, load_library)

vp, i64 = C.c_void_p, C.c_int64


def x_chunk(k: int, n: int, world: int) -> int:
    """Floats per rank when X (k x n) is uploaded in `world` equal chunks
    (the last padded): the all-gather of spmk_mg_allgather_x."""
    return -(-(k * n) // world) if k * n else 0


def upload_range(k: int, n: int, world: int, g: int) -> Tuple[int, int]:
    """[lo, hi) of X's flat elements rank g uploads from the host."""
    c = x_chunk(k, n, world)
    lo = min(g * c, k * n)
    return lo, min(lo + c, k * n)


def nccl_available() -> Optional[int]:
    """NCCL version if libnccl.so.2 loads, else None."""
    v = C.c_int()
    return v.value if load_library().spmk_mg_available(C.byref(v)) == 0 else None


class Communicator:
    """spmk_mg_t — this rank's NCCL communicator, bound to one GPU."""

    def __init__(self, unique_id: bytes, world: int, rank: int, device: int):
        self.lib = load_library()
        if len(unique_id) != 128:
            raise Error("NCCL unique id must be 128 bytes")
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        h = vp()
        _check(self.lib.spmk_mg_init(C.cast(buf, vp), int(world), int(rank), int(device), C.byref(h)))
        self._h = h
        self.world, self.rank, self.device = int(world), int(rank), int(device)

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_char * 128)()
        _check(load_library().spmk_mg_unique_id(C.cast(buf, vp)))
        return bytes(buf)

    @classmethod
    def from_torch_distributed(cls, group=None, device: Optional[int] = None) -> "Communicator":
        """Rank 0 of the torch.distributed group creates the id; it is shipped
        with broadcast_object_list (gloo or nccl), then NCCL is initialised by
        the library."""
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(obj, src=src, group=group)
        dev = torch.cuda.current_device() if device is None else device
        return cls(obj[0], world, rank, dev)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.spmk_mg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stream(stream):
        import torch

        st = stream if stream is not None else torch.cuda.current_stream()
        return vp(st.cuda_stream)

    def slice(self, full: DeviceCsr) -> Tuple[DeviceCsr, int, int]:
        """This rank's equal-nnz row slice of `full` (on this rank's GPU)."""
        h, lo, hi = vp(), i64(), i64()
        _check(self.lib.spmk_mg_slice(self._h, full._h, C.byref(h), C.byref(lo), C.byref(hi)))
        return DeviceCsr(h.value), lo.value, hi.value

    def broadcast(self, t, root: int = 0, stream=None) -> None:
        """In-place broadcast of a contiguous float32 CUDA tensor."""
        _check(self.lib.spmk_mg_broadcast(self._h, vp(t.data_ptr()), t.numel(), int(root), self._stream(stream)))

    def allgather_x(self, x_padded, chunk: int, stream=None) -> None:
        """In-place chunked all-gather: rank g owns x_padded[g*chunk:(g+1)*chunk]."""
        if x_padded.numel() < chunk * self.world:
            raise Error("X buffer smaller than world * chunk")
        _check(self.lib.spmk_mg_allgather_x(self._h, vp(x_padded.data_ptr()), int(chunk), self._stream(stream)))

    def allgather_rows(self, y, bounds: Sequence[int], n: int = 1, stream=None) -> None:
        """Rank g's rows [bounds[g], bounds[g+1]) of y (rows x n) to every rank
        (one NCCL group of broadcasts)."""
        b = (i64 * (self.world + 1))(*[int(v) for v in bounds])
        _check(self.lib.spmk_mg_allgather_rows(self._h, vp(y.data_ptr()), b, int(n), self._stream(stream)))

    def allreduce(self, t, stream=None) -> None:
        """In-place sum all-reduce of a float64 or int32 CUDA tensor."""
        import torch

        fn = {torch.float64: self.lib.spmk_mg_allreduce_f64, torch.int32: self.lib.spmk_mg_allreduce_i32}.get(t.dtype)
        if fn is None:
            raise Error("allreduce takes float64 or int32 tensors")
        _check(fn(self._h, vp(t.data_ptr()), t.numel(), self._stream(stream)))

    def barrier(self, stream=None) -> None:
        _check(self.lib.spmk_mg_barrier(self._h, self._stream(stream)))

    def spmm(self, a: DeviceCsr, x, y, stream=None, cfg: Optional[KernelConfig] = None,
             t: SelectorThresholds = SelectorThresholds()) -> KernelId:
        """This rank's SpMM on its slice with the per-slice rule (no collective)."""
        c, tc, kid = (cfg or KernelConfig())._c(), t._c(), C.c_int()
        n = x.shape[1] if x.dim() == 2 else 1
        _check(self.lib.spmk_mg_spmm(self._h, a._h, C.byref(tc), C.byref(c), vp(x.data_ptr()), n,
                                     vp(y.data_ptr()), self._stream(stream), C.byref(kid)))
        return KernelId(kid.value)


def slice_sizes(bounds: Sequence[int]) -> List[int]:
    return [int(bounds[g + 1]) - int(bounds[g]) for g in range(len(bounds) - 1)]
