"""Iterative SpMV driver, PageRank-style (BASELINE cfg5).

The reference has no iterative driver; this is the "next" item built on its
hot path: every iteration is one spmm(select_kernel(features, 1)) — par-ws
(VSR) on the BASELINE graphs — plus one fused update kernel:

    x_{t+1} = alpha * A x_t + (1 - alpha)/M + alpha * dangling(x_t)/M

with A column-stochastic (values 1/outdeg(col), set on the device by
spmk_csr_values_inv_column_counts) and dangling(x) the mass on columns with no
nonzeros.  Reductions (residual |x_{t+1}-x_t|_1, dangling mass) are
fixed-order, so a run is bit-reproducible.

Single GPU: the whole iteration loop is captured once into a CUDA graph
(plans are built in a warm-up step first) and replayed — no per-iteration
host work.

Multi-GPU (one process per GPU, torch.distributed over NCCL): A is cut into
equal-nnz row slices (spmk_row_slices, bit-exact vs the reference's
partition arithmetic), each rank keeps a full replica of x, computes its
slice of A x, updates its slice of x in place, then the slices are exchanged
with one broadcast per rank (slices are unequal in rows, so this is not a
padded all-gather); residual and dangling mass are all-reduced (2 doubles).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from .spmk import DeviceCsr, KernelId, _check, load_library

vp = C.c_void_p


def _lib():
    lib = load_library()
    return lib


def column_counts(a: DeviceCsr, stream=None):
    import torch

    counts = torch.empty(a.num_cols, dtype=torch.int32, device="cuda")
    st = stream or torch.cuda.current_stream()
    _check(_lib().spmk_column_counts(a._h, vp(counts.data_ptr()), vp(st.cuda_stream)))
    return counts


def make_column_stochastic(a: DeviceCsr, counts, stream=None) -> None:
    import torch

    st = stream or torch.cuda.current_stream()
    _check(_lib().spmk_csr_values_inv_column_counts(a._h, vp(counts.data_ptr()), vp(st.cuda_stream)))


class PageRank:
    """Single-GPU iterative SpMV on a resident, square A (values are rewritten
    to 1/outdeg(col) unless ``stochastic=False``)."""

    def __init__(self, a: DeviceCsr, alpha: float = 0.85, kernel=None,
                 stochastic: bool = True, counts=None, l2_persist_bytes: int = 0):
        import torch

        if a.num_rows != a.num_cols:
            raise ValueError("PageRank needs a square matrix")
        self.a, self.alpha, self.m = a, float(alpha), a.num_rows
        self.stream = torch.cuda.current_stream()
        self.counts = counts if counts is not None else column_counts(a, self.stream)
        if stochastic:
            make_column_stochastic(a, self.counts, self.stream)
        # kernel: a KernelId, None (the selection rule, select_kernel) or
        # "tuned" (the fastest variant measured on this graph, selection.tuned_kernel)
        if kernel == "tuned":
            from .selection import tuned_kernel

            self.kid, self.tune_times = tuned_kernel(a, 1)
        else:
            self.kid = kernel if kernel is not None else a.select(1)
        self.x = torch.full((self.m, 1), 1.0 / self.m, dtype=torch.float32, device="cuda")
        self.y = torch.empty((self.m, 1), dtype=torch.float32, device="cuda")
        self.state = torch.zeros(3, dtype=torch.float64, device="cuda")
        self.scratch = torch.empty(int(_lib().spmk_pagerank_scratch_doubles()), dtype=torch.float64, device="cuda")
        self.graph = None
        self.hist = None
        # bytes of x (from its start: the hot low-index columns of R-MAT
        # graphs) kept in L2 by an access-policy window on the captured stream
        self.l2_persist_bytes = int(l2_persist_bytes)

    def reset(self, x0=None):
        if x0 is None:
            self.x.fill_(1.0 / self.m)
        else:
            self.x.copy_(x0.reshape(self.m, 1))
        _check(_lib().spmk_pagerank_init(vp(self.x.data_ptr()), vp(self.counts.data_ptr()), self.m, self.m,
                                         C.c_double(self.alpha), vp(self.state.data_ptr()),
                                         vp(self.scratch.data_ptr()), vp(self.stream.cuda_stream)))

    def _step(self, t: int, hist_ptr: int):
        self.a.spmm(self.kid, self.x, self.y, stream=self.stream)
        _check(_lib().spmk_pagerank_step(vp(self.y.data_ptr()), vp(self.x.data_ptr()), vp(self.counts.data_ptr()),
                                         self.m, self.m, C.c_double(self.alpha), vp(self.state.data_ptr()),
                                         vp(self.scratch.data_ptr()), vp(hist_ptr), int(t),
                                         vp(self.stream.cuda_stream)))

    def step(self):
        """One iteration, eagerly (teacher-forced parity tests use this)."""
        self._step(0, 0)

    def capture(self, iters: int):
        """Capture `iters` iterations into one CUDA graph (after a warm-up
        iteration so every plan/scratch buffer exists)."""
        import torch

        self.hist = torch.zeros(iters, dtype=torch.float64, device="cuda")
        saved = self.x.clone()
        self.reset()
        self._step(0, 0)  # warm-up: builds the plans outside the capture
        torch.cuda.synchronize()
        self.x.copy_(saved)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        if self.l2_persist_bytes > 0:
            from .spmk import l2_persist_x

            l2_persist_x(s, self.x, min(self.l2_persist_bytes, self.m * 4))
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.stream = s
            with torch.cuda.graph(g, stream=s):
                for t in range(iters):
                    self._step(t, self.hist.data_ptr())
        torch.cuda.current_stream().wait_stream(s)
        self.stream = torch.cuda.current_stream()
        self.graph, self.iters = g, iters
        return g

    def run(self, iters: int = 50, graph: bool = True):
        """x_0 = 1/M, `iters` iterations; returns (x, per-iteration l1 residuals)."""
        import torch

        if graph:
            if self.graph is None or self.iters != iters:
                self.capture(iters)
            self.reset()
            self.graph.replay()
            return self.x, self.hist
        self.hist = torch.zeros(iters, dtype=torch.float64, device="cuda")
        self.reset()
        for t in range(iters):
            self._step(t, self.hist.data_ptr())
        return self.x, self.hist


# --------------------------------------------------------------------- multi-GPU
def _ipc_handle(t) -> bytes:
    buf = (C.c_char * 64)()
    _check(_lib().spmk_ipc_handle(vp(t.data_ptr()), C.cast(buf, vp)))
    return bytes(buf)


def _ipc_open(handle: bytes) -> int:
    buf = (C.c_char * 64).from_buffer_copy(handle)
    out = vp()
    _check(_lib().spmk_ipc_open(C.cast(buf, vp), C.byref(out)))
    return out.value


class DistributedPageRank:
    """One rank of the row-partitioned iterative SpMV.  ``full`` is the whole
    square A on this rank's GPU (each rank keeps only its slice afterwards).

    Collectives go through the library's NCCL layer (``multigpu.Communicator``,
    spmk_mg_*): the global out-degree and (residual, dangling) all-reduces, and
    for exchange="nccl" the Y exchange — update this rank's slice of x in
    place, then spmk_mg_allgather_rows (one grouped broadcast per rank's
    unequal slice).  exchange="p2p": x is double-buffered
    and every rank's update kernel stores its slice of x_next straight into
    all ranks' replicas (CUDA-IPC-mapped peer buffers, P2P over NVLink) —
    update and all-gather fused into one kernel; the residual all-reduce that
    follows is the barrier before the next SpMV reads x_next."""

    def __init__(self, full: DeviceCsr, alpha: float = 0.85, group=None, exchange: str = "nccl", kernel=None,
                 comm=None):
        import torch
        import torch.distributed as dist

        from .multigpu import Communicator

        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' or 'p2p'")
        self.comm = comm if comm is not None else Communicator.from_torch_distributed(group)
        self.rank, self.world = self.comm.rank, self.comm.world
        self.group, self.alpha, self.m, self.exchange = group, float(alpha), full.num_rows, exchange
        dev = torch.cuda.current_device()
        self.bounds = [int(b) for b in full.row_slices(self.world)]
        lo, hi = self.bounds[self.rank], self.bounds[self.rank + 1]
        self.lo, self.hi = lo, hi
        self.a = full.slice(lo, hi, device=dev)
        counts = column_counts(self.a)
        self.comm.allreduce(counts)  # global out-degrees (integer: exact)
        self.counts = counts
        make_column_stochastic(self.a, counts)
        # per-slice choice: the rule on this slice's features (None), "tuned"
        # (fastest variant measured on this slice) or a fixed KernelId
        if kernel == "tuned":
            from .selection import tuned_kernel

            self.kid, self.tune_times = tuned_kernel(self.a, 1)
        else:
            self.kid = kernel if kernel is not None else self.a.select(1)
        self.y = torch.empty((hi - lo, 1), dtype=torch.float32, device="cuda")
        self.state = torch.zeros(3, dtype=torch.float64, device="cuda")
        self.scratch = torch.empty(int(_lib().spmk_pagerank_scratch_doubles()), dtype=torch.float64, device="cuda")
        self.xbuf = [torch.full((self.m, 1), 1.0 / self.m, dtype=torch.float32, device="cuda")]
        self.cur = 0
        self.opened: List[int] = []
        if exchange == "p2p":
            if self.world > 8:
                raise ValueError("p2p exchange supports up to 8 ranks")
            self.xbuf.append(torch.empty_like(self.xbuf[0]))
            torch.cuda.synchronize()
            self.peers = []
            for b in range(2):
                mine = _ipc_handle(self.xbuf[b])
                handles = [None] * self.world
                dist.all_gather_object(handles, mine, group=group)
                ptrs = []
                for r in range(self.world):
                    if r == self.rank:
                        ptrs.append(self.xbuf[b].data_ptr())
                    else:
                        p = _ipc_open(handles[r])
                        self.opened.append(p)
                        ptrs.append(p)
                self.peers.append((vp * self.world)(*ptrs))
            dist.barrier(group=group)

    @property
    def x(self):
        return self.xbuf[self.cur]

    def close(self):
        for p in self.opened:
            _lib().spmk_ipc_close(vp(p))
        self.opened = []

    def _global_base(self):
        red = self.state[1:3].clone()
        self.comm.allreduce(red)
        self.state[1:3] = red
        self.state[0] = (1.0 - self.alpha) / self.m + self.alpha * red[1] / self.m

    def reset(self):
        import torch
        import torch.distributed as dist

        for b in self.xbuf:
            b.fill_(1.0 / self.m)
        self.cur = 0
        st = torch.cuda.current_stream()
        _check(_lib().spmk_pagerank_init(vp(self.x[self.lo:self.hi].data_ptr()),
                                         vp(self.counts[self.lo:].data_ptr()), self.hi - self.lo, self.m,
                                         C.c_double(self.alpha), vp(self.state.data_ptr()),
                                         vp(self.scratch.data_ptr()), vp(st.cuda_stream)))
        self._global_base()
        if self.exchange == "p2p":
            torch.cuda.synchronize()
            dist.barrier(group=self.group)  # every replica initialised before peers write

    def step(self):
        import torch

        st = torch.cuda.current_stream()
        x = self.x
        if self.hi > self.lo:
            self.a.spmm(self.kid, x, self.y, stream=st)
        if self.exchange == "p2p":
            nxt = 1 - self.cur
            _check(_lib().spmk_pagerank_step_p2p(vp(self.y.data_ptr()), vp(x.data_ptr()), self.peers[nxt],
                                                 self.world, vp(self.counts.data_ptr()), self.lo,
                                                 self.hi - self.lo, self.m, C.c_double(self.alpha),
                                                 vp(self.state.data_ptr()), vp(self.scratch.data_ptr()),
                                                 vp(st.cuda_stream)))
            self._global_base()  # all-reduce: also the barrier before x_next is read
            self.cur = nxt
            return
        xs = x[self.lo:self.hi]
        _check(_lib().spmk_pagerank_step(vp(self.y.data_ptr()), vp(xs.data_ptr()),
                                         vp(self.counts[self.lo:].data_ptr()), self.hi - self.lo, self.m,
                                         C.c_double(self.alpha), vp(self.state.data_ptr()),
                                         vp(self.scratch.data_ptr()), vp(0), 0, vp(st.cuda_stream)))
        self._global_base()
        self.comm.allgather_rows(x, self.bounds, 1)

    def run(self, iters: int = 50):
        self.reset()
        hist = []
        for _ in range(iters):
            self.step()
            hist.append(self.state[1].clone())
        return self.x, hist
