"""Host-side multi-GPU bookkeeping on CPU with world_size 2 over gloo
(SURVEY §8e).  On the GPU box the same steps run through the library's NCCL
layer (spmk_mg_*, csrc/capi_mg.cu); here gloo collectives stand in for them
with the same call semantics, and the CPU oracle stands in for the kernels:

  * the equal-nnz row partition (the reference's partition arithmetic,
    kernels.hpp:124-129, applied to nonzeros: spmk_row_slices / spmk_mg_slice);
  * X replication by the chunked upload + all-gather of spmk_mg_allgather_x
    (multigpu.x_chunk / upload_range);
  * each rank's Y slice from its rebased slice (per-slice rule), then the Y
    exchange of the iterative driver, spmk_mg_allgather_rows: one broadcast
    of every rank's unequal slice from its owner;
  * the residual all-reduce.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2106_16064_b200.multigpu import slice_sizes, upload_range, x_chunk

HEAVY = (0.57, 0.19, 0.19, 0.05)


def mirror_allgather_rows(y, bounds, n):
    """gloo statement of spmk_mg_allgather_rows: rank g's rows from g."""
    flat = y.view(-1)
    for g in range(len(bounds) - 1):
        lo, hi = int(bounds[g]) * n, int(bounds[g + 1]) * n
        if hi > lo:
            dist.broadcast(flat[lo:hi], src=g)


def mirror_allgather_x(buf, chunk, rank, world):
    """gloo statement of spmk_mg_allgather_x (in place, equal chunks)."""
    parts = [torch.empty(chunk) for _ in range(world)]
    dist.all_gather(parts, buf[rank * chunk:(rank + 1) * chunk].clone())
    buf.copy_(torch.cat(parts))


def slice_csr(a, lo, hi):
    from oracle.oracle import Csr

    s, e = int(a.row_ptr[lo]), int(a.row_ptr[hi])
    return Csr(hi - lo, a.k, a.row_ptr[lo:hi + 1] - s, a.col_idx[s:e], a.val[s:e])


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _spmm_worker(rank, world, port, q):
    from oracle.oracle import Oracle

    _init(rank, world, port)
    try:
        orc = Oracle()
        a = orc.generate_rmat(10, 8, HEAVY, 3)
        n = 5
        bounds = orc.row_slices(a, world)
        # X: this rank uploads only its chunk of the host X, the all-gather
        # assembles the replica
        xh = orc.make_dense(a.k, n, 77)
        chunk = x_chunk(a.k, n, world)
        buf = torch.zeros(chunk * world)
        lo, hi = upload_range(a.k, n, world, rank)
        buf[lo:hi] = torch.from_numpy(xh.reshape(-1)[lo:hi])
        mirror_allgather_x(buf, chunk, rank, world)
        x = buf[: a.k * n].view(a.k, n).numpy()
        assert np.array_equal(x, xh)
        # this rank's slice, its rule, its Y rows
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        s = slice_csr(a, r0, r1)
        f = orc.extract_features(s) if s.m else (0.0, 0.0, 0.0)
        kid = orc.select_kernel(f[0], f[2], n)
        y = torch.zeros((a.m, n))
        if s.m:
            y[r0:r1] = torch.from_numpy(orc.spmm(s, kid, x))
        mirror_allgather_rows(y, bounds, n)
        res = torch.tensor([float(r1 - r0), float(rank)], dtype=torch.float64)
        dist.all_reduce(res)
        q.put((rank, kid, y.numpy().copy(), res.numpy().copy()))
    finally:
        dist.destroy_process_group()


def _run(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + (os.getpid() * 7 + hash(target.__name__)) % 2000
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def test_partitioned_spmm_bookkeeping_world2(orc):
    """Chunked X replication, per-slice rule, Y exchange: every rank ends with
    the concatenation of the per-slice reference results (row-split kernels:
    equal to the full product's rows)."""
    world = 2
    out = _run(_spmm_worker, world)
    a = orc.generate_rmat(10, 8, HEAVY, 3)
    x = orc.make_dense(a.k, 5, 77)
    bounds = orc.row_slices(a, world)
    want = np.zeros((a.m, 5), np.float32)
    for g in range(world):
        s = slice_csr(a, int(bounds[g]), int(bounds[g + 1]))
        f = orc.extract_features(s)
        kid = orc.select_kernel(f[0], f[2], 5)
        assert kid == out[g][1]
        want[bounds[g]:bounds[g + 1]] = orc.spmm(s, kid, x)
        if kid in (0, 2):  # row-split: a slice's rows equal the full product's
            assert np.array_equal(want[bounds[g]:bounds[g + 1]], orc.spmm(a, kid, x)[bounds[g]:bounds[g + 1]])
    for rank, _, y, res in out:
        assert np.array_equal(y.view(np.uint32), want.view(np.uint32)), rank
        assert res[0] == a.m and res[1] == 1


def _rows_worker(rank, world, port, bounds, q):
    _init(rank, world, port)
    try:
        m = bounds[-1]
        x = torch.full((m, 1), -1.0)
        lo, hi = bounds[rank], bounds[rank + 1]
        x[lo:hi, 0] = torch.arange(lo, hi, dtype=torch.float32) * (rank + 1)
        mirror_allgather_rows(x, bounds, 1)
        q.put((rank, x.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_exchange_unequal_slices_world2():
    world, bounds = 2, [0, 3, 17]  # unequal rows, as equal-nnz slices are
    out = _run(_rows_worker, world, bounds)
    want = np.concatenate([np.arange(0, 3) * 1.0, np.arange(3, 17) * 2.0]).astype(np.float32)
    for rank, x in out:
        assert np.array_equal(x[:, 0], want), rank


def test_upload_ranges_cover_x():
    for k, n, world in ((1000, 7, 3), (5, 1, 8), (0, 4, 2), (64, 64, 8)):
        c = x_chunk(k, n, world)
        assert c * world >= k * n
        ranges = [upload_range(k, n, world, g) for g in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == k * n
        for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
            assert a1 == b0 and a1 - a0 <= c


def test_equal_nnz_bounds_follow_partition(orc):
    """bounds[g] = lower_bound(rowPtr, partition(nnz, G, g).lo): the oracle
    restatement matches a direct numpy evaluation on a skewed matrix."""
    a = orc.generate_rmat(12, 8, HEAVY, 5)
    for parts in (1, 2, 4, 8):
        b = orc.row_slices(a, parts)
        want = [0] + [int(np.searchsorted(a.row_ptr, a.nnz * g // parts, side="left")) for g in range(1, parts)]
        want = [min(w, a.m) for w in want] + [a.m]
        assert list(b) == want
        sizes = [a.row_ptr[b[g + 1]] - a.row_ptr[b[g]] for g in range(parts)]
        assert sum(sizes) == a.nnz and sum(slice_sizes(b)) == a.m


def test_library_exports_nccl_layer():
    """The C ABI's multi-GPU entry points load without a GPU; NCCL itself is
    resolved at run time (a unique id can be made on any host with it)."""
    import ctypes as C

    from paper_2106_16064_b200.multigpu import Communicator, nccl_available

    v = nccl_available()
    if v is None:
        pytest.skip("libnccl.so.2 not loadable here")
    assert v >= 22000
    assert len(Communicator.unique_id()) == 128
