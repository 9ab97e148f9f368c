"""Host-side multi-GPU logic on CPU with world_size 2 over gloo:
the equal-nnz row partition (restated from the reference's partition
arithmetic, kernels.hpp:124-129) and the unequal-slice exchange used by the
iterative driver (pagerank.exchange_slices), with the residual all-reduce."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2106_16064_b200.pagerank import exchange_slices


def _worker(rank, world, port, bounds, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = bounds[-1]
        x = torch.full((m,), -1.0)
        lo, hi = bounds[rank], bounds[rank + 1]
        x[lo:hi] = torch.arange(lo, hi, dtype=torch.float32) * (rank + 1)
        exchange_slices(x, bounds)
        res = torch.tensor([float(hi - lo), float(rank)], dtype=torch.float64)
        dist.all_reduce(res)
        q.put((rank, x.numpy().copy(), res.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_exchange_unequal_slices_world2():
    world, bounds = 2, [0, 3, 17]  # unequal rows, as equal-nnz slices are
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, bounds, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    want = np.concatenate([np.arange(0, 3) * 1.0, np.arange(3, 17) * 2.0]).astype(np.float32)
    for rank, x, res in out:
        assert np.array_equal(x, want), rank
        assert res[0] == 17 and res[1] == 1


def test_equal_nnz_bounds_follow_partition(orc):
    """bounds[g] = lower_bound(rowPtr, partition(nnz, G, g).lo): the oracle
    restatement matches a direct numpy evaluation on a skewed matrix."""
    a = orc.generate_rmat(12, 8, (0.57, 0.19, 0.19, 0.05), 5)
    for parts in (1, 2, 4, 8):
        b = orc.row_slices(a, parts)
        want = [0] + [int(np.searchsorted(a.row_ptr, a.nnz * g // parts, side="left")) for g in range(1, parts)]
        want = [min(w, a.m) for w in want] + [a.m]
        assert list(b) == want
        sizes = [a.row_ptr[b[g + 1]] - a.row_ptr[b[g]] for g in range(parts)]
        assert sum(sizes) == a.nnz
