"""The library's NCCL layer (spmk_mg_*, csrc/capi_mg.cu) on the device at
world size 1 (the box has one GPU; N>1 runs under torchrun in bench.py): the
communicator, slicing, the X broadcast / chunked all-gather, the grouped row
exchange and the all-reduces are exercised end to end; the host bookkeeping
at world size 2 is covered over gloo (test_multigpu_gloo.py)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200.inputs import SKEWS  # noqa: E402
from paper_2106_16064_b200.multigpu import Communicator, nccl_available, upload_range, x_chunk  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    if nccl_available() is None:
        pytest.fail("libnccl.so.2 must be loadable on the GPU box")
    c = Communicator(Communicator.unique_id(), 1, 0, 0)
    yield c
    c.close()


def test_world1_collectives(comm):
    x = torch.arange(1000, dtype=torch.float32, device="cuda")
    comm.broadcast(x, root=0)
    y = torch.arange(40, dtype=torch.float32, device="cuda").view(20, 2)
    want = y.clone()
    comm.allgather_rows(y, [0, 20], n=2)
    c = torch.tensor([1.5, -2.0], dtype=torch.float64, device="cuda")
    comm.allreduce(c)
    i = torch.tensor([3, 4], dtype=torch.int32, device="cuda")
    comm.allreduce(i)
    comm.barrier()
    assert torch.equal(x, torch.arange(1000, dtype=torch.float32, device="cuda"))
    assert torch.equal(y, want) and c.tolist() == [1.5, -2.0] and i.tolist() == [3, 4]
    k, n = 37, 3
    chunk = x_chunk(k, n, 1)
    xp = torch.zeros(chunk, device="cuda")
    lo, hi = upload_range(k, n, 1, 0)
    xp[lo:hi] = torch.arange(hi - lo, dtype=torch.float32, device="cuda")
    comm.allgather_x(xp, chunk)
    assert torch.equal(xp[:k * n], torch.arange(k * n, dtype=torch.float32, device="cuda"))


def test_world1_slice_spmm_matches_single_gpu(comm):
    full = spmk.DeviceCsr.generate_rmat(14, 8, SKEWS["heavy"], 3)
    s, lo, hi = comm.slice(full)
    assert (lo, hi) == (0, full.num_rows) and s.nnz == full.nnz
    x = spmk.make_dense_device(full.num_cols, 8, 99)
    y = torch.empty((s.num_rows, 8), device="cuda")
    kid = comm.spmm(s, x, y)
    assert kid == full.select(8)
    ref = full.spmm(kid, x)
    torch.cuda.synchronize()
    assert torch.equal(y, ref)


def test_bad_arguments_raise(comm):
    y = torch.zeros(10, device="cuda")
    with pytest.raises(spmk.Error):
        comm.allgather_rows(y, [5, 2], n=1)  # decreasing bounds
    with pytest.raises(spmk.Error):
        comm.broadcast(y, root=3)
