"""Iterative SpMV (PageRank-style, BASELINE cfg5 workload) on the device vs
the fp64 oracle: teacher-forced steps within the north-star bound, the
free-running iteration within eps/(1-alpha), graph replay bit-identical to
eager steps, residual history monotone."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2106_16064_b200 as spmk  # noqa: E402
from oracle.oracle import Csr, pagerank64, pagerank_step64  # noqa: E402
from paper_2106_16064_b200 import pagerank as prk  # noqa: E402

pytestmark = pytest.mark.gpu
ALPHA = 0.85


def host(d):
    h = d.download()
    return Csr(h.num_rows, h.num_cols, h.row_ptr, h.col_idx, h.values)


@pytest.fixture(scope="module")
def graph():
    d = spmk.DeviceCsr.generate_rmat(12, 8, (0.57, 0.19, 0.19, 0.05), 3)
    pr = prk.PageRank(d, ALPHA)
    torch.cuda.synchronize()
    return d, pr, host(d), pr.counts.cpu().numpy()


def test_column_stochastic_values(graph):
    d, pr, a, counts = graph
    assert np.array_equal(counts, np.bincount(a.col_idx, minlength=a.k))
    want = (np.float32(1.0) / counts[a.col_idx].astype(np.float32)).astype(np.float32)
    assert np.array_equal(a.val, want)
    assert pr.kid == d.select(1)


def test_teacher_forced_steps(graph, orc):
    d, pr, a, counts = graph
    pr.reset()
    for t in range(3):
        x = pr.x.cpu().numpy().reshape(-1).copy()
        pr.step()
        got = pr.x.cpu().numpy().reshape(-1).astype(np.float64)
        want, bound = pagerank_step64(orc, a, x, counts, ALPHA)
        # SpMV within 1e-5*sum|a x| (north_star), plus the fp32 rounding of the update
        assert np.all(np.abs(got - want) <= 1e-5 * bound + 2e-7 * np.abs(want)), f"step {t}"
        st = pr.state.cpu().numpy()
        assert st[1] == pytest.approx(np.abs(got - x).sum(), rel=1e-6)


def test_free_running_and_graph_replay(graph, orc):
    d, pr, a, counts = graph
    iters = 30
    x_eager, h_eager = pr.run(iters, graph=False)
    x_eager = x_eager.cpu().numpy().copy()
    h_eager = h_eager.cpu().numpy().copy()
    x_graph, h_graph = pr.run(iters, graph=True)
    assert np.array_equal(x_graph.cpu().numpy(), x_eager), "graph replay must equal eager steps"
    assert np.array_equal(h_graph.cpu().numpy(), h_eager)
    ref = pagerank64(orc, a, counts, ALPHA, iters)
    assert np.abs(x_eager.reshape(-1) - ref).sum() <= 1e-5 / (1 - ALPHA)
    assert abs(x_eager.sum() - 1.0) < 1e-4
    assert h_eager[-1] < 1e-3 * h_eager[0]  # geometric contraction (alpha^t) down to the fp32 floor


def test_distributed_driver_single_rank_matches(graph, orc):
    """The multi-GPU driver at world_size 1 (gloo-free path: 1-rank NCCL group)
    computes the same iteration as the single-GPU driver."""
    import os

    import torch.distributed as dist

    d, pr, a, counts = graph
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        d2 = spmk.DeviceCsr.generate_rmat(12, 8, (0.57, 0.19, 0.19, 0.05), 3)
        dp = prk.DistributedPageRank(d2, ALPHA)
        x, _ = dp.run(10)
        x1, _ = pr.run(10, graph=False)
        assert np.array_equal(x.cpu().numpy(), x1.cpu().numpy())
        # fused update + exchange (P2P stores into every replica; here the
        # rank's own buffer) computes the same iterates bit for bit
        d3 = spmk.DeviceCsr.generate_rmat(12, 8, (0.57, 0.19, 0.19, 0.05), 3)
        dq = prk.DistributedPageRank(d3, ALPHA, exchange="p2p")
        xq, hq = dq.run(10)
        assert np.array_equal(xq.cpu().numpy(), x1.cpu().numpy())
        dq.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kidx", [0, 2])
def test_graph_replay_row_split_hub_path(graph, kidx):
    """PageRank with a row-split kernel (what a hub-heavy slice selects) and
    most rows on the hub path: graph replay (hub kernels captured on the side
    stream) equals eager steps bit for bit."""
    d, _, a, _ = graph
    old = d.get_tuning("hub_nnz")
    d.set_tuning("hub_nnz", 32)
    try:
        pr = prk.PageRank(d, ALPHA, kernel=spmk.KernelId(kidx))
        x_eager, h_eager = pr.run(10, graph=False)
        x_eager = x_eager.cpu().numpy().copy()
        h_eager = h_eager.cpu().numpy().copy()
        x_graph, h_graph = pr.run(10, graph=True)
        assert np.array_equal(x_graph.cpu().numpy(), x_eager)
        assert np.array_equal(h_graph.cpu().numpy(), h_eager)
    finally:
        d.set_tuning("hub_nnz", old)


def test_tuned_kernel_choice(graph, orc):
    """kernel="tuned": the fastest measured variant; any variant stays within
    the north-star bound, so the free-running iteration keeps its contract."""
    d, _, a, counts = graph
    pr = prk.PageRank(d, ALPHA, kernel="tuned")
    assert set(pr.tune_times) == {k.name for k in spmk.kAllKernels}
    assert pr.tune_times[pr.kid.name] == min(pr.tune_times.values())
    x, _ = pr.run(30, graph=True)
    ref = pagerank64(orc, a, counts, ALPHA, 30)
    assert np.abs(x.cpu().numpy().reshape(-1) - ref).sum() <= 1e-5 / (1 - ALPHA)
