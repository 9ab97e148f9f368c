"""bench.py contract on the device: one JSON line with the required keys, both
plain (N=1) and under torchrun (the distributed code path: NCCL group,
equal-nnz slicing, X broadcast, max over ranks), and the reference arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"}


def run(cmd, timeout=900):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_single_gpu_line():
    d = run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-extras"])
    assert KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["matches_device_path"] is True and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["run"]["kernel"] == "seq-ws"  # the rule's pick for cfg2
    assert d["config"]["nnz_total"] == 16083729


@pytest.mark.gpu
def test_bench_torchrun_world1():
    d = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
             "--master-addr", "127.0.0.1", "--master-port", "29561", "bench.py", "--gpus", "1", "--steps", "3",
             "--warmup", "3", "--no-cpu-baseline", "--no-extras"])
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0
    # the distributed path at world size 1: library NCCL communicator, slice = whole matrix
    assert d["config"]["nnz_total"] == 16083729 and d["e2e"]["matches_device_path"] is True


@pytest.mark.gpu
@pytest.mark.slow
def test_bench_cfg4_strong_scaling_world1():
    """--workload cfg4 under torchrun (world 1): the strong-scaling code path
    (library NCCL layer, chunked X upload + all-gather in e2e) at full size."""
    d = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
             "--master-addr", "127.0.0.1", "--master-port", "29563", "bench.py", "--gpus", "1", "--steps", "2",
             "--warmup", "3", "--no-cpu-baseline", "--no-extras", "--workload", "cfg4"])
    assert d["scaling"] == "strong" and d["config"]["n"] == 64 and d["value"] > 0
    assert d["e2e"]["matches_device_path"] is True


def test_bench_reference_arm_cpu():
    """The reference arm runs on the host (no GPU needed): small config."""
    d = run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0", "--scale", "12"])
    assert d["config"]["n"] == 32 and d["config"]["nnz_total"] > 0
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0
