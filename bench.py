#!/usr/bin/env python3
"""Benchmark of the adaptive SpMV/SpMM hot path (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Workload (a "step" = one Y = A*X over the whole operand with the rule-selected
variant, exactly as spmk::spmm(select_kernel(...), A, X) computes it):
  * N=1 : BASELINE cfg2 — SpMM, X width 32, fp32, R-MAT 2^20 nodes avg degree 16
          (Graph500 skew .57/.19/.19/.05, seed 1; nnz 16,083,729), 1 B200.
  * N>1 : weak scaling of the same shape: R-MAT 2^(20+log2 N) e16 seed 1 split
          into N equal-nnz row slices, one per GPU; X (K x 32) is
          replicated once by an NCCL broadcast from rank 0 outside the timed
          region (reported separately); each GPU writes its own Y slice; no
          collective inside the timed region.
Inputs are generated on the device by the bit-exact R-MAT / make_dense
generators (tests pin them to the reference streams).

value   : GFLOP/s (2*nnz*N / t) of the timed steps, inputs resident in HBM,
          L2 flushed (256 MiB write) before every step, CUDA events on the
          launching stream, max over ranks.
e2e     : the same metric through the C-ABI host path (spmk_spmm_host_async):
          every step copies X H2D from pinned host memory, runs the kernels and
          copies Y D2H; steps alternate two streams so one step's D2H overlaps
          the next step's H2D (both PCIe directions busy).
roofline: the dominant (variant) kernel: compulsory bytes (rowPtr, colIdx, val,
          X once, Y) / its CUDA-event duration vs MEASURED_PEAKS.json hbm_gbs.
cpu_baseline: the reference's own multithreaded CPU path (oracle/_ref, the
          unmodified reference headers) on this host, same matrix and X.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV/SpMM GFLOP/s and % of HBM roofline at N=1..128, 1/2/4/8 B200; selection loss"
HEAVY = (0.57, 0.19, 0.19, 0.05)
DENSE_SEED = 0x00D5EED  # bench.hpp:112


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=32, help="X width (cfg2: 32)")
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel", default="auto", help="auto (rule) or par-rs/par-ws/seq-rs/seq-ws")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


# --------------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's own CPU implementation (unmodified headers via
    oracle/_ref), rule-selected variant, on the same config; rank 0 only."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    from oracle.oracle import Oracle, load_ref

    ref = load_ref()
    kind = "reference" if ref is not None else "port"
    scale = args.scale + int(round(math.log2(max(args.gpus, 1))))
    n = args.n
    t0 = time.time()
    if ref is not None:
        a = ref.generate_rmat(scale, args.edge_factor, HEAVY, 1)
        x = ref.make_dense(a.k, n, DENSE_SEED + n)
        h = ref.handle(a)
        feats = h.extract_features()
        kidx = ref.select_kernel(feats[0], feats[2], n)
        cores = ref.hardware_concurrency()

        def step():
            return h.time_spmm(kidx, x, repeats=1, warmup=0, worker_count=0)
    else:
        orc = Oracle()
        a = orc.generate_rmat(scale, args.edge_factor, HEAVY, 1)
        x = orc.make_dense(a.k, n, DENSE_SEED + n)
        feats = orc.extract_features(a)
        kidx = orc.select_kernel(feats[0], feats[2], n)
        cores = 1

        def step():
            t = time.perf_counter()
            orc.spmm(a, kidx, x)
            return time.perf_counter() - t
    gen_s = time.time() - t0
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    flops = 2.0 * a.nnz * n
    val = flops * args.steps / total / 1e9
    names = ("par-rs", "par-ws", "seq-rs", "seq-ws")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"R-MAT s{scale} e{args.edge_factor} heavy seed 1, SpMM N={n} fp32, whole matrix "
                               f"on the host CPU", "kernel": names[kidx], "nnz": int(a.nnz),
                   "parallelism": f"{cores} host threads (reference ThreadPool)"},
        "cpu_baseline": {"value": round(val, 3), "unit": "GFLOP/s", "cores": int(cores), "kind": kind,
                         "sample": f"{args.steps} timed calls of spmm({names[kidx]}) on the full matrix "
                                   f"after {args.warmup} warm-up calls (Y allocation included, bench.hpp:65-98)"},
        "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "input_generation_s": round(gen_s, 2),
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2106_16064_b200 as spmk

    ws, rank, local = dist_env()
    G = max(ws, 1)
    # torchrun (any world size, including 1) runs the distributed code path:
    # NCCL process group, equal-nnz slicing, X broadcast, max-over-ranks.
    use_dist = "WORLD_SIZE" in os.environ
    if args.gpus != G and use_dist:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if use_dist:
        dist.init_process_group("nccl", device_id=dev)

    n = args.n
    scale = args.scale + int(round(math.log2(G)))
    assert 1 << (scale - args.scale) == G, "--gpus must be a power of two"
    t0 = time.time()
    full = spmk.DeviceCsr.generate_rmat(scale, args.edge_factor, HEAVY, 1, device=local)
    if use_dist:
        bounds = full.row_slices(G)
        a = full.slice(int(bounds[rank]), int(bounds[rank + 1]), device=local)
        del full
    else:
        bounds = np.array([0, full.num_rows])
        a = full
    K = a.num_cols
    # X replicated once: generated on rank 0, NCCL broadcast (outside timing)
    x = torch.empty((K, n), dtype=torch.float32, device=dev)
    bcast_ms = 0.0
    if rank == 0:
        x.copy_(spmk.make_dense_device(K, n, DENSE_SEED + n, device=dev))
    if use_dist:
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dist.broadcast(x, src=0)
        e1.record()
        torch.cuda.synchronize()
        bcast_ms = e0.elapsed_time(e1)
    y = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
    kid = a.select(n) if args.kernel == "auto" else spmk.parse_kernel(args.kernel)
    gen_s = time.time() - t0
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def one_step():
        a.spmm(kid, x, y, stream=stream)

    for _ in range(args.warmup):
        flush.zero_()
        one_step()
    spmk.timing_enable(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    main_ms = []
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = spmk.launch_count()
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()  # L2 flush, outside the timed interval
            ev[i][0].record(stream)
            one_step()
            ev[i][1].record(stream)
            main_ms.append(spmk.timing_last()[0])
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    launches = spmk.launch_count() - launches0
    spmk.timing_enable(False)
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    dev_ms = sum(e0.elapsed_time(e1) for e0, e1 in ev)
    t_local = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    t_max_ms = float(t_local.item())
    nnz_all = torch.tensor([a.nnz], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(nnz_all)
    flops_step = 2.0 * float(nnz_all.item()) * n
    value = flops_step * args.steps / (t_max_ms * 1e-3) / 1e9

    # ---------------- e2e through the C-ABI host path (pinned H2D/D2H per step)
    # spmk_spmm_host_async: every step enqueues H2D(X) -> kernels -> D2H(Y) on
    # one of two streams (the handle rotates two device staging slots), so one
    # step's D2H overlaps the next step's H2D on the two PCIe directions.
    hx = [torch.empty((K, n), dtype=torch.float32, pin_memory=True) for _ in range(2)]
    for h in hx:
        h.copy_(x.cpu())
    hy = [torch.empty((a.num_rows, n), dtype=torch.float32, pin_memory=True) for _ in range(2)]
    hxn, hyn = [h.numpy() for h in hx], [h.numpy() for h in hy]
    streams = [stream, torch.cuda.Stream(dev)]
    for i in range(2):
        a.spmm_host_async(kid, hxn[i], hyn[i], streams[i].cuda_stream)
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    streams[1].wait_event(e0)
    for i in range(args.steps):
        a.spmm_host_async(kid, hxn[i % 2], hyn[i % 2], streams[i % 2].cuda_stream)
    streams[0].wait_stream(streams[1])
    e1.record(streams[0])
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    # the synchronous call shape (spmk_spmm_host: one call, one sync) for reference
    sync_ms = 0.0
    for _ in range(3):
        t0 = time.perf_counter()
        a.spmm_host(kid, hxn[0], stream=stream.cuda_stream, out=hyn[0])
        sync_ms += (time.perf_counter() - t0) * 1e3
    t_e2e = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_value = flops_step * args.steps / (float(t_e2e.item()) * 1e-3) / 1e9
    ok_e2e = bool(torch.equal(torch.from_numpy(hyn[0].copy()).to(dev), y))

    # ---------------- roofline of the dominant kernel (rank-local)
    M, nnz = a.num_rows, a.nnz
    m_ne = M - a.empty_rows
    alg_bytes = 4 * (M + 1) + 8 * nnz + 4 * K * n + 4 * m_ne * n  # zero-fill of empty rows is a separate kernel
    main_avg_ms = statistics.mean(main_ms)
    achieved = alg_bytes / (main_avg_ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        key = f"{spmk.kernel_name(kid)}_n{n}_s{scale}"
        traffic = tr.get(key)
    except Exception:
        pass
    step_bytes = 4 * (M + 1) + 8 * nnz + 4 * K * n + 4 * M * n
    result = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": G,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_max_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (device R-MAT/make_dense generators, bit-identical to rmat.hpp/corpus.hpp)",
        "config": {
            "workload": ("cfg2: SpMM N=32 fp32 on R-MAT 2^20 power-law (avg degree 16), 1 B200" if G == 1 else
                         f"weak-scaled cfg2 shape: R-MAT 2^{scale} e{args.edge_factor}, {G} equal-nnz row "
                         f"slices (one per GPU), X broadcast once over NCCL"),
            "matrix": f"R-MAT s{scale} e{args.edge_factor} skew {HEAVY} seed 1", "nnz_total": int(nnz_all.item()),
            "n": n, "kernel": spmk.kernel_name(kid), "selected_by": "select_kernel" if args.kernel == "auto" else "forced",
            "l2": "flushed (256 MiB write) before every timed step",
            "parallelism": "single GPU" if G == 1 else f"row-partition x{G} (equal nnz), no collective in timed region",
            "x_broadcast_ms": round(bcast_ms, 3), "input_generation_s": round(gen_s, 2),
            "effective_GBps_compulsory": round(step_bytes * args.steps / (t_max_ms * 1e-3) / 1e9 * G, 1),
            "wall_s_timed_loop": round(wall, 4),
        },
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": f"{spmk.kernel_name(kid)} (dominant launch, avg {main_avg_ms * 1e3:.1f} us)",
                     "algorithmic_bytes_per_launch": int(alg_bytes)},
        "e2e": {"value": round(e2e_value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(K * n * 4),
                "d2h_bytes_per_step": int(M * n * 4),
                "path": "spmk_spmm_host_async (C ABI), pinned host X/Y, 2 streams x 2 staging slots",
                "sync_call_ms": round(sync_ms / 3, 3), "matches_device_path": ok_e2e},
        "gpu_launches": int(launches),
    }
    clocks = clk.summary()
    result["clocks"] = clocks
    if rank == 0 and G == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(a, x, kid, n)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def cpu_baseline(a, x, kid, n):
    """The reference's multithreaded CPU spmm on the same matrix/X (bounded
    sample: 2 warm-up + median of 5 calls of the full matrix)."""
    import numpy as np

    from oracle.oracle import Csr, Oracle, load_ref

    h = a.download()
    xh = x.cpu().numpy()
    ref = load_ref()
    if ref is not None:
        rh = ref.handle(Csr(h.num_rows, h.num_cols, h.row_ptr, h.col_idx, h.values))
        sec = rh.time_spmm(kid.index, xh, repeats=5, warmup=2, worker_count=0)
        cores, kind = ref.hardware_concurrency(), "reference"
        sample = "full cfg2 matrix, reference spmm() median of 5 after 2 warm-up (bench.hpp:65-98)"
    else:
        orc = Oracle()
        t0 = time.perf_counter()
        orc.spmm(Csr(h.num_rows, h.num_cols, h.row_ptr, h.col_idx, h.values), kid.index, xh)
        sec = time.perf_counter() - t0
        cores, kind = 1, "port"
        sample = "full cfg2 matrix, C oracle port (1 thread), one call"
    return {"value": round(2.0 * a.nnz * n / sec / 1e9, 3), "unit": "GFLOP/s", "cores": int(cores),
            "kind": kind, "sample": sample, "seconds_per_call": round(sec, 4)}


if __name__ == "__main__":
    main()
