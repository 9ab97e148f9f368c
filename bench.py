#!/usr/bin/env python3
"""Benchmark of the adaptive SpMV/SpMM hot path (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload cfg2|cfg4]

A "step" is one Y = A*X over the whole operand with the rule-selected variant,
exactly as spmk::spmm(select_kernel(...), A, X) computes it.  Workloads
(`--workload auto`, the default, picks cfg2 on one GPU and cfg4 on several):
  * cfg2 (BASELINE configs[1], "1 B200"): SpMM, X width 32, fp32, R-MAT 2^20
    nodes avg degree 16 (Graph500 skew .57/.19/.19/.05, seed 1; 16,083,729
    nonzeros).  The N=1 headline.
  * cfg4 (BASELINE configs[3]): SpMM N=64 on R-MAT 2^24 avg degree 32
    (520.8M nonzeros), STRONG scaling: the fixed matrix is cut into N
    equal-nnz row slices, one per GPU, through the library's
    multi-GPU C ABI (spmk_mg_*: NCCL over NVLink); X (4.3 GB) is replicated
    once by an NCCL broadcast from rank 0 outside the timed region
    (x_broadcast_ms); each GPU writes its own Y slice with its slice's rule;
    no collective inside the timed region.  On one GPU the cfg2 line carries
    the cfg4 single-GPU time as `strong_scaling` (the base of the series).
Inputs are generated on the device by the bit-exact R-MAT / make_dense
generators (tests pin them to the reference streams, full size included).

value   : GFLOP/s (2*nnz*N / t) of the timed steps, whole job, inputs resident
          in HBM, L2 flushed (256 MiB write) before every step, CUDA events on
          the launching stream, max over ranks.
e2e     : the same metric with host operands, host<->device copies inside the
          timed region.  1 GPU: spmk_spmm_host_async (C ABI) — every step copies
          X H2D from pinned memory, runs the kernels, copies Y D2H, on two
          alternating streams.  N GPUs: every rank uploads 1/N of the host X
          over its own PCIe link, spmk_mg_allgather_x assembles the replica
          over NVLink, the slice SpMM runs, the rank's Y slice goes D2H.
roofline: the dominant (variant) kernel: compulsory bytes (rowPtr, colIdx, val,
          X once, Y) / its CUDA-event duration vs MEASURED_PEAKS.json hbm_gbs.
cpu_baseline / --impl reference: the reference's own multithreaded CPU path
          (oracle/_ref, the unmodified reference headers) on this host.
selection_loss (1 GPU): a reduced cfg3 sweep (uniform / banded / heavy at
          2^18 and 2^20, N = 1..128, all four kernels timed) summarised with
          the reference's protocol (bench.hpp:136-196).
"""
from __future__ import annotations

import argparse
import json
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
WORKLOADS = {
    "cfg2": dict(scale=20, ef=16, n=32,
                 label="cfg2: SpMM N=32 fp32 on R-MAT 2^20 power-law (avg degree 16), 1 B200"),
    "cfg4": dict(scale=24, ef=32, n=64,
                 label="cfg4: SpMM N=64 fp32 on R-MAT 2^24 (avg degree 32), equal-nnz row slices over the GPUs "
                       "(strong scaling), X broadcast once over NVLink"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "cfg2", "cfg4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip strong_scaling / selection_loss / call shapes")
    ap.add_argument("--kernel", default="auto", help="auto (rule) or par-rs/par-ws/seq-rs/seq-ws")
    ap.add_argument("--scale", type=int, default=None, help="override the workload's R-MAT scale (tests)")
    return ap.parse_args()


def workload_of(args, G):
    name = args.workload if args.workload != "auto" else ("cfg2" if G == 1 else "cfg4")
    wl = dict(WORKLOADS[name])
    if args.scale is not None and args.scale != wl["scale"]:
        wl["scale"] = args.scale
        wl["label"] = f"{name} shape at R-MAT 2^{args.scale} (reduced: test run)"
    return name, wl


def common_config(wl, nnz_total):
    """The `config` both arms print (identical keys and values)."""
    return {"workload": wl["label"], "matrix": f"R-MAT s{wl['scale']} e{wl['ef']} skew {HEAVY} seed 1",
            "n": wl["n"], "nnz_total": int(nnz_total), "x": f"make_dense(K, {wl['n']}, 0x00D5EED + {wl['n']})",
            "selected_by": "select_kernel (reference thresholds)"}


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
    oracle/_ref), rule-selected variant, on the same workload; rank 0 only.
    cfg2: every step is the whole matrix.  cfg4 (10 s per whole-matrix call
    on the host): every step is a bounded sample — 1/16 of the rows drawn at
    random (default_rng(0)) as one CSR (~1/16 of the work), with the kernel the rule picks for
    the whole matrix; the value is the sample's GFLOP/s."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    from oracle.oracle import Csr, Oracle, load_ref

    G = max(ws, args.gpus, 1)
    name, wl = workload_of(args, G)
    ref = load_ref()
    kind = "reference" if ref is not None else "port"
    n = wl["n"]
    t0 = time.time()
    gen = ref if ref is not None else Oracle()
    a = gen.generate_rmat(wl["scale"], wl["ef"], HEAVY, 1)
    x = gen.make_dense(a.k, n, DENSE_SEED + n)
    nnz_total = a.nnz
    if ref is not None:
        feats = ref.handle(a).extract_features() if name == "cfg2" else None
    if name == "cfg2":
        s, sample = a, "the whole matrix"
    else:
        rows = np.sort(np.random.default_rng(0).choice(a.m, size=a.m // 16, replace=False))
        lens = np.diff(a.row_ptr)[rows]
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        idx = np.repeat(a.row_ptr[rows] - rp[:-1], lens) + np.arange(int(rp[-1]), dtype=np.int64)
        s = Csr(len(rows), a.k, rp, a.col_idx[idx], a.val[idx])
        sample = f"1/16 of the rows drawn at random ({s.nnz} of {a.nnz} nonzeros) as one CSR"
    if ref is not None:
        if feats is None:
            feats = ref.handle(a).extract_features()
        kidx = ref.select_kernel(feats[0], feats[2], n)
        h = ref.handle(s)
        cores = ref.hardware_concurrency()

        def step():
            return h.time_spmm(kidx, x, repeats=1, warmup=0, worker_count=0)
    else:
        orc = gen
        feats = orc.extract_features(a)
        kidx = orc.select_kernel(feats[0], feats[2], n)
        cores = 1

        def step():
            t = time.perf_counter()
            orc.spmm(s, kidx, x)
            return time.perf_counter() - t
    del a
    gen_s = time.time() - t0
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    val = 2.0 * s.nnz * n * args.steps / total / 1e9
    names = ("par-rs", "par-ws", "seq-rs", "seq-ws")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if name == "cfg4" else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generate_rmat / make_dense)",
        "config": common_config(wl, nnz_total),
        "run": {"kernel": names[kidx], "parallelism": f"{cores} host threads (reference ThreadPool)",
                "sample": sample, "input_generation_s": round(gen_s, 2)},
        "cpu_baseline": {"value": round(val, 3), "unit": "GFLOP/s", "cores": int(cores), "kind": kind,
                         "sample": f"{args.steps} timed calls of spmm({names[kidx]}) on {sample} after "
                                   f"{args.warmup} warm-up calls (Y allocation included, bench.hpp:65-98)"},
        "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- our arm
class Ranks:
    """Max/sum over ranks through the library's NCCL layer (or identity)."""

    def __init__(self, comm, G, rank, dev):
        self.comm, self.G, self.rank, self.dev = comm, G, rank, dev

    def gather(self, v, dtype="f64"):
        import torch

        if self.comm is None:
            return [v]
        t = torch.zeros(self.G, dtype=torch.float64 if dtype == "f64" else torch.int32, device=self.dev)
        t[self.rank] = v
        self.comm.allreduce(t)
        torch.cuda.synchronize()
        return t.tolist()

    def barrier(self):
        if self.comm is not None:
            self.comm.barrier()


def run_workload(wl, args, ranks: Ranks, local: int, steps: int, e2e: bool, roofline: bool):
    import torch

    import paper_2106_16064_b200 as spmk
    from paper_2106_16064_b200.multigpu import upload_range, x_chunk

    comm, G, rank = ranks.comm, ranks.G, ranks.rank
    dev = torch.device("cuda", local)
    n = wl["n"]
    t0 = time.time()
    full = spmk.DeviceCsr.generate_rmat(wl["scale"], wl["ef"], HEAVY, 1, device=local)
    nnz_total = full.nnz
    if comm is not None:
        a, row0, row1 = comm.slice(full)
        del full
    else:
        a, row0, row1 = full, 0, full.num_rows
    torch.cuda.empty_cache()
    K = a.num_cols
    # X replicated once: generated on rank 0, broadcast over NVLink (outside timing)
    x = torch.empty((K, n), dtype=torch.float32, device=dev)
    bcast_ms = 0.0
    if rank == 0:
        x.copy_(spmk.make_dense_device(K, n, DENSE_SEED + n, device=dev))
    if comm is not None:
        torch.cuda.synchronize()
        ranks.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        comm.broadcast(x, root=0)
        e1.record()
        torch.cuda.synchronize()
        bcast_ms = e0.elapsed_time(e1)
    y = torch.empty((a.num_rows, n), dtype=torch.float32, device=dev)
    kid = a.select(n) if args.kernel == "auto" else spmk.parse_kernel(args.kernel)
    gen_s = time.time() - t0
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def one_step():
        if a.num_rows:
            a.spmm(kid, x, y, stream=stream)

    for _ in range(args.warmup):
        flush.zero_()
        one_step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    ranks.barrier()
    torch.cuda.synchronize()
    launches0 = spmk.launch_count()
    # The timed steps: no host sync and no library instrumentation inside the
    # loop (a per-step sync let the host's enqueue latency leak into the device
    # interval: +10 us per cfg2 step, measured); the host runs ahead of the device.
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for i in range(steps):
            flush.zero_()  # L2 flush, outside the timed interval
            ev[i][0].record(stream)
            one_step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    launches = spmk.launch_count() - launches0
    # The dominant kernel's duration for the roofline: the same steps again with
    # the library's per-call events on the launching stream (spmk_timing_summary)
    main_ms = []
    if a.num_rows:
        spmk.timing_enable(True)
        for i in range(steps):
            flush.zero_()
            one_step()
        m_tot, _, m_calls = spmk.timing_summary()
        spmk.timing_enable(False)
        main_ms = [m_tot / max(m_calls, 1)]
    ranks.barrier()
    dev_ms = sum(e0.elapsed_time(e1) for e0, e1 in ev)
    per_rank_ms = ranks.gather(dev_ms)
    t_max_ms = max(per_rank_ms)
    flops_step = 2.0 * nnz_total * n
    value = flops_step * steps / (t_max_ms * 1e-3) / 1e9
    kernels = [spmk.kernel_name(spmk.KernelId(int(k))) for k in ranks.gather(kid.index, "i32")]
    out = {"value": value, "ms_per_step": t_max_ms / steps, "nnz_total": nnz_total, "kernels": kernels,
           "per_rank_ms_per_step": [round(v / steps, 4) for v in per_rank_ms], "x_broadcast_ms": bcast_ms,
           "input_generation_s": gen_s, "wall_s_timed_loop": wall, "launches": launches,
           "clocks": clk.summary(), "kid": kid, "a": a, "x": x, "y": y, "rows": (row0, row1)}

    if e2e:
        if comm is None:
            # spmk_spmm_host_async: H2D(X) -> kernels -> D2H(Y) per step on one of
            # two streams (two device staging slots), so one step's D2H overlaps
            # the next step's H2D on the two PCIe directions.
            hx = [torch.empty((K, n), dtype=torch.float32, pin_memory=True) for _ in range(2)]
            for h in hx:
                h.copy_(x.cpu())
            hy = [torch.empty((a.num_rows, n), dtype=torch.float32, pin_memory=True) for _ in range(2)]
            hxn, hyn = [h.numpy() for h in hx], [h.numpy() for h in hy]
            streams = [stream, torch.cuda.Stream(dev)]
            for i in range(2):
                a.spmm_host_async(kid, hxn[i], hyn[i], streams[i].cuda_stream)
            torch.cuda.synchronize()
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(streams[0])
            streams[1].wait_event(e0)
            for i in range(steps):
                a.spmm_host_async(kid, hxn[i % 2], hyn[i % 2], streams[i % 2].cuda_stream)
            streams[0].wait_stream(streams[1])
            e1.record(streams[0])
            torch.cuda.synchronize()
            e2e_ms = e0.elapsed_time(e1)
            ok = bool(torch.equal(torch.from_numpy(hyn[(steps - 1) % 2].copy()).to(dev), y))
            h2d, d2h = K * n * 4, a.num_rows * n * 4
            path = "spmk_spmm_host_async (C ABI), pinned host X/Y, 2 streams x 2 staging slots"
        else:
            # every rank uploads its 1/G of the host X (own PCIe link), NVLink
            # all-gather assembles the replica, slice SpMM, Y slice D2H
            chunk = x_chunk(K, n, G)
            lo, hi = upload_range(K, n, G, rank)
            hx = torch.empty(K * n, dtype=torch.float32, pin_memory=True)
            hx.copy_(x.view(-1).cpu())
            hy = torch.empty((a.num_rows, n), dtype=torch.float32, pin_memory=True)
            xp = torch.empty(chunk * G, dtype=torch.float32, device=dev)
            xv = xp[: K * n].view(K, n)

            def e2e_step():
                xp[lo:hi].copy_(hx[lo:hi], non_blocking=True)
                comm.allgather_x(xp, chunk)
                if a.num_rows:
                    a.spmm(kid, xv, y, stream=stream)
                hy.copy_(y, non_blocking=True)

            e2e_step()
            torch.cuda.synchronize()
            ranks.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                e2e_step()
            e1.record(stream)
            torch.cuda.synchronize()
            e2e_ms = e0.elapsed_time(e1)
            ok = bool(torch.equal(hy.to(dev), y))
            h2d, d2h = K * n * 4, int(sum(ranks.gather(a.num_rows))) * n * 4  # whole job, all ranks
            path = ("per rank: H2D of 1/N of the pinned host X + spmk_mg_allgather_x (NVLink) + slice spmm "
                    "+ D2H of the rank's Y slice")
        e2e_max = max(ranks.gather(e2e_ms))
        out["e2e"] = {"value": round(flops_step * steps / (e2e_max * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                      "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "path": path,
                      "matches_device_path": ok}

    if roofline and a.num_rows:
        M, nnz = a.num_rows, a.nnz
        m_ne = M - a.empty_rows
        path = a.spmm_path(kid, n)
        # lane-per-job seq-ws: the sweep writes every row of Y (empty rows too)
        # and the timed region is sweep + fold pass; otherwise the empty-row
        # zero-fill is a separate side-stream kernel outside the timed region
        y_rows = M if path == "sell" else m_ne
        alg_bytes = 4 * (M + 1) + 8 * nnz + 4 * K * n + 4 * y_rows * n
        main_avg_ms = statistics.mean(main_ms)
        achieved = alg_bytes / (main_avg_ms * 1e-3) / 1e9
        peak, peak_kind = peaks()
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic = json.load(f).get(f"{spmk.kernel_name(kid)}_n{n}_s{wl['scale']}")
        except Exception:
            pass
        out["roofline"] = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                           "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                           "kernel": f"{spmk.kernel_name(kid)} ("
                                     + ("lane-per-job sweep + fold pass" if path == "sell" else "dominant launch")
                                     + f", avg {main_avg_ms * 1e3:.1f} us"
                                     + (f", rank {rank}" if G > 1 else "") + ")",
                           "algorithmic_bytes_per_launch": int(alg_bytes),
                           "l2_gather_bytes_per_launch": int(nnz * ((4 * n + 127) // 128) * 128),
                           # vs the measured ceiling of 128-B row gathers with R-MAT column
                           # statistics (11.4 TB/s, profiles/r02e_microbench_gather.txt)
                           "l2_gather_frac": round(nnz * ((4 * n + 127) // 128) * 128 / (main_avg_ms * 1e-3)
                                                   / 11.4e12, 4)}
    return out


def selection_loss_summary():
    """Reduced cfg3 sweep: uniform / banded / heavy at 2^18 and 2^20, N in
    {1, 2, 4, ..., 128}, the four kernels timed (median of 3 after 1 warm-up,
    L2 flushed), the rule's choice with the reference thresholds and with the
    B200-calibrated ones; loss per bench.hpp:136-196."""
    import torch

    from paper_2106_16064_b200 import inputs
    from paper_2106_16064_b200.selection import (B200_THRESHOLDS, BenchRecord, SelectorThresholds,
                                                 kAllKernels, make_dense_device, mean_per_n_loss,
                                                 measure_kernel, min_single_kernel_loss,
                                                 summarize_selection_loss)

    t0 = time.time()
    recs = {"reference": [], "b200": []}
    ns = (1, 2, 4, 8, 16, 32, 64, 128)
    per_n = {}
    peak, _ = peaks()
    for name, a in inputs.sweep_corpus(scales=(18, 20)):
        for n in ns:
            x = make_dense_device(a.num_cols, n, DENSE_SEED + n)
            cell = []
            for kid in kAllKernels:
                rec, y = measure_kernel(name, a, x, kid, repeats=3, warmup=1)
                cell.append(rec)
                del y
            for key, t in (("reference", SelectorThresholds()), ("b200", B200_THRESHOLDS)):
                chosen = a.select(n, t)
                recs[key] += cell + [BenchRecord(**{**cell[chosen.index].__dict__, "selected_by_rule": True})]
            if name == "rmat-heavy-s20-e16":  # the cfg2 matrix: the metric's "at N = 1..128" row
                chosen = a.select(n)
                r = cell[chosen.index]
                comp = 4 * (a.num_rows + 1) + 8 * a.nnz + 4 * a.num_cols * n + 4 * a.num_rows * n
                per_n[str(n)] = {"kernel": chosen.name, "gflops": round(r.gflops, 1),
                                 "us": round(r.time_seconds * 1e6, 1),
                                 "roofline_frac": round(comp / r.time_seconds / 1e9 / peak, 4)}
            del x
        del a
        torch.cuda.empty_cache()
    out = {}
    for key, r in recs.items():
        s = summarize_selection_loss(r)
        out[key] = {"mean_per_n_loss": round(mean_per_n_loss(s), 4),
                    "per_n_loss": {str(k): round(v, 4) for k, v in s.per_n_loss.items()},
                    "best_single_kernel_loss": round(min_single_kernel_loss(s), 4)}
    out["cfg2_matrix_per_n"] = {"matrix": "R-MAT s20 e16 heavy seed 1 (cfg2)", "selected_by": "select_kernel (reference thresholds)",
                                "roofline": "compulsory bytes 4(M+1) + 8 nnz + 4 K N + 4 M N over measured HBM, whole call",
                                "n": per_n}
    out["cells"] = len(recs["reference"]) // 5
    out["sweep"] = "uniform/banded/heavy x 2^18, 2^20 x N=1..128 (reduced cfg3), median of 3, L2 flushed"
    out["thresholds"] = {"reference": "SelectorThresholds{} (selector.hpp:16-22)",
                         "b200": "calibrate_thresholds on the full cfg3 sweep (t_parallel_avg 16, profiles/r02f_sweep_summary.json)"}
    out["seconds"] = round(time.time() - t0, 1)
    return out


def call_shapes(a, x, kid):
    """The reference's value-returning call shape spmm(id, CsrMatrix,
    DenseMatrix) through spmk_spmm_csr_host (create + upload + validate +
    spmm + download + destroy), and the handle creation alone."""
    import paper_2106_16064_b200 as spmk

    h = a.download()
    xh = x.cpu().numpy()
    t0 = time.perf_counter()
    y1 = spmk.spmm(kid, h, xh)
    first = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    spmk.spmm(kid, h, xh)
    second = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    d = spmk.DeviceCsr.from_host(h)
    create = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    d.select(x.shape[1])
    sel = (time.perf_counter() - t0) * 1e3
    d.close()
    return {"value_returning_call_ms": {"first": round(first, 2), "second": round(second, 2)},
            "handle_create_ms": round(create, 2), "features_and_rule_ms": round(sel, 2),
            "value_returning_gflops": round(2.0 * a.nnz * x.shape[1] / (second * 1e-3) / 1e9, 2),
            "path": "spmk_spmm_csr_host (C ABI): host int64 CSR + host X in, host Y out", "y_rows": int(y1.shape[0])}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2106_16064_b200 as spmk
    from paper_2106_16064_b200.multigpu import Communicator

    ws, rank, local = dist_env()
    G = max(ws, 1)
    use_dist = "WORLD_SIZE" in os.environ
    if args.gpus != G and use_dist:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    torch.cuda.set_device(local)
    comm = None
    if use_dist:
        # torch.distributed (gloo, host) only ships NCCL's unique id; every
        # device collective below is the library's (spmk_mg_*)
        dist.init_process_group("gloo")
        comm = Communicator.from_torch_distributed(device=local)
    ranks = Ranks(comm, G, rank, torch.device("cuda", local))
    name, wl = workload_of(args, G)
    r = run_workload(wl, args, ranks, local, args.steps, e2e=True, roofline=True)
    n = wl["n"]
    result = {
        "metric": METRIC, "value": round(r["value"], 3), "unit": "GFLOP/s", "n_gpus": G,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["ms_per_step"], 4),
        "higher_is_better": True, "scaling": "strong" if name == "cfg4" else "weak", "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (device R-MAT/make_dense generators, bit-identical to rmat.hpp/corpus.hpp)",
        "config": common_config(wl, r["nnz_total"]),
        "run": {"kernel": r["kernels"][0] if G == 1 else r["kernels"],
                "parallelism": "single GPU" if G == 1 else
                f"{G} equal-nnz row slices, one per GPU (spmk_mg_*, NCCL); no collective in the timed region",
                "per_rank_ms_per_step": r["per_rank_ms_per_step"],
                "x_broadcast_ms": round(r["x_broadcast_ms"], 3),
                "l2": "flushed (256 MiB write) before every timed step",
                "input_generation_s": round(r["input_generation_s"], 2),
                "effective_GBps_compulsory": None, "wall_s_timed_loop": round(r["wall_s_timed_loop"], 4)},
        "roofline": r.get("roofline"),
        "e2e": r["e2e"],
        "gpu_launches": int(r["launches"]),
        "clocks": r["clocks"],
    }
    a, x = r["a"], r["x"]
    K, M = a.num_cols, a.num_rows
    if G == 1:
        step_bytes = 4 * (M + 1) + 8 * a.nnz + 4 * K * n + 4 * M * n
        result["run"]["effective_GBps_compulsory"] = round(step_bytes / (r["ms_per_step"] * 1e-3) / 1e9, 1)
    # the reference's call shape first: host-side copies, timed before the
    # CPU baseline loads the reference library and its worker threads
    if rank == 0 and G == 1 and not args.no_extras:
        result["call_shapes"] = call_shapes(a, x, r["kid"]) if name == "cfg2" else None
    if rank == 0 and G == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(a, x, r["kid"], n, name)
    del r, a, x
    torch.cuda.empty_cache()
    if G == 1 and name == "cfg2" and not args.no_extras:
        # the strong-scaling series' base: cfg4 on this one GPU, same method
        c4 = run_workload(WORKLOADS["cfg4"], args, ranks, local, min(args.steps, 10), e2e=False, roofline=True)
        result["strong_scaling"] = {
            "workload": WORKLOADS["cfg4"]["label"], "n_gpus": 1, "value": round(c4["value"], 3),
            "unit": "GFLOP/s", "ms_per_step": round(c4["ms_per_step"], 4), "kernel": c4["kernels"][0],
            "steps": min(args.steps, 10), "roofline_frac": c4["roofline"]["frac"],
            "note": "bench.py --gpus N (torchrun) reports cfg4 at N GPUs as its top-level value"}
        del c4
        torch.cuda.empty_cache()
        result["selection_loss"] = selection_loss_summary()
    if rank == 0:
        print(json.dumps(result), flush=True)
    if comm is not None:
        comm.close()
        dist.destroy_process_group()


def cpu_baseline(a, x, kid, n, name):
    """The reference's multithreaded CPU spmm on the same matrix/X (bounded
    sample: 2 warm-up + median of 5 calls of the full matrix)."""
    from oracle.oracle import Csr, Oracle, load_ref

    h = a.download()
    xh = x.cpu().numpy()
    ref = load_ref()
    if ref is not None:
        rh = ref.handle(Csr(h.num_rows, h.num_cols, h.row_ptr, h.col_idx, h.values))
        sec = rh.time_spmm(kid.index, xh, repeats=5, warmup=2, worker_count=0)
        cores, kind = ref.hardware_concurrency(), "reference"
        sample = f"full {name} matrix, reference spmm() median of 5 after 2 warm-up (bench.hpp:65-98)"
    else:
        orc = Oracle()
        t0 = time.perf_counter()
        orc.spmm(Csr(h.num_rows, h.num_cols, h.row_ptr, h.col_idx, h.values), kid.index, xh)
        sec = time.perf_counter() - t0
        cores, kind = 1, "port"
        sample = f"full {name} matrix, C oracle port (1 thread), one call"
    return {"value": round(2.0 * a.nnz * n / sec / 1e9, 3), "unit": "GFLOP/s", "cores": int(cores),
            "kind": kind, "sample": sample, "seconds_per_call": round(sec, 4)}


if __name__ == "__main__":
    main()
