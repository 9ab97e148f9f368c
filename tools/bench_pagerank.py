#!/usr/bin/env python3
"""BASELINE cfg5 workload on one B200: PageRank-style iterative SpMV, 50
iterations on R-MAT 2^25 heavy e16 seed 1 (528.7M nnz), graph-captured.
Reports per-iteration time, GFLOP/s (2*nnz per iteration) and the HBM
roofline fraction of the compulsory bytes per iteration."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200 import pagerank as prk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=25)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--l2", type=float, default=0.0, help="MB of x (its hot low-index prefix) pinned in L2")
ap.add_argument("--kernel", default="rule", help="rule | tuned | par-rs | par-ws | seq-rs | seq-ws")
ap.add_argument("--lib", default=None, help="dev: another build of libspmk_b200.so")
args = ap.parse_args()
if args.lib:
    spmk.spmk.load_library(args.lib)
t0 = time.time()
d = spmk.DeviceCsr.generate_rmat(args.scale, args.ef, (0.57, 0.19, 0.19, 0.05), 1)
torch.cuda.synchronize()
gen = time.time() - t0
kern = None if args.kernel == "rule" else ("tuned" if args.kernel == "tuned" else spmk.parse_kernel(args.kernel))
pr = prk.PageRank(d, 0.85, kernel=kern, l2_persist_bytes=int(args.l2 * (1 << 20)))
pr.capture(args.iters)
ts = []
for _ in range(args.reps):
    pr.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pr.graph.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e-3)
t = sorted(ts)[len(ts) // 2]
per = t / args.iters
M, nnz = d.num_rows, d.nnz
byts = 4 * (M + 1) + 8 * nnz + 4 * M + 4 * M  # rowPtr, col+val, x, y (per iteration)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
hist = pr.hist.cpu().numpy()
print(json.dumps({
    "workload": f"cfg5 iterative SpMV (PageRank, alpha 0.85) on R-MAT s{args.scale} e{args.ef} heavy seed 1, 1 B200",
    "nnz": nnz, "kernel": pr.kid.name, "kernel_choice": args.kernel, "l2_persist_MB": args.l2, "iters": args.iters, "ms_total": round(t * 1e3, 3),
    "us_per_iter": round(per * 1e6, 1), "gflops": round(2.0 * nnz / per / 1e9, 1),
    "GBps_compulsory": round(byts / per / 1e9, 1), "roofline_frac_of_measured_hbm": round(byts / per / 1e9 / peak, 4),
    "l1_residual_first_last": [float(hist[0]), float(hist[-1])], "generation_s": round(gen, 1)}))
