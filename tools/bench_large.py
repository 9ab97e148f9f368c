#!/usr/bin/env python3
"""BASELINE cfg4 on one B200: SpMM N=64 on R-MAT 2^24 heavy e32 seed 1
(520.8M nnz; X and Y 4.3 GB each), the rule-selected variant, L2 flushed.
Then the equal-nnz row partition for G = 2, 4, 8 (spmk_row_slices, the
multi-GPU plan): every slice is run standalone on this GPU and timed; the
slowest slice is the critical path a G-GPU run would see (no collective in
the SpMM), giving a projected speed-up t_1 / max_g t_g."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200 import selection  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--ef", type=int, default=32)
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--parts", default="2,4,8")
ap.add_argument("--kernel", default="rule", help="rule (select_kernel per matrix / slice) or tuned (fastest measured)")
args = ap.parse_args()
t0 = time.time()
full = spmk.DeviceCsr.generate_rmat(args.scale, args.ef, (0.57, 0.19, 0.19, 0.05), 1)
torch.cuda.synchronize()
gen = time.time() - t0
n = args.n
x = spmk.make_dense_device(full.num_cols, n, 0x00D5EED + n)
def choose(a):
    return selection.tuned_kernel(a, n)[0] if args.kernel == "tuned" else a.select(n)


kid = choose(full)
rec, y = selection.measure_kernel("cfg4", full, x, kid, repeats=args.reps, warmup=1)
t1 = rec.time_seconds
del y
torch.cuda.empty_cache()
M, K, nnz = full.num_rows, full.num_cols, full.nnz
byts = 4 * (M + 1) + 8 * nnz + 4 * K * n + 4 * M * n
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
out = {"workload": f"SpMM N={n} on R-MAT s{args.scale} e{args.ef} heavy seed 1", "nnz": nnz,
       "kernel_choice": args.kernel,
       "kernel": kid.name, "t1_ms": round(t1 * 1e3, 3), "gflops_1gpu": round(rec.gflops, 1),
       "roofline_frac_of_measured_hbm": round(byts / t1 / 1e9 / peak, 4), "generation_s": round(gen, 1),
       "partitions": {}}
for G in [int(g) for g in args.parts.split(",")]:
    b = full.row_slices(G)
    ts, kinds = [], []
    for g in range(G):
        s = full.slice(int(b[g]), int(b[g + 1]))
        k = choose(s)
        r, yy = selection.measure_kernel(f"slice{g}", s, x, k, repeats=args.reps, warmup=1)
        ts.append(r.time_seconds)
        kinds.append(k.name)
        del s, yy
        torch.cuda.empty_cache()
    out["partitions"][G] = {"rows": [int(b[g + 1] - b[g]) for g in range(G)], "kernels": kinds,
                            "slice_ms": [round(t * 1e3, 3) for t in ts],
                            "projected_speedup": round(t1 / max(ts), 2)}
print(json.dumps(out), flush=True)
