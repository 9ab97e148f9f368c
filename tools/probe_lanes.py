"""par-rs / par-ws at every lane_width on equal-nnz slices of an R-MAT graph (dev tool)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200 import selection  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=25)
ap.add_argument("--parts", type=int, default=8)
ap.add_argument("--slices", default="0,3,7")
ap.add_argument("--n", type=int, default=1)
args = ap.parse_args()
full = spmk.DeviceCsr.generate_rmat(args.scale, 16, (0.57, 0.19, 0.19, 0.05), 1)
b = full.row_slices(args.parts)
x = spmk.make_dense_device(full.num_cols, args.n, 7)
for g in [int(v) for v in args.slices.split(",")]:
    s = full.slice(int(b[g]), int(b[g + 1]))
    f = s.features()
    line = [f"slice {g}: rows {s.num_rows} avg {f.avg_row:.1f}"]
    for kid in (spmk.kParRowSplit, spmk.kParBalanced):
        for w in (4, 8, 16, 32):
            r, y = selection.measure_kernel("p", s, x, kid, cfg=spmk.KernelConfig(lane_width=w), repeats=5, warmup=1)
            line.append(f"{kid.name}/W{w} {r.time_seconds * 1e3:.3f}")
            del y
    print(" | ".join(line), flush=True)
    del s
    torch.cuda.empty_cache()
