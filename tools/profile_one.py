"""Run a few SpMM launches of one variant for ncu capture (dev tool)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--skew", default="heavy")
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--kernels", default="seq-ws")
ap.add_argument("--iters", type=int, default=3)
args = ap.parse_args()
skew = {"heavy": (0.57, 0.19, 0.19, 0.05), "uniform": (0.25, 0.25, 0.25, 0.25)}[args.skew]
d = spmk.DeviceCsr.generate_rmat(args.scale, args.ef, skew, 1)
x = spmk.make_dense_device(d.num_cols, args.n, 0x00D5EED + args.n)
y = torch.empty((d.num_rows, args.n), device="cuda")
for name in args.kernels.split(","):
    kid = spmk.parse_kernel(name)
    for _ in range(args.iters):
        d.spmm(kid, x, y)
torch.cuda.synchronize()
print("done")
