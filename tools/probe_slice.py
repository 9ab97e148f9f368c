"""One equal-nnz row slice of an R-MAT graph, its rule-selected kernel, a few calls (ncu launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=25)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--parts", type=int, default=8)
ap.add_argument("--slice", type=int, default=0)
ap.add_argument("--n", type=int, default=1)
ap.add_argument("--calls", type=int, default=2)
args = ap.parse_args()
full = spmk.DeviceCsr.generate_rmat(args.scale, args.ef, (0.57, 0.19, 0.19, 0.05), 1)
b = full.row_slices(args.parts)
s = full.slice(int(b[args.slice]), int(b[args.slice + 1]))
del full
torch.cuda.empty_cache()
h = s.download()
lens = np.diff(np.asarray(h.row_ptr))
for L in (1024, 4096, 32768):
    m = lens >= L
    print(f"rows >= {L}: {int(m.sum())} rows, {int(lens[m].sum())} nnz of {s.nnz}")
print(f"max row {int(lens.max())}, rows {s.num_rows}")
kid = s.select(args.n)
print("kernel", kid.name, flush=True)
x = spmk.make_dense_device(s.num_cols, args.n, 7)
y = torch.empty((s.num_rows, args.n), device="cuda")
for _ in range(args.calls):
    s.spmm(kid, x, y)
torch.cuda.synchronize()
