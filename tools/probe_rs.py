"""Row-split variants on an R-MAT graph: one call each (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200.inputs import SKEWS  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ns = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,32").split(",")]
d = spmk.DeviceCsr.generate_rmat(scale, 16, SKEWS["heavy"], 1)
torch.cuda.synchronize()
print(f"s{scale}: nnz={d.nnz} maxrow={d.max_row_nnz}", flush=True)
for n in ns:
    x = spmk.make_dense_device(d.num_cols, n, 7 + n)
    y = torch.empty((d.num_rows, n), device="cuda")
    for kid in (spmk.kParRowSplit, spmk.kSeqRowSplit):
        for _ in range(2):
            d.spmm(kid, x, y)
    torch.cuda.synchronize()
