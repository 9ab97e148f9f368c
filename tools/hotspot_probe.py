"""Dev probe: is the heavy R-MAT column distribution slow to gather (L2 hot
spots)?  torch.index_select of X rows by (a) uniform random columns, (b) the
heavy matrix's colIdx in CSR order, (c) the same colIdx randomly permuted."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402

d = spmk.DeviceCsr.generate_rmat(20, 16, (0.57, 0.19, 0.19, 0.05), 1)
col = torch.from_numpy(d.download().col_idx).cuda()
nnz = col.numel()
K = d.num_cols
g = torch.Generator(device="cuda").manual_seed(0)
uni = torch.randint(0, K, (nnz,), device="cuda", generator=g)
perm = col[torch.randperm(nnz, device="cuda", generator=g)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in (1, 8, 32):
    x = torch.randn(K, n, device="cuda")
    for name, idx in (("uniform", uni), ("heavy-csr", col), ("heavy-perm", perm)):
        out = torch.empty(nnz, n, device="cuda")
        for _ in range(2):
            torch.index_select(x, 0, idx, out=out)
        ts = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.index_select(x, 0, idx, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = sorted(ts)[2]
        print(f"N={n:3d} {name:11s} {t*1e3:8.1f} us  {nnz/t/1e6:7.1f} G rows/s", flush=True)
