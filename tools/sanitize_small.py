"""Dev: every variant once on small matrices (for compute-sanitizer runs),
including the lane-per-job sweep at every width and shape and the hub-row
kernels on most rows."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402

for skew in ((0.57, 0.19, 0.19, 0.05), (0.25, 0.25, 0.25, 0.25)):
    d = spmk.DeviceCsr.generate_rmat(10, 8, skew, 3)
    for n in (1, 2, 3, 4, 8, 16, 32, 64):
        x = spmk.make_dense_device(d.num_cols, n, 5 + n)
        for kid in spmk.kAllKernels:
            for cfg in (None, spmk.KernelConfig(lane_width=8, seq_chunk=16)):
                d.spmm(kid, x, cfg=cfg)
                if kid in (spmk.kParRowSplit, spmk.kSeqRowSplit):  # hub-row kernels on most rows
                    d.set_tuning("hub_nnz", 8)
                    d.spmm(kid, x, cfg=cfg)
                    d.set_tuning("hub_two_pass", 0)
                    d.spmm(kid, x, cfg=cfg)
                    d.set_tuning("hub_two_pass", -1)
                    d.set_tuning("hub_nnz", -1)
                if kid in (spmk.kSeqBalanced, spmk.kSeqRowSplit) and n in (8, 16, 32, 64):
                    for shape in (1, 2, 3):
                        d.set_tuning("sell_cfg", shape)
                        d.spmm(kid, x, cfg=cfg)
                    d.set_tuning("sell_cfg", 0)
                    xi = x.clone()
                    xi[0, 0] = float("inf")  # X row 0 not finite: the sweep's per-job length test
                    d.spmm(kid, xi, cfg=cfg)
                    d.set_tuning("seq_impl", 3)
                    d.spmm(kid, x, cfg=cfg)
                    d.set_tuning("seq_impl", 2)
    torch.cuda.synchronize()
print("sanitize run ok")
