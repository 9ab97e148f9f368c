"""Dev: a few eager PageRank iterations (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200 import pagerank as prk  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 25
d = spmk.DeviceCsr.generate_rmat(scale, 16, (0.57, 0.19, 0.19, 0.05), 1)
pr = prk.PageRank(d)
pr.reset()
for _ in range(3):
    pr.step()
torch.cuda.synchronize()
print("ok")
