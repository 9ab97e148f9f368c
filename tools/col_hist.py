"""Dev probe: share of gathers landing on the top-H most frequent columns."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200 import pagerank as prk  # noqa: E402

for scale, ef in ((20, 16), (22, 16), (25, 16), (24, 32)):
    d = spmk.DeviceCsr.generate_rmat(scale, ef, (0.57, 0.19, 0.19, 0.05), 1)
    c = prk.column_counts(d).long()
    s, _ = torch.sort(c, descending=True)
    cs = torch.cumsum(s, 0).double() / d.nnz
    out = {h: round(float(cs[h - 1]), 3) for h in (1024, 4096, 8192, 16384, 32768, 65536, 262144, 1 << 20)}
    print(f"s{scale} e{ef} nnz {d.nnz} distinct cols {(c > 0).sum().item()} top-H share {out}", flush=True)
    del d, c, s, cs
    torch.cuda.empty_cache()
