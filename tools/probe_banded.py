"""Dev probe: the four variants on wide-band matrices (avg row >= 32, where
the rule picks par-rs at N <= 4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200 import inputs, selection  # noqa: E402

for half in (32, 128):
    a = inputs.banded(1 << 20, half)
    f = a.features()
    for n in (1, 4, 32):
        x = spmk.make_dense_device(a.num_cols, n, 7)
        res = {}
        for kid in spmk.kAllKernels:
            r, _ = selection.measure_kernel("b", a, x, kid, repeats=5, warmup=2)
            res[kid.name] = round(r.time_seconds * 1e6, 1)
        print(f"banded half={half} avg={f.avg_row:.1f} N={n} rule={spmk.select_kernel(f, n).name} us={res}", flush=True)
