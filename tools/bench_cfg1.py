#!/usr/bin/env python3
"""BASELINE cfg1 on one B200: SpMV (N=1) on the uniform R-MAT 2^16 e16
(65,536^2, ~16 nnz/row, seed 1) — the reference's CPU-runnable case.  Times
the rule's pick per call (events, warm L2 and flushed L2) and as a CUDA graph
of 100 back-to-back calls (launch overhead amortised)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200 import selection  # noqa: E402

a = spmk.DeviceCsr.generate_rmat(16, 16, (0.25, 0.25, 0.25, 0.25), 1)
x = spmk.make_dense_device(a.num_cols, 1, 0x00D5EED + 1)
kid = a.select(1)
out = {"workload": "cfg1 SpMV N=1, R-MAT uniform s16 e16 seed 1 (65,536^2)", "nnz": a.nnz, "kernel": kid.name}
for flush in (False, True):
    r, y = selection.measure_kernel("cfg1", a, x, kid, repeats=21, warmup=5, flush_l2=flush)
    out["us_per_call_" + ("flushed" if flush else "warm")] = round(r.time_seconds * 1e6, 2)
y = torch.empty((a.num_rows, 1), device="cuda")
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    a.spmm(kid, x, y, stream=s)  # warm-up (plans)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(100):
            a.spmm(kid, x, y, stream=s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
per = e0.elapsed_time(e1) * 1e3 / 100
out["us_per_call_graph"] = round(per, 2)
out["gflops_graph"] = round(2.0 * a.nnz / (per * 1e-6) / 1e9, 1)
print(json.dumps(out), flush=True)
