"""Dev probe: per-warp timeline of the lane-per-job seq-ws sweep (cfg2 shape).
SPMK_SELL_TRACE=1 python tools/trace_sell.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402

d = spmk.DeviceCsr.generate_rmat(int(os.environ.get("SCALE", 20)), 16, (0.57, 0.19, 0.19, 0.05), 1)
n = 32
x = spmk.make_dense_device(d.num_cols, n, 0x00D5EED + n)
y = torch.empty((d.num_rows, n), device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.zero_()
    d.spmm(spmk.kSeqBalanced, x, y)
torch.cuda.synchronize()
lib = spmk.spmk.load_library()
buf = (C.c_ulonglong * (4 * 8192))()
cnt = lib.spmk_sell_trace(buf, 8192)
a = np.frombuffer(buf, dtype=np.uint64, count=4 * cnt).reshape(cnt, 4).astype(np.int64)
live = a[:, 1] > 0
a = a[live]
t0 = a[:, 0].min()
st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
dur = en - st
print(f"warps {len(a)}: start max {st.max():.1f} us, end min/median/p90/max {en.min():.1f} / {np.median(en):.1f} / "
      f"{np.percentile(en, 90):.1f} / {en.max():.1f} us")
idx = np.arange(len(a))
for q in range(0, 10):
    sel = (idx * 10 // len(a)) == q
    print(f"  decile {q}: steps {a[sel, 2].mean():7.1f} slices {a[sel, 3].mean():7.1f} dur {dur[sel].mean():6.1f} us "
          f"(max {dur[sel].max():6.1f})  us/step {np.mean(dur[sel] / a[sel, 2]):.3f}")
