import sys, time; sys.path.insert(0, ".")
import numpy as np, torch, paper_2106_16064_b200 as spmk
d = spmk.DeviceCsr.generate_rmat(20, 16, (0.57, 0.19, 0.19, 0.05), 1)
t0 = time.perf_counter(); h = d.download(); print("download ms", (time.perf_counter() - t0) * 1e3)
for i in range(4):
    t0 = time.perf_counter(); d2 = spmk.DeviceCsr.from_host(h); torch.cuda.synchronize(); print("from_host ms", round((time.perf_counter() - t0) * 1e3, 1))
    del d2
import ctypes
rp = np.ascontiguousarray(h.row_ptr, np.int64); ci = np.ascontiguousarray(h.col_idx, np.int64); va = np.ascontiguousarray(h.values, np.float32)
t0 = time.perf_counter(); x = torch.from_numpy(ci).cuda(); torch.cuda.synchronize(); print("torch H2D 128MB pageable ms", round((time.perf_counter() - t0) * 1e3, 1))
