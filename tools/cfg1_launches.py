"""Dev: the launches of one cfg1 call per variant (run under ncu for durations)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2106_16064_b200 as spmk  # noqa: E402

a = spmk.DeviceCsr.generate_rmat(16, 16, (0.25, 0.25, 0.25, 0.25), 1)
x = spmk.make_dense_device(a.num_cols, 1, 0x00D5EED + 1)
y = torch.empty((a.num_rows, 1), device="cuda")
print("rule:", a.select(1).name)
for kid in [a.select(1)] + list(spmk.kAllKernels):
    for _ in range(3):
        a.spmm(kid, x, y)
    torch.cuda.synchronize()
