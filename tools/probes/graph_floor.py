"""Dev: per-node time of a CUDA graph of back-to-back tiny kernels (the launch
floor a graph-replayed cfg1 call sits on)."""
import torch

y = torch.empty(65536, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    y.zero_()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(100):
            y.add_(1.0)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) * 1e3 / 100)
print(f"graph node (64K-float elementwise kernel): {best:.2f} us per node")
