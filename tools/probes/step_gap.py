"""Dev: cfg2 step time with / without a host sync per step, and from a CUDA graph
(does host enqueue latency leak into the device-timed step?)."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2106_16064_b200 as spmk  # noqa: E402

a = spmk.DeviceCsr.generate_rmat(20, 16, (0.57, 0.19, 0.19, 0.05), 1)
x = spmk.make_dense_device(a.num_cols, 32, 0x00D5EED + 32)
y = torch.empty((a.num_rows, 32), device="cuda")
kid = a.select(32)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for _ in range(3):
    a.spmm(kid, x, y, stream=st)
torch.cuda.synchronize()


def run(mode, steps=20):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    main = []
    spmk.timing_enable(mode == "sync")
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(st)
        if mode == "graph":
            g.replay()
        else:
            a.spmm(kid, x, y, stream=st)
        ev[i][1].record(st)
        if mode == "sync":
            main.append(spmk.timing_last())
    torch.cuda.synchronize()
    spmk.timing_enable(False)
    ts = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
    print(mode, "median step us", round(ts[len(ts) // 2], 1), "min", round(ts[0], 1),
          ("main/whole us %.1f / %.1f" % (main[-1][0] * 1e3, main[-1][1] * 1e3)) if main else "")


s2 = torch.cuda.Stream()
s2.wait_stream(st)
with torch.cuda.stream(s2):
    a.spmm(kid, x, y, stream=s2)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s2):
        a.spmm(kid, x, y, stream=s2)
torch.cuda.synchronize()
for m in ("sync", "nosync", "graph", "sync", "nosync", "graph"):
    run(m)
