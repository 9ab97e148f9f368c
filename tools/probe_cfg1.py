import sys, json; sys.path.insert(0, ".")
import torch, paper_2106_16064_b200 as spmk
if len(sys.argv) > 1:
    spmk.spmk.load_library(sys.argv[1])
QUICK = len(sys.argv) > 2
a = spmk.DeviceCsr.generate_rmat(16, 16, (0.25, 0.25, 0.25, 0.25), 1)
x = spmk.make_dense_device(a.num_cols, 1, 0x00D5EED + 1)
kid = a.select(1)
y = torch.empty((a.num_rows, 1), device="cuda")
def graph_us(**tune):
    for k, v in tune.items(): a.set_tuning(k, v)
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        a.spmm(kid, x, y, stream=s); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(100): a.spmm(kid, x, y, stream=s)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / 100)
    return best
if QUICK:
    if len(sys.argv) > 3:  # extra knob=value pairs for the par-ws line
        for kv in sys.argv[3:]:
            k_, v_ = kv.split("=")
            a.set_tuning(k_, int(v_))
    print(sys.argv[1], sys.argv[3:], "par-ws", round(graph_us(), 2), "par-rs", end=" ")
    kid = spmk.kParRowSplit
    print(round(graph_us(), 2))
    sys.exit(0)
for v in [dict(parws_impl=2, parws_cpt=0), dict(parws_impl=2, parws_cpt=8), dict(parws_impl=2, parws_cpt=16), dict(parws_impl=2, parws_cpt=32), dict(parws_impl=2, parws_cpt=64), dict(parws_impl=1, parws_t=4)]:
    print(v, round(graph_us(**v), 2), flush=True)
for k2 in spmk.kAllKernels:
    kid = k2
    print(k2.name, round(graph_us(parws_impl=2, parws_cpt=0), 2))
