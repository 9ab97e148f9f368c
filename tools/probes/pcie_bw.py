"""Dev: pinned H2D / D2H bandwidth alone and concurrent (134 MB, the cfg2 X / Y size)."""
import torch

n = 1 << 25  # floats = 134 MB
hx = torch.empty(n, dtype=torch.float32, pin_memory=True).fill_(1)
hy = torch.empty(n, dtype=torch.float32, pin_memory=True)
dx = torch.empty(n, device="cuda")
dy = torch.ones(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def h2d():
    dx.copy_(hx, non_blocking=True)


def d2h():
    hy.copy_(dy, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        dx.copy_(hx, non_blocking=True)
    with torch.cuda.stream(s2):
        hy.copy_(dy, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms  {n * 4 / ms / 1e6:.1f} GB/s per direction")

ss = [torch.cuda.Stream() for _ in range(8)]


def h2d_split(k):
    def fn():
        cur = torch.cuda.current_stream()
        m = n // k
        for i in range(k):
            ss[i].wait_stream(cur)
            with torch.cuda.stream(ss[i]):
                dx[i * m:(i + 1) * m].copy_(hx[i * m:(i + 1) * m], non_blocking=True)
        for i in range(k):
            cur.wait_stream(ss[i])
    return fn


def h2d_kernel():
    # device-side pull through the mapped (pinned) host pointer: a copy kernel
    dx.copy_(hx.cuda(non_blocking=True))


for k in (2, 4, 8):
    ms = t(h2d_split(k))
    print(f"h2d split {k}: {ms:.3f} ms  {n * 4 / ms / 1e6:.1f} GB/s")
# zero-copy read: a kernel reading the pinned buffer directly over PCIe
import ctypes
ptr = ctypes.c_void_p()
cudart = ctypes.CDLL("libcudart.so") if False else None
