"""Dev probe: seq-ws under several tuning-knob settings on a generated R-MAT:
bit equality against the first setting and device time (L2 flushed).
    python tools/probe_sell.py --ns 32 --variants "seq_impl=1;seq_impl=2;seq_impl=2,sell_fold=0" """
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402


def timeit(fn, flush, reps):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--skew", default="heavy")
    ap.add_argument("--ns", default="32")
    ap.add_argument("--chunks", default="256")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--variants", default="seq_impl=1;seq_impl=2")
    ap.add_argument("--lib", default=None)
    ap.add_argument("--kernel", default="seq-ws")
    args = ap.parse_args()
    if args.lib:
        spmk.spmk.load_library(args.lib)
    skew = {"heavy": (0.57, 0.19, 0.19, 0.05), "uniform": (0.25, 0.25, 0.25, 0.25)}[args.skew]
    d = spmk.DeviceCsr.generate_rmat(args.scale, args.ef, skew, 1)
    torch.cuda.synchronize()
    print(f"s{args.scale} e{args.ef} {args.skew}: nnz={d.nnz} maxrow={d.max_row_nnz}", flush=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    kid = spmk.parse_kernel(args.kernel)
    variants = [dict(kv.split("=") for kv in v.split(",")) for v in args.variants.split(";")]
    keys = sorted({k for v in variants for k in v})
    defaults = {k: d.get_tuning(k) for k in keys}
    for ch in [int(c) for c in args.chunks.split(",")]:
        cfg = spmk.KernelConfig(seq_chunk=ch)
        for n in [int(v) for v in args.ns.split(",")]:
            x = spmk.make_dense_device(d.num_cols, n, 0x00D5EED + n)
            ref = None
            t_ref = None
            for v in variants:
                for k in keys:
                    d.set_tuning(k, int(v.get(k, defaults[k])))
                y = torch.full((d.num_rows, n), float("nan"), device="cuda")
                t0 = time.time()
                d.spmm(kid, x, y, cfg=cfg)
                torch.cuda.synchronize()
                first = time.time() - t0
                t = timeit(lambda: d.spmm(kid, x, y, cfg=cfg), flush, args.reps)
                if ref is None:
                    ref, t_ref = y, t
                ndiff = int((ref.view(torch.int32) != y.view(torch.int32)).sum().item())
                name = ",".join(f"{k}={v[k]}" for k in v)
                print(f"  chunk={ch} N={n} [{name}]: {t * 1e6:8.1f} us {2 * d.nnz * n / t / 1e9:8.1f} GF/s "
                      f"x{t_ref / t:.3f} differing={ndiff} (first call {first * 1e3:.1f} ms)", flush=True)


if __name__ == "__main__":
    main()
