"""Quick device timing of the four variants on a generated R-MAT (dev tool)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--skew", default="heavy")
    ap.add_argument("--ns", default="1,4,32")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--l2", action="store_true")
    args = ap.parse_args()
    skew = {"heavy": (0.57, 0.19, 0.19, 0.05), "uniform": (0.25, 0.25, 0.25, 0.25)}[args.skew]
    t0 = time.time()
    d = spmk.DeviceCsr.generate_rmat(args.scale, args.ef, skew, 1)
    torch.cuda.synchronize()
    print(f"gen s{args.scale} e{args.ef} {args.skew}: nnz={d.nnz} empty={d.empty_rows} maxrow={d.max_row_nnz} "
          f"{time.time() - t0:.2f}s", flush=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    for n in [int(v) for v in args.ns.split(",")]:
        x = spmk.make_dense_device(d.num_cols, n, 0x00D5EED + n)
        y = torch.empty((d.num_rows, n), device="cuda")
        if args.l2:
            spmk.l2_persist_x(st, x)
        byts = 4 * (d.num_rows + 1) + 8 * d.nnz + 4 * d.num_cols * n + 4 * d.num_rows * n
        res = {}
        for kid in spmk.kAllKernels:
            for _ in range(2):
                d.spmm(kid, x, y)
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                d.spmm(kid, x, y)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
            t = sorted(ts)[len(ts) // 2]
            res[kid.name] = t
            print(f"  N={n:4d} {kid.name}: {t * 1e6:9.1f} us  {2 * d.nnz * n / t / 1e9:9.1f} GF/s  "
                  f"{byts / t / 1e9:7.1f} GB/s ({byts / t / 6538.9e9 * 100:5.1f}% of measured HBM)", flush=True)
        print(json.dumps({"n": n, "rule": d.select(n).name, "times": res}), flush=True)
        if args.l2:
            spmk.l2_persist_x(st, None)


if __name__ == "__main__":
    main()
