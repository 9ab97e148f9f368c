"""Workloads for the per-kernel ncu captures (dev tool; runs on the GPU box).

    python tools/profile_workloads.py <name> [--iters K]

Each workload builds its operands (device generators), runs one warm-up call
outside NVTX range "prof", then K calls inside it, and writes the workload's
algorithmic byte counts to gpurun_out/prof_<name>.json so tools/ncu_table.py
can compute achieved GB/s and the X L2 hit rate (SURVEY §5:
1 - (dram read - rowPtr/colIdx/val bytes) / (gathered X bytes = nnz*4N)).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200 import pagerank as prk  # noqa: E402

HEAVY = (0.57, 0.19, 0.19, 0.05)
UNIFORM = (0.25, 0.25, 0.25, 0.25)
# name: (scale, edge factor, skew, N, kernel, config)
W = {
    "cfg2_seqws_n32": (20, 16, HEAVY, 32, "seq-ws", {}),
    "s20_seqws_n8": (20, 16, HEAVY, 8, "seq-ws", {}),
    "s20_seqws_n2": (20, 16, HEAVY, 2, "seq-ws", {}),
    "s20_seqrs_n32": (20, 16, HEAVY, 32, "seq-rs", {}),
    "s20_seqrs_n1": (20, 16, HEAVY, 1, "seq-rs", {}),
    "s20_parrs_n1": (20, 16, HEAVY, 1, "par-rs", {}),
    "s20_parrs_n4": (20, 16, HEAVY, 4, "par-rs", {}),
    "s20_parrs_n32": (20, 16, HEAVY, 32, "par-rs", {}),
    "s20u_parrs_n1": (20, 16, UNIFORM, 1, "par-rs", {}),
    "s20_parws_n1": (20, 16, HEAVY, 1, "par-ws", {}),
    "s20_parws_n4": (20, 16, HEAVY, 4, "par-ws", {}),
    "s20_parws64_n4": (20, 16, HEAVY, 4, "par-ws", {"lane_width": 64}),
    "cfg1_parws_n1": (16, 16, UNIFORM, 1, "par-ws", {}),
    "cfg4_seqws_n64": (24, 32, HEAVY, 64, "seq-ws", {}),
    "cfg5_parws_n1": (25, 16, HEAVY, 1, "par-ws", {}),
    "cfg5_parrs_n1": (25, 16, HEAVY, 1, "par-rs", {}),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--iters", type=int, default=2)
    args = ap.parse_args()
    out = {"name": args.name}
    if args.name.startswith("pagerank"):
        scale = 22
        d = spmk.DeviceCsr.generate_rmat(scale, 16, HEAVY, 1)
        pr = prk.PageRank(d)
        pr.reset()
        pr.step()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("prof")
        for _ in range(args.iters):
            pr.step()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        m = d.num_rows
        out.update(m=m, k=m, nnz=d.nnz, n=1, kernel=pr.kid.name,
                   update_bytes=16 * m, matrix=f"R-MAT s{scale} e16 heavy")
    else:
        scale, ef, skew, n, kname, cfg = W[args.name]
        d = spmk.DeviceCsr.generate_rmat(scale, ef, skew, 1)
        x = spmk.make_dense_device(d.num_cols, n, 0x00D5EED + n)
        y = torch.empty((d.num_rows, n), device="cuda")
        kid = spmk.parse_kernel(kname)
        c = spmk.KernelConfig(**cfg)
        d.spmm(kid, x, y, cfg=c)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("prof")
        for _ in range(args.iters):
            d.spmm(kid, x, y, cfg=c)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        m, k, nnz = d.num_rows, d.num_cols, d.nnz
        out.update(m=m, k=k, nnz=nnz, n=n, kernel=kname, cfg=cfg, max_row=d.max_row_nnz, empty=d.empty_rows,
                   matrix=f"R-MAT s{scale} e{ef} {'heavy' if skew == HEAVY else 'uniform'}")
    out["a_bytes"] = 4 * (out["m"] + 1) + 8 * out["nnz"]
    out["x_bytes"] = 4 * out["k"] * out["n"]
    out["y_bytes"] = 4 * out["m"] * out["n"]
    out["x_gather_bytes"] = out["nnz"] * 4 * out["n"]
    out["iters"] = args.iters
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/prof_{args.name}.json", "w") as f:
        json.dump(out, f)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
