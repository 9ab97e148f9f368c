#!/usr/bin/env python3
"""BASELINE cfg5 across GPUs (torchrun, one process per GPU, NCCL):
PageRank-style iterative SpMV on R-MAT 2^25 heavy e16, equal-nnz row slices,
per-iteration exchange of the x slices by NCCL broadcasts or by the fused
P2P update kernel (--exchange p2p).  Times `iters` iterations on the device,
max over ranks.

  python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 \\
      tools/bench_pagerank_dist.py --exchange p2p
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200 import pagerank as prk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=25)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"])
args = ap.parse_args()
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
full = spmk.DeviceCsr.generate_rmat(args.scale, args.ef, (0.57, 0.19, 0.19, 0.05), 1, device=local)
dp = prk.DistributedPageRank(full, 0.85, exchange=args.exchange)
nnz_local = dp.a.nnz
del full
dp.run(2)  # warm-up (plans, NCCL channels)
torch.cuda.synchronize()
dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
x, hist = dp.run(args.iters)
e1.record()
torch.cuda.synchronize()
t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
dist.all_reduce(t, op=dist.ReduceOp.MAX)
nnz = torch.tensor([float(nnz_local)], dtype=torch.float64, device="cuda")
dist.all_reduce(nnz)
if dist.get_rank() == 0:
    ms = float(t.item())
    print(json.dumps({"workload": f"cfg5 PageRank R-MAT s{args.scale} e{args.ef}, {dist.get_world_size()} GPUs",
                      "exchange": args.exchange, "iters": args.iters, "ms_total_max_over_ranks": round(ms, 3),
                      "ms_per_iter": round(ms / args.iters, 4),
                      "gflops": round(2.0 * float(nnz.item()) * args.iters / (ms * 1e-3) / 1e9, 1),
                      "final_l1_residual": float(hist[-1].item())}), flush=True)
dp.close()
dist.destroy_process_group()
