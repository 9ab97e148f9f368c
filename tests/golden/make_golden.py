"""Generate tests/golden/golden.json from the REFERENCE ITSELF.

Runs the unmodified reference headers (via oracle/_ref/libspmk_ref.so, built
from /root/reference/proj/include by oracle/Makefile) and records SHA-256
digests of their outputs: the pinned corpus (corpus.hpp:108-113), R-MAT and
make_dense streams, features, selector choices, plan_balanced chunk starts,
and the four fp32 kernels' Y bits on a subset of the corpus.  The digests
travel with the repo, so the GPU box (which has no /root/reference) checks
the CUDA path and the C oracle against the reference's own outputs.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import RefLib  # noqa: E402

NS = (1, 2, 3, 4, 5, 8, 16, 32, 64, 128)
KERNEL_SUBSET = ("rmat_s8_e4_uniform", "rmat_s8_e16_heavy", "rmat_s10_e8_mild", "rmat_s10_e16_heavy",
                 "rmat_s12_e4_heavy", "single_long_row", "singleton_rows", "empty_row_riddled",
                 "dense_block", "empty")
RMAT_CASES = ((4, 8, (0.57, 0.19, 0.19, 0.05), 1), (8, 8, (0.25, 0.25, 0.25, 0.25), 1234),
              (12, 8, (0.57, 0.19, 0.19, 0.05), 3), (14, 16, (0.45, 0.22, 0.22, 0.11), 9),
              (16, 16, (0.25, 0.25, 0.25, 0.25), 1))
DENSE_CASES = ((1000, 7, 17), (4096, 32, 0x00D5EED + 32), (256, 1, 1001), (65536, 1, 0x00D5EED + 1))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    R = RefLib()
    out = {"source": "reference headers /root/reference/proj/include via oracle/_ref (g++ -O3, no -march)",
           "corpus": [], "select": {}, "plan": {}, "spmm": [], "rmat": [], "dense": []}
    corpus = R.full_corpus(42)
    for a in corpus:
        h = R.handle(a)
        feats = h.extract_features() if a.m >= 1 else None
        out["corpus"].append({
            "name": a.name, "m": a.m, "k": a.k, "nnz": a.nnz, "max_row": a.max_row_nnz(),
            "row_ptr": sha(a.row_ptr), "col_idx": sha(a.col_idx), "values": sha(a.val),
            "features": feats,
        })
        out["select"][a.name] = {str(n): R.select_kernel(feats[0], feats[2], n, stdv=feats[1],
                                                         num_rows=a.m, nnz=a.nnz) for n in range(1, 130)}
        plans = {}
        for ch in (1, 2, 32, 256):
            er, nch = h.plan_balanced(ch)
            plans[str(ch)] = {"num_chunks": nch, "chunk_first_row": sha(er[::ch].astype(np.int64)),
                              "elem_row": sha(er)}
        out["plan"][a.name] = plans
        if a.name in KERNEL_SUBSET:
            for n in NS:
                x = R.make_dense(a.k, n, 1000 + n)
                for kidx in range(4):
                    widths = (32, 4, 2) if kidx < 2 else (32,)
                    chunks = (256, 16, 7) if kidx == 3 else (256,)
                    for W in widths:
                        for S in chunks:
                            y = h.spmm(kidx, x, lane_width=W, seq_chunk=S)
                            out["spmm"].append({"matrix": a.name, "n": n, "kernel": kidx, "lane_width": W,
                                                "seq_chunk": S, "x_seed": 1000 + n, "y": sha(y)})
    for scale, ef, skew, seed in RMAT_CASES:
        a = R.generate_rmat(scale, ef, skew, seed)
        out["rmat"].append({"scale": scale, "edge_factor": ef, "skew": list(skew), "seed": seed, "nnz": a.nnz,
                            "row_ptr": sha(a.row_ptr), "col_idx": sha(a.col_idx)})
    for rows, cols, seed in DENSE_CASES:
        out["dense"].append({"rows": rows, "cols": cols, "seed": seed, "sha": sha(R.make_dense(rows, cols, seed))})
    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("wrote", path, len(out["spmm"]), "kernel digests")


if __name__ == "__main__":
    main()
