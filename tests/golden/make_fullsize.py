"""Generate tests/golden/fullsize.json from the REFERENCE ITSELF at the full
BASELINE sizes of cfg4 and cfg5 (the matrices the device path is timed on).

For each case the unmodified reference (oracle/_ref/libspmk_ref.so over
/root/reference/proj/include) generates the matrix (rmat.hpp:61-88) and X
(corpus.hpp:116-122), extracts features and picks the kernel
(csr.hpp:166-181, selector.hpp:28-34), runs the fp32 kernels
(kernels.hpp:157-464) and records SHA-256 digests of
  * the CSR arrays (row_ptr int64, col_idx as the device's int32, values),
  * the WHOLE Y of the rule's kernel,
  * Y restricted to a fixed row sample (every row with >= 1024 nonzeros plus
    4096 rows drawn with numpy default_rng(0)) for all four kernels,
so tests/test_fullsize_gpu.py can check the device path bit for bit against
the reference on the GPU box, which has no /root/reference.

    python tests/golden/make_fullsize.py            # ~30 min on 8 cores, ~25 GB RAM
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import RefLib  # noqa: E402

HEAVY = (0.57, 0.19, 0.19, 0.05)
DENSE_SEED = 0x00D5EED  # bench.hpp: X = make_dense(K, n, 0x00D5EED + n)
CASES = {
    # BASELINE configs[3]: SpMM N=64 on R-MAT 2^24, avg degree 32
    "cfg4": dict(scale=24, ef=32, n=64, stochastic=(False,)),
    # BASELINE configs[4]: iterative SpMV on the 2^25-node graph (values as
    # generated, and column-stochastic 1/outdeg(col) as PageRank uses them)
    "cfg5": dict(scale=25, ef=16, n=1, stochastic=(False, True)),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_rows(row_ptr: np.ndarray, m: int) -> np.ndarray:
    """Every row with >= 1024 nonzeros plus 4096 rows from default_rng(0)."""
    lens = np.diff(row_ptr)
    long_rows = np.flatnonzero(lens >= 1024)
    rnd = np.random.default_rng(0).choice(m, size=min(4096, m), replace=False)
    return np.unique(np.concatenate([long_rows, rnd])).astype(np.int64)


def column_stochastic(col: np.ndarray, k: int) -> np.ndarray:
    """val[e] = 1 / outdeg(col[e]) in fp32 (pagerank.py make_column_stochastic)."""
    counts = np.bincount(col, minlength=k).astype(np.float32)
    with np.errstate(divide="ignore"):  # columns without nonzeros are never indexed
        return (np.float32(1.0) / counts)[col]


def main(names=None):
    R = RefLib()
    path = os.path.join(HERE, "fullsize.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out["source"] = "reference headers /root/reference/proj/include via oracle/_ref (g++ -O3, no -march)"
    for name, c in CASES.items():
        if names and name not in names:
            continue
        t0 = time.time()
        a = R.generate_rmat(c["scale"], c["ef"], HEAVY, 1)
        print(f"{name}: generated m={a.m} nnz={a.nnz} in {time.time() - t0:.0f}s", flush=True)
        rows = sample_rows(a.row_ptr, a.m)
        rec = {"scale": c["scale"], "ef": c["ef"], "seed": 1, "skew": list(HEAVY), "n": c["n"],
               "m": a.m, "k": a.k, "nnz": a.nnz, "max_row": a.max_row_nnz(),
               "row_ptr": sha(a.row_ptr), "col_idx_i32": sha(a.col_idx.astype(np.int32)),
               "sample_rows": int(len(rows)), "sample_rows_sha": sha(rows), "values": {}}
        x = R.make_dense(a.k, c["n"], DENSE_SEED + c["n"])
        rec["x"] = sha(x)
        for stoch in c["stochastic"]:
            key = "stochastic" if stoch else "generated"
            if stoch:
                a.val = column_stochastic(a.col_idx, a.k)
            h = R.handle(a)
            feats = h.extract_features()
            rule = R.select_kernel(feats[0], feats[2], c["n"], stdv=feats[1], num_rows=a.m, nnz=a.nnz)
            v = {"values": sha(a.val), "features": feats, "rule": rule, "y_sample": {}}
            for kidx in range(4):
                t1 = time.time()
                y = h.spmm(kidx, x)
                v["y_sample"][str(kidx)] = sha(y[rows])
                if kidx == rule:
                    v["y_full"] = sha(y)
                print(f"  {key} kernel {kidx}: {time.time() - t1:.0f}s", flush=True)
                del y
            rec["values"][key] = v
            del h
        out[name] = rec
        json.dump(out, open(path, "w"), indent=1)
        del a, x


if __name__ == "__main__":
    main(sys.argv[1:] or None)
