import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import paper_2106_16064_b200 as spmk
if len(sys.argv) > 1: spmk.spmk.load_library(sys.argv[1])
from oracle.oracle import load_oracle, Csr
from test_sell_gpu import mixed_matrix, csr_of, run
orc = load_oracle()
a = mixed_matrix(np.random.default_rng(5)); d = spmk.DeviceCsr.from_host(a)
for chunk in (1, 7, 256):
    for n in (8, 16, 32):
        x = orc.make_dense(a.num_cols, n, 77 + chunk)
        want = orc.spmm(csr_of(a), 3, x, seq_chunk=chunk)
        bad = []
        for rep in range(5):
            y = run(d, x, spmk.KernelConfig(seq_chunk=chunk), seq_impl=2)
            diff = np.nonzero(np.any(y.view(np.uint32) != want.view(np.uint32), axis=1))[0]
            bad.append(len(diff))
        print(sys.argv[1:2], chunk, n, "rows differing per rep", bad, "e.g.", diff[:5], np.diff(np.asarray(a.row_ptr))[diff[:5]] if len(diff) else "")
