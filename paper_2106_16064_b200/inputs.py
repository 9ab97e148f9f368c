"""Synthetic operand families for the BASELINE configs, built in HBM.

  rmat(scale, ef, skew, seed)  generate_rmat<float> (rmat.hpp:61-88 +
                               csr.hpp:123-164), bit-identical, on the device
                               (spmk_generate_rmat; gen_kernels.cuh)
  banded(m, half)              new family of the selection sweep:
                               row i -> columns [i-half, i+half] ∩ [0, m),
                               values 1 (avg ~2*half+1, cv ~0)
  SKEWS                        corpus_skews (corpus.hpp:25-32)
"""
from __future__ import annotations

from .spmk import DeviceCsr

SKEWS = {
    "uniform": (0.25, 0.25, 0.25, 0.25),
    "mild": (0.45, 0.22, 0.22, 0.11),
    "heavy": (0.57, 0.19, 0.19, 0.05),
}


def rmat(scale: int, edge_factor: int, skew="heavy", seed: int = 1, device: int = 0) -> DeviceCsr:
    sk = SKEWS[skew] if isinstance(skew, str) else tuple(skew)
    return DeviceCsr.generate_rmat(scale, edge_factor, sk, seed, device=device)


def banded(m: int, half: int = 8, device: int = 0) -> DeviceCsr:
    """Band matrix with canonical rows, generated with torch on the device."""
    import torch

    dev = torch.device("cuda", device)
    rows = torch.arange(m, device=dev, dtype=torch.int64)
    lo = torch.clamp(rows - half, min=0)
    hi = torch.clamp(rows + half, max=m - 1)
    lens = (hi - lo + 1).to(torch.int64)
    row_ptr = torch.zeros(m + 1, dtype=torch.int64, device=dev)
    torch.cumsum(lens, 0, out=row_ptr[1:])
    nnz = int(row_ptr[-1].item())
    pos = torch.arange(nnz, device=dev, dtype=torch.int64)
    r = torch.repeat_interleave(rows, lens, output_size=nnz)
    col = lo[r] + (pos - row_ptr[r])
    vals = torch.ones(nnz, dtype=torch.float32, device=dev)
    return DeviceCsr.from_device(m, m, row_ptr.to(torch.int32), col.to(torch.int32), vals, copy=True)


def sweep_corpus(scales=(18, 19, 20, 21, 22), families=("uniform", "banded", "heavy"), edge_factor=16,
                 seed=1, device=0):
    """The cfg3 selection-sweep corpus (generator; one matrix resident at a time)."""
    for s in scales:
        for fam in families:
            if fam == "banded":
                yield f"banded-s{s}", banded(1 << s, 8, device)
            else:
                yield f"rmat-{fam}-s{s}-e{edge_factor}", rmat(s, edge_factor, fam, seed, device)
