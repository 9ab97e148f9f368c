"""paper_2106_16064_b200 — B200-native adaptive SpMV/SpMM engine.

Drop-in for the hot path of the arxiv 2106.16064 artifact (`spmk`): the four
kernel variants {par-rs, par-ws, seq-rs, seq-ws}, the nnz-balanced partition,
the feature extractor and the selection rule, as hand-written sm_100a kernels
behind a C ABI (include/spmk_capi.h; C++ drop-in headers include/spmk/*.hpp).
"""
from .spmk import (  # noqa: F401
    CsrMatrix,
    DeviceCsr,
    Error,
    KernelConfig,
    KernelId,
    MatrixFeatures,
    SelectorThresholds,
    UnsupportedError,
    check_config,
    extract_features,
    kAllKernels,
    kParBalanced,
    kParRowSplit,
    kSeqBalanced,
    kSeqRowSplit,
    kernel_index,
    kernel_name,
    kernel_tolerance,
    l2_persist_x,
    launch_count,
    timing_enable,
    timing_last,
    timing_summary,
    load_library,
    make_dense_device,
    parse_kernel,
    partition,
    select_kernel,
    spmm,
)
from .mmio import MatrixMarketHeader, csr_from_coo, read_matrix_market, write_matrix_market  # noqa: F401,E402
