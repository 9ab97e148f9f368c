"""CPU tests of the C-ABI library: it loads, exports every symbol the public
header declares, and its host-only logic (config checks, selector, features,
partition, tolerance, names) matches the oracle — no device calls."""
import os
import re

import numpy as np
import pytest

import paper_2106_16064_b200 as spmk
from paper_2106_16064_b200 import spmk as mod

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "spmk_capi.h")).read()
    return sorted(set(re.findall(r"\b(spmk_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = spmk.load_library()
    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(mod.EXPORTED_SYMBOLS), set(names) ^ set(mod.EXPORTED_SYMBOLS)
    assert lib.spmk_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", mod.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_kernel_names_roundtrip():
    for i, k in enumerate(spmk.kAllKernels):
        assert spmk.kernel_index(k) == i
        assert spmk.parse_kernel(spmk.kernel_name(k)) == k
        assert spmk.load_library().spmk_kernel_name(i).decode() == spmk.kernel_name(k)
    with pytest.raises(spmk.Error):
        spmk.parse_kernel("nope")


def test_config_validation_matches_reference_rules(orc):
    for lw in (1, 2, 3, 4, 16, 32, 48, 64, 128):
        for vg in (0, 1, 2, 3, 4, 8):
            for sc in (0, 1, 256):
                cfg = spmk.KernelConfig(lane_width=lw, vdl_group=vg, seq_chunk=sc)
                ok = orc.check_config(lw, vg, sc)
                if ok:
                    spmk.check_config(cfg)
                else:
                    with pytest.raises(spmk.Error):
                        spmk.check_config(cfg)


def test_selector_matches_oracle_and_reference_kats(orc):
    rng = np.random.default_rng(5)
    for _ in range(2000):
        f = spmk.MatrixFeatures(avg_row=float(rng.uniform(0, 200)), cv=float(rng.uniform(0, 4)))
        n = int(rng.integers(1, 257))
        t = spmk.SelectorThresholds(int(rng.integers(1, 9)), float(rng.choice([8, 16, 32, 64])),
                                    float(rng.choice([0.5, 1.0, 2.0])))
        assert spmk.select_kernel(f, n, t).index == orc.select_kernel(f.avg_row, f.cv, n, t.n_parallel_max,
                                                                       t.t_parallel_avg, t.t_cv)
    kat = lambda avg, cv, n: spmk.select_kernel(spmk.MatrixFeatures(avg_row=avg, cv=cv), n).name
    assert kat(5, 2.0, 1) == "par-ws" and kat(100, 0.1, 128) == "seq-rs"
    assert kat(10, 3.0, 32) == "seq-ws" and kat(64, 0.5, 2) == "par-rs"
    assert kat(32.0, 0.5, 1) == "par-rs" and kat(10.0, 1.0, 32) == "seq-rs"


def test_host_features_match_oracle(orc, corpus):
    for a in corpus:
        f = spmk.extract_features(spmk.CsrMatrix(a.m, a.k, a.row_ptr, a.col_idx, a.val))
        assert (f.avg_row, f.stdv_row, f.cv) == orc.extract_features(a)
    with pytest.raises(spmk.Error):
        spmk.extract_features(spmk.CsrMatrix(0, 3, [0], [], []))


def test_partition_and_tolerance(orc):
    for items in (0, 5, 16083729, 520756886):
        for parts in (1, 2, 4, 8):
            for w in range(parts):
                assert spmk.partition(items, parts, w) == orc.partition(items, parts, w)
    for mr in (0, 1, 100, 406321):
        assert spmk.kernel_tolerance(mr) == orc.kernel_tolerance(mr)


def test_double_is_unsupported():
    with pytest.raises(spmk.UnsupportedError):
        spmk.CsrMatrix(1, 1, [0, 1], [0], np.array([1.0]))
