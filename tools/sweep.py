#!/usr/bin/env python3
"""BASELINE cfg3 selection-rule sweep on one B200: N in {1..128} over
uniform / banded / heavy R-MAT matrices 2^18-2^22 rows, all four variants and
the rule, bench.hpp semantics (median of repeats, L2 flushed).  Writes the
reference's CSV (emit_csv) and a JSON summary.

    python tools/sweep.py [--scales 18,20,22] [--ns 1,2,4,8,16,32,64,128] [--out profiles/r01_sweep]
    python tools/sweep.py --mtx a.mtx,b.mtx      # real matrices (Matrix Market) instead
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2106_16064_b200 as spmk  # noqa: E402
from paper_2106_16064_b200 import inputs, selection  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scales", default="18,19,20,21,22")
    ap.add_argument("--families", default="uniform,banded,heavy")
    ap.add_argument("--ns", default="1,2,4,8,16,32,64,128")
    ap.add_argument("--repeats", type=int, default=7)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--out", default="gpurun_out/sweep")
    ap.add_argument("--mtx", default="", help="comma-separated Matrix Market files (replaces the synthetic corpus)")
    args = ap.parse_args()
    scales = [int(s) for s in args.scales.split(",")]
    ns = [int(n) for n in args.ns.split(",")]
    t0 = time.time()
    records, feats = [], {}
    if args.mtx:
        corpus = ((os.path.splitext(os.path.basename(p))[0], spmk.DeviceCsr.from_host(spmk.read_matrix_market(p)))
                  for p in args.mtx.split(","))
    else:
        corpus = inputs.sweep_corpus(scales, args.families.split(","))
    for name, a in corpus:
        feats[name] = a.features()
        print(f"{name}: rows {a.num_rows} nnz {a.nnz} avg {feats[name].avg_row:.2f} cv {feats[name].cv:.3f}",
              flush=True)
        recs = selection.run_benchmark([(name, a)], ns, repeats=args.repeats, warmup=args.warmup,
                                       check=not args.no_check)
        for r in recs:
            if not r.selected_by_rule:
                print(f"   n={r.n:4d} {r.kernel}: {r.time_seconds * 1e6:10.1f} us {r.gflops:9.1f} GF/s"
                      f"{'' if r.correct else '  MISMATCH'}", flush=True)
        records += recs
        del a
    s = selection.summarize_selection_loss(records)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".csv", "w") as f:
        selection.emit_csv(records, s, f)
    crecs = selection.calibration_records(records, feats)
    cal = selection.calibrate_thresholds(crecs)
    cal_ext = selection.calibrate_thresholds_extended(crecs)
    # held-out split: calibrate on the even scales, evaluate on the odd ones
    def scale_of(r):
        return int(r.matrix_name.split("-s")[1].split("-")[0]) if "-s" in r.matrix_name else 0
    train = selection.calibration_records([r for r in records if scale_of(r) % 2 == 0], feats)
    test = selection.calibration_records([r for r in records if scale_of(r) % 2 == 1], feats)
    holdout = selection.holdout_calibration(train, test) if train and test else None
    summary = {
        "per_n_loss": s.per_n_loss, "mean_per_n_loss": selection.mean_per_n_loss(s),
        "single_kernel_loss": s.single_kernel_loss,
        "min_single_kernel_loss": selection.min_single_kernel_loss(s),
        "all_correct": all(r.correct for r in records), "cells": len(records) // 5,
        "calibrated_thresholds": cal.__dict__,
        "calibrated_thresholds_extended": cal_ext.__dict__,
        "calibration_loss": {"default": selection.calibration_loss(crecs, selection.SelectorThresholds()),
                             "calibrated": selection.calibration_loss(crecs, cal),
                             "extended": selection.calibration_loss(crecs, cal_ext)},
        "holdout_even_train_odd_test": holdout, "wall_s": round(time.time() - t0, 1),
    }
    with open(args.out + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
