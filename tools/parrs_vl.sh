#!/bin/bash
# par-rs virtual lanes per physical lane (SPMK_PARRS_VL): parity + timing.
for V in 4 8; do SPMK_PARRS_VL=$V timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "lane_width or full_corpus" 2>&1 | tail -1; done
for V in 1 4 8; do
  echo "== VL=$V"
  SPMK_PARRS_VL=$V python tools/probe_perf.py --scale 22 --ef 16 --ns 1,2,4 2>&1 | grep -E "N=.*par-rs"
  SPMK_PARRS_VL=$V python tools/probe_perf.py --scale 20 --ef 16 --skew uniform --ns 1,4 2>&1 | grep -E "N=.*par-rs"
  SPMK_PARRS_VL=$V python tools/probe_lanes.py --slices 7 2>&1 | tail -1
done
