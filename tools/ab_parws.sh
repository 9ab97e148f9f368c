#!/bin/bash
# par-ws implementations A/B (dev tool): SPMK_PARWS_IMPL=1 (tile kernel) vs 2 (streaming
# head-flag kernel) at pipeline depth SPMK_PARWS_T = 4 / 8
for r in 1 2; do
  for cfg in "1 4" "2 4" "2 2"; do
    set -- $cfg
    echo "== impl $1 depth $2"
    SPMK_PARWS_IMPL=$1 SPMK_PARWS_T=$2 python tools/probe_perf.py --scale 20 --ef 16 --ns 1,2,4 --reps 20 2>&1 | grep -E "par-ws"
    SPMK_PARWS_IMPL=$1 SPMK_PARWS_T=$2 python tools/probe_perf.py --scale 16 --ef 16 --skew uniform --ns 1 --reps 20 2>&1 | grep -E "par-ws"
    SPMK_PARWS_IMPL=$1 SPMK_PARWS_T=$2 python tools/probe_perf.py --scale 25 --ef 16 --ns 1 --reps 5 2>&1 | grep -E "par-ws"
  done
done
