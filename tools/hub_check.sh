#!/bin/bash
# Hub-row path: parity, launch list, timing of the row-split variants.
mkdir -p gpurun_out
python -m pytest tests/test_hub_rows_gpu.py -x -q 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rs_launches.csv \
  python tools/probe_rs.py 20 1,32 > /dev/null 2>&1
for M in 122880; do
  echo "== SPMK_HUB_SMEM=$M"
  SPMK_HUB_SMEM=$M python tools/probe_perf.py --scale 20 --ef 16 --ns 1,8,32,128 2>&1 | grep -E "N=.*-rs"
done
