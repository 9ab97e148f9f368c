#!/bin/bash
# Hub-row path: parity, cfg5 8-way slice 0 launch list, partition projection.
mkdir -p gpurun_out
python -m pytest tests/test_hub_rows_gpu.py -x -q 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/slice_launches.csv python tools/probe_slice.py > gpurun_out/slice.log 2>&1
python tools/bench_large.py --scale 25 --ef 16 --n 1 --parts 2,4,8 > gpurun_out/cfg5_part.json 2> gpurun_out/cfg5_part.err
cat gpurun_out/cfg5_part.json
python tools/probe_perf.py --scale 20 --ef 16 --ns 1,4 2>&1 | grep -E "N=.*par-rs"
