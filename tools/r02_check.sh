# Round-2 GPU check: tests, bench, launch list, ncu of the cfg2 kernels, per-warp trace.
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/gputest.log; cat gpurun_out/gputest.log
timeout 900 python bench.py --steps 10 --warmup 3 2> gpurun_out/bench.err | tail -1 > gpurun_out/bench.json; tail -c 1500 gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
bash tools/ncu_export.sh ncu_sell_cfg2 seq_sell python tools/profile_one.py --n 32 --kernels seq-ws --iters 2
bash tools/ncu_export.sh ncu_fold_cfg2 sell_fold python tools/profile_one.py --n 32 --kernels seq-ws --iters 2
head -22 gpurun_out/ncu_sell_cfg2_summary.txt; head -22 gpurun_out/ncu_fold_cfg2_summary.txt
SPMK_SELL_TRACE=1 timeout 300 python tools/trace_sell.py > gpurun_out/trace_sell.txt 2>&1; cat gpurun_out/trace_sell.txt
