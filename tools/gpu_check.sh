# Round-end style check on the GPU box: tests, smoke, bench, launch list,
# ncu capture of the bench's dominant kernel (text summaries under gpurun_out/).
set -x
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/bench.json
cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
bash tools/ncu_export.sh prof_bench_dominant seq_async2 python tools/profile_one.py --n 32 --kernels seq-ws --iters 2
cat gpurun_out/prof_bench_dominant_summary.txt
