timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_dropin_cpp.py -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_r01d.json
cat gpurun_out/bench_r01d.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 2400 python tools/sweep.py --repeats 5 --warmup 2 --out gpurun_out/sweep_r01d > gpurun_out/sweep_r01d.log 2>&1
tail -1 gpurun_out/sweep_r01d.log
