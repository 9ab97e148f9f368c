timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_r01c.json
cat gpurun_out/bench_r01c.json
timeout 1500 python tools/sweep.py --repeats 5 --out gpurun_out/sweep_r01c > gpurun_out/sweep_r01c.log 2>&1
tail -1 gpurun_out/sweep_r01c.log
timeout 600 python tools/bench_pagerank.py --scale 25 2>&1 | tail -1
