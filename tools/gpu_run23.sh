timeout 1500 python tools/sweep.py --repeats 5 --warmup 2 --out gpurun_out/sweep_r01e > gpurun_out/sweep_r01e.log 2>&1
tail -1 gpurun_out/sweep_r01e.log
timeout 600 python tools/bench_pagerank.py --scale 25 2>&1 | tail -1
timeout 1200 python tools/bench_large.py 2>&1 | tail -1
