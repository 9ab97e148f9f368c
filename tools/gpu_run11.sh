timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 600 python tools/sweep.py --scales 18 --ns 1,4,32 --repeats 3 --out gpurun_out/sweep_small 2>&1 | tail -3
timeout 900 python tools/bench_pagerank.py --scale 25 2>&1 | tail -2
