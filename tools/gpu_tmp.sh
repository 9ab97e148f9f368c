timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_pagerank_gpu.py -x -q 2>&1 | tail -1
for sk in heavy uniform; do timeout 300 python tools/probe_perf.py --skew $sk --scale 20 --ef 16 --ns 1,4 2>&1 | grep "par-ws"; done
timeout 600 python tools/bench_pagerank.py --scale 25 2>&1 | tail -1
