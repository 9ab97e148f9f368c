timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_pagerank_gpu.py -x -q 2>&1 | tail -2
for v in 1 2; do echo "V=$v"; for sk in heavy uniform; do SPMK_PARWS_V=$v timeout 300 python tools/probe_perf.py --skew $sk --scale 20 --ef 16 --ns 1,2,4 2>&1 | grep "par-ws"; done; done
timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 32 2>&1 | grep "seq-ws"
timeout 600 python tools/bench_pagerank.py --scale 25 2>&1 | tail -1
