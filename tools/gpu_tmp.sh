timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -1
timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 4,8,16 2>&1 | grep "seq-"
timeout 300 python tools/probe_perf.py --skew uniform --scale 20 --ef 16 --ns 8,16 2>&1 | grep "seq-"
