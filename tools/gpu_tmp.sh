timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_dropin_cpp.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 32,64,128 2>&1 | grep "seq-"
