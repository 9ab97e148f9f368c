timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 5,6,7,8,12,24 2>&1 | grep "seq-ws\|par-ws"
