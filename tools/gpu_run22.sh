timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 1,8,32 2>&1 | grep "seq-ws\|par-ws"; done
timeout 300 python tools/probe_perf.py --skew uniform --scale 20 --ef 16 --ns 1,8,32 2>&1 | grep -v "^{"
timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | tail -1
