timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 1,2,4,8,32,64 2>&1 | grep -v "^{"
SPMK_PARWS_MINB=5 timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 1,4 2>&1 | grep "par-ws"
timeout 300 python tools/probe_perf.py --skew uniform --scale 20 --ef 16 --ns 1,8,32 2>&1 | grep -v "^{"
for v in 1 2 9 15; do echo "variant $v"; SPMK_SEQ_VARIANT=$v timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 8,32 2>&1 | grep "seq-ws"; done
