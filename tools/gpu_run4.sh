timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for v in 1 3 4 5; do echo "variant $v"; SPMK_SEQ_VARIANT=$v timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 8,32,64 2>&1 | grep "seq-"; done
for v in 1 3 5; do echo "uniform variant $v"; SPMK_SEQ_VARIANT=$v timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --skew uniform --ns 32 2>&1 | grep "seq-"; done
