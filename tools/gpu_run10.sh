for v in 9 13 14 15 16; do echo "variant $v"; SPMK_SEQ_VARIANT=$v timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 8,32,64 2>&1 | grep "seq-ws"; done
for v in 9 13; do echo "uniform variant $v"; SPMK_SEQ_VARIANT=$v timeout 300 python tools/probe_perf.py --skew uniform --scale 20 --ef 16 --ns 8,32 2>&1 | grep "seq-"; done
