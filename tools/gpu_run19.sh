for i in 1 2; do for v in 9 17; do echo "variant $v"; SPMK_SEQ_VARIANT=$v timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 32 2>&1 | grep "seq-"; SPMK_SEQ_VARIANT=$v timeout 300 python tools/probe_perf.py --skew uniform --scale 20 --ef 16 --ns 32 2>&1 | grep "seq-"; done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
