for v in 1 8 9 10 11 12; do echo "variant $v"; SPMK_SEQ_VARIANT=$v timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 8,32,64 2>&1 | grep "seq-ws"; done
for v in 8; do echo "variant $v"; SPMK_SEQ_VARIANT=$v timeout 300 python -m pytest -x -q tests/test_parity_gpu.py 2>&1 | tail -2; done
