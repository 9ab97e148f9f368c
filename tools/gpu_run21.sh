SPMK_SEQ_EXT=32 SPMK_PARWS_EXT=32 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
SPMK_SEQ_EXT=1 SPMK_PARWS_EXT=1 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
for e in 256 128 64 32 16; do echo "EXT $e"; SPMK_SEQ_EXT=$e SPMK_PARWS_EXT=$e timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 1,8,32 2>&1 | grep "seq-ws\|par-ws"; done
