for ts in 256 512 1024 2048; do echo "TS=$ts"; SPMK_SEQ_TILE_NNZ=$ts timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 8,32 2>&1 | grep "seq-ws"; done
