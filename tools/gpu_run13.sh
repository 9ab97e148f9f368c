timeout 300 python -m pytest tests/test_pagerank_gpu.py -x -q 2>&1 | grep -E "assert|Error|passed|failed" | head -20
for T in 8 4 2; do echo "T=$T"; SPMK_PARWS_T=$T timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 1,4 2>&1 | grep "par-ws"; SPMK_PARWS_T=$T timeout 300 python tools/probe_perf.py --skew uniform --scale 20 --ef 16 --ns 1 2>&1 | grep "par-ws"; done
SPMK_PARWS_T=4 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
SPMK_PARWS_T=2 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
timeout 600 python tools/col_hist.py
ncu --set full --clock-control none --import-source on -k regex:seq_async2 -s 1 -c 1 -o gpurun_out/prof_a2_n32 python tools/profile_one.py --n 32 --kernels seq-ws --iters 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:par_ws -s 1 -c 1 -o gpurun_out/prof_parws_s25 python tools/profile_one.py --scale 25 --n 1 --kernels par-ws --iters 2 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
