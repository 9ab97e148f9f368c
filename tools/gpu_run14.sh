timeout 300 python -m pytest tests/test_pagerank_gpu.py -x -q 2>&1 | tail -2
bash tools/ncu_export.sh prof_a2_n32 seq_async2 python tools/profile_one.py --n 32 --kernels seq-ws --iters 2
bash tools/ncu_export.sh prof_parws_s25 par_ws python tools/profile_one.py --scale 25 --n 1 --kernels par-ws --iters 2
bash tools/ncu_export.sh prof_parws_s20 par_ws python tools/profile_one.py --scale 20 --n 1 --kernels par-ws --iters 2
ls -la gpurun_out
