timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py 2>&1 | tail -6 > gpurun_out/sanitizer_memcheck.txt
cat gpurun_out/sanitizer_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_small.py 2>&1 | tail -6 > gpurun_out/sanitizer_racecheck.txt
cat gpurun_out/sanitizer_racecheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_small.py 2>&1 | tail -4 > gpurun_out/sanitizer_synccheck.txt
cat gpurun_out/sanitizer_synccheck.txt
timeout 300 ./tests/cpp/test_dropin 2>&1 | tail -3
bash tools/ncu_export.sh prof_parws_b_s20 par_ws python tools/profile_one.py --scale 20 --n 1 --kernels par-ws --iters 2
cat gpurun_out/prof_parws_b_s20_summary.txt
