./tools/mb 2>&1 | head -12 > gpurun_out/mb_word.txt
cat gpurun_out/mb_word.txt
ncu --set full --clock-control none --import-source on -k regex:seq_kernel -s 1 -c 1 -o gpurun_out/prof_seqws_n32 python tools/profile_one.py --n 32 --kernels seq-ws --iters 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:par_ws -s 1 -c 1 -o gpurun_out/prof_parws_n1 python tools/profile_one.py --n 1 --kernels par-ws --iters 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:par_ws -s 1 -c 1 -o gpurun_out/prof_parws_n1u python tools/profile_one.py --n 1 --skew uniform --kernels par-ws --iters 2 > /dev/null 2>&1
ls gpurun_out
