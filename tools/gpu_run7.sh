ncu --set full --clock-control none --import-source on -k regex:seq_kernel -s 1 -c 1 -o gpurun_out/prof_seqws_n8h python tools/profile_one.py --n 8 --kernels seq-ws --iters 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:seq_kernel -s 1 -c 1 -o gpurun_out/prof_seqws_n8u python tools/profile_one.py --n 8 --skew uniform --kernels seq-ws --iters 2 > /dev/null 2>&1
ls gpurun_out
