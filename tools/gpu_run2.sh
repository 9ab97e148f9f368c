timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
tail -15 gpurun_out/pytest_gpu.txt
timeout 600 python tools/probe_perf.py --scale 20 --ef 16 --ns 1,2,4 > gpurun_out/probe_s20.txt 2>&1
timeout 600 python tools/probe_perf.py --scale 20 --ef 16 --skew uniform --ns 1,4,32 > gpurun_out/probe_s20u.txt 2>&1
cat gpurun_out/probe_s20.txt gpurun_out/probe_s20u.txt | grep -v "^{"
