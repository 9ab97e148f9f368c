set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 300 ./tools/mb > gpurun_out/mb.txt 2>&1
timeout 600 python tools/probe_perf.py --scale 20 --ef 16 --ns 1,4,8,32,64,128 > gpurun_out/probe_s20.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/mb.txt | head -50; cat gpurun_out/probe_s20.txt; tail -1 gpurun_out/bench.txt
