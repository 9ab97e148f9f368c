timeout 300 python tools/bench_cfg1.py 2>&1 | tail -2
timeout 300 python bench.py --impl reference --scale 16 --steps 5 --warmup 2 2>&1 | tail -1
