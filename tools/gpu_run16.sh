timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/bench_pagerank.py --scale 25 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pr_launches.csv python tools/pagerank_once.py 25 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/pr_launches.csv')))
h=None
for r in rows:
    if 'Kernel Name' in r: h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r))
        if int(d['ID'])>=42: print(d['ID'], d['Kernel Name'][:60], d['Metric Value'])
PY
timeout 300 python tools/probe_perf.py --scale 20 --ef 16 --ns 1,4,32 2>&1 | grep -v "^{"
