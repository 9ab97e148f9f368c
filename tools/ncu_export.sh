# usage: tools/ncu_export.sh <name> <kernel regex> <command...>   (on the GPU box)
# Captures one launch with the full set, writes text summaries under gpurun_out/
# (details, raw metrics subset, hot SASS lines); keeps the .ncu-rep only if small.
name=$1; kre=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s 1 -c 1 -o gpurun_out/$name "$@" > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/$name.ncu-rep > gpurun_out/${name}_summary.txt 2>&1
python tools/ncu_hot.py gpurun_out/$name.ncu-rep 60 top > gpurun_out/${name}_hot.txt 2>&1
python tools/ncu_hot.py gpurun_out/$name.ncu-rep 60 seq > gpurun_out/${name}_seq.txt 2>&1
ncu -i gpurun_out/$name.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keep=[i for i,k in enumerate(h) if any(s in k for s in ('dram__bytes','lts__t_sector','lts__t_request','l1tex__t_sector_hit','gpu__time_duration','sm__throughput','sm__warps_active','launch__','smsp__inst_executed.sum','lts__throughput','l1tex__throughput','dram__throughput'))]
for row in r[2:]:
  for i in keep: print(h[i], r[1][i], row[i])
" > gpurun_out/${name}_raw.txt
sz=$(stat -c %s gpurun_out/$name.ncu-rep 2>/dev/null || echo 0)
[ "$sz" -gt 20000000 ] && rm -f gpurun_out/$name.ncu-rep
true
