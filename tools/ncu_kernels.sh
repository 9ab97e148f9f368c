#!/bin/bash
# Per-kernel ncu captures of every kernel on the path (GPU box):
#   bash tools/ncu_kernels.sh [workload ...]      (default: all of tools/profile_workloads.py)
# For each workload: every launch inside NVTX range "prof" with the metric set
# below (time, DRAM bytes, L2 hit rate, warp instructions, issue activity,
# occupancy, registers, per-opcode SASS counts for the SHFL share, thread
# efficiency).  Raw CSV -> gpurun_out/ncu_<workload>.csv; tools/ncu_table.py
# reduces them.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,\
smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,\
sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,\
smsp__thread_inst_executed_per_inst_executed.ratio,sass__inst_executed_per_opcode,\
lts__t_bytes.sum,l1tex__t_bytes.sum,launch__grid_size,launch__block_size
ALL="cfg2_seqws_n32 s20_seqws_n8 s20_seqws_n2 s20_seqrs_n32 s20_seqrs_n1 s20_parrs_n1 s20_parrs_n4 s20_parrs_n32 s20u_parrs_n1 s20_parws_n1 s20_parws_n4 s20_parws64_n4 cfg1_parws_n1 cfg4_seqws_n64 cfg5_parws_n1 cfg5_parrs_n1 pagerank"
mkdir -p gpurun_out
for w in ${@:-$ALL}; do
  timeout 900 ncu --metrics $M --print-metric-instances details --clock-control none --nvtx --nvtx-include "prof/" \
    --csv --log-file gpurun_out/ncu_$w.csv python tools/profile_workloads.py $w > gpurun_out/prof_$w.log 2>&1
  echo "$w: $(grep -c '"' gpurun_out/ncu_$w.csv) rows"
done
python tools/ncu_table.py gpurun_out > gpurun_out/ncu_table.md
cat gpurun_out/ncu_table.md
