M=gpu__time_duration.sum,lts__t_sectors.avg,lts__t_sectors.max,lts__t_sectors.min,lts__t_requests.avg,lts__t_requests.max,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,sm__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum
for sk in heavy uniform; do for n in 1 8 32; do
 k=seq-ws; [ $n = 1 ] && k=par-ws
 echo "== $sk n=$n $k"
 ncu --metrics $M --clock-control none -k regex:"seq_kernel|par_ws" -s 1 -c 1 python tools/profile_one.py --n $n --skew $sk --kernels $k --iters 2 2>&1 | grep -E "^\s+(gpu__|lts__|l1tex|dram|sm__)"
done; done
