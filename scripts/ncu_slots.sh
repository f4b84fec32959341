M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
for v in "HANF_SLOTS=0" "HANF_SLOTS_HOT=4194304" "HANF_SLOTS_HOT=0"; do
  ncu --metrics $M -k regex:union_kernel -c 1 --clock-control none --csv python scripts/policy_sweep.py 5 "$v" > gpurun_out/ncu_slots_${v}.csv 2>&1
done
