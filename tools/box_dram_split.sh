#!/bin/bash
# where the DRAM bytes beyond the algorithmic ones go (cfg5): ncu memory counters of an
# isolated F-apply launch (mode 1, 4 applies) and of a one-step launch (never a bench number)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum
for c in ${CFGS:-cfg5}; do
timeout 900 ncu --metrics $M --clock-control none -k regex:k_steps -c 1 --csv --log-file gpurun_out/split_fapply_$c.csv python tools/fapply_only.py $c 4 > gpurun_out/split_fapply_$c.log 2>&1; echo fapply $c rc=$? >> gpurun_out/split.log
timeout 900 ncu --metrics $M --clock-control none -k regex:k_steps -c 1 --csv --log-file gpurun_out/split_step_$c.csv python tools/one_pass.py $c 1 > gpurun_out/split_step_$c.log 2>&1; echo step $c rc=$? >> gpurun_out/split.log
done
