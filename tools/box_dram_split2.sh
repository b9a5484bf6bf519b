#!/bin/bash
# DRAM bytes of (a) a one-step cfg5 launch with 0 PCG iterations (the per-step fixed part),
# (b) the first full k_steps launch of the bench command on cfg5 / cfg3 / cfg4 (current build)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:k_steps -c 1 --csv --log-file gpurun_out/split_fixed_cfg5.csv python tools/one_pass.py cfg5 1 0.99 > gpurun_out/split_fixed_cfg5.log 2>&1; echo fixed rc=$? >> gpurun_out/split2.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-roofline --no-extras"
for c in cfg5 cfg3 cfg4; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_steps -c 1 --csv --log-file gpurun_out/k_steps_${c}_dram.csv $B --config $c > gpurun_out/ncu_dram_$c.log 2>&1; echo dram $c rc=$? >> gpurun_out/split2.log
done
