#!/bin/bash
# ncu evidence for profiles/: launch list of the bench command (cfg2), full captures of the
# first k_steps launch for cfg2 and cfg3 (exported to csv on the box, reports deleted: the
# merge-back limit is 64 MiB), DRAM bytes + duration of the first cfg5 k_steps launch.
# Never a bench number: timings come from plain runs.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-roofline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
for c in cfg2 cfg3; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_steps -c 1 -o /tmp/k_steps_$c -f $B --config $c > gpurun_out/ncu_full_$c.log 2>&1; echo full $c rc=$?
  ncu -i /tmp/k_steps_$c.ncu-rep --page raw --csv > gpurun_out/k_steps_${c}_raw.csv 2>/dev/null
  ncu -i /tmp/k_steps_$c.ncu-rep --page details --csv > gpurun_out/k_steps_${c}_details.csv 2>/dev/null
  ncu -i /tmp/k_steps_$c.ncu-rep --page source --csv --print-source sass > /tmp/src_$c.csv 2>/dev/null; head -c 3000000 /tmp/src_$c.csv > gpurun_out/k_steps_${c}_source_head.csv
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_steps -c 1 --csv --log-file gpurun_out/k_steps_cfg5_dram.csv $B --config cfg5 > gpurun_out/ncu_cfg5.log 2>&1; echo cfg5 rc=$?
ls -la gpurun_out
