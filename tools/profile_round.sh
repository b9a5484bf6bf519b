#!/bin/bash
# ncu evidence for profiles/: launch list of the bench command (cfg2) and full captures of
# the first k_steps launch for cfg2 and cfg3 (never a bench number: timings come from plain runs)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv $B --no-roofline > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
for c in cfg2 cfg3; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_steps -c 1 -o gpurun_out/k_steps_$c -f $B --config $c --no-roofline > gpurun_out/ncu_full_$c.log 2>&1; echo full $c rc=$?
done
