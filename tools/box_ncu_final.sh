#!/bin/bash
# ncu --set full captures of a one-step k_steps launch of the final library: cfg5 (headline) and
# cfg4 (S_bb^-1 side items under the coarse solve); csv exports only (never a bench number)
mkdir -p gpurun_out
for c in cfg5 cfg4; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_steps -c 1 -o /tmp/k_steps_$c -f python tools/one_pass.py $c 1 > gpurun_out/ncu_full_$c.log 2>&1; echo full $c rc=$? >> gpurun_out/ncu_final.log
  ncu -i /tmp/k_steps_$c.ncu-rep --page details --csv > gpurun_out/k_steps_${c}_final_details.csv 2>/dev/null
  ncu -i /tmp/k_steps_$c.ncu-rep --page raw --csv > gpurun_out/k_steps_${c}_final_raw.csv 2>/dev/null
done
