#!/bin/bash
# round-2 ncu evidence (never a bench number): launch list of the bench command (cfg5), DRAM
# bytes of the first full k_steps launch (cfg5, cfg3), a --set full capture of a 1-step cfg5
# k_steps launch (csv exports), and of k_nl_assemble (nl2)
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-roofline --no-extras"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_cfg5_bench.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$? >> gpurun_out/ncu_r2.log
for c in cfg5 cfg3; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_steps -c 1 --csv --log-file gpurun_out/k_steps_${c}_dram.csv $B --config $c > gpurun_out/ncu_dram_$c.log 2>&1; echo dram $c rc=$? >> gpurun_out/ncu_r2.log
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_steps -c 1 -o /tmp/k_steps_cfg5 -f python tools/one_pass.py cfg5 1 > gpurun_out/ncu_full5.log 2>&1; echo full5 rc=$? >> gpurun_out/ncu_r2.log
ncu -i /tmp/k_steps_cfg5.ncu-rep --page raw --csv > gpurun_out/k_steps_cfg5_raw.csv 2>/dev/null
ncu -i /tmp/k_steps_cfg5.ncu-rep --page details --csv > gpurun_out/k_steps_cfg5_details.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:k_nl_assemble -c 1 -o /tmp/k_nl -f python tools/one_pass.py nl2 1 > gpurun_out/ncu_nl.log 2>&1; echo fullnl rc=$? >> gpurun_out/ncu_r2.log
ncu -i /tmp/k_nl.ncu-rep --page details --csv > gpurun_out/k_nl_assemble_nl2_details.csv 2>/dev/null
ls -la gpurun_out >> gpurun_out/ncu_r2.log
