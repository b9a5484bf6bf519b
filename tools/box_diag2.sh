#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for v in "TCG_LIBPATH=$PWD/ab_base/libtcg_r1.so" "TCG_X=0"; do
  for c in cfg2 cfg3; do
    echo "== $v $c rep $rep" >> gpurun_out/ab8.txt
    env $v timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],2), 'roof', round(d['roofline']['frac'],4), 'fapply_us', round(d['fapply']['us_per_apply'],2), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab8.txt
  done
done
done
timeout 300 python tools/phase_timing.py cfg2 > gpurun_out/phase_cfg2.txt 2>&1
TCG_LIBPATH=$PWD/ab_base/libtcg_r1.so timeout 300 python tools/phase_timing.py cfg2 >> gpurun_out/phase_cfg2.txt 2>&1
E2E_REPS=3 timeout 300 python tools/e2e_breakdown.py cfg5 > gpurun_out/e2e_cfg5.txt 2>&1
for c in cfg5 cfg3; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_steps -c 1 --csv python tools/one_pass.py $c > gpurun_out/ncu_dram_$c.csv 2> gpurun_out/ncu_dram_$c.err
done
