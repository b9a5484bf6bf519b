#!/bin/bash
# A/B of P5 item merging + one ncu --set full capture of k_steps (cfg5, 1 step)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_golden.py -q -x -k "cfg5 or cfg4_s10" > gpurun_out/pytest_ncu5.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_ncu5.log
for rep in 1 2; do
for v in "TCG_P5_SPLIT=1" "TCG_P5_SPLIT=0"; do
  for c in cfg5; do
    echo "== $v $c rep $rep" >> gpurun_out/ab4.txt
    env $v timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],2), 'roof', round(d['roofline']['frac'],4), 'fapply_us', round(d['fapply']['us_per_apply'],1), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])
" >> gpurun_out/ab4.txt
  done
done
done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_steps -c 1 -o gpurun_out/k_steps_cfg5_r2 python tools/one_pass.py cfg5 1 > gpurun_out/ncu_full5.log 2>&1
