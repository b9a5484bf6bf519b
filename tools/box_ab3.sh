#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -q -x -k "golden or small_cases or warm_start_matches or cfg1_full" > gpurun_out/pytest_ab3.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_ab3.log
for rep in 1 2; do
for v in "TCG_STEP_FLAGS=2" "TCG_STEP_FLAGS=0"; do
  for c in ${AB_CFGS:-cfg5 cfg3 cfg4}; do
    echo "== $v $c rep $rep" >> gpurun_out/ab3.txt
    env $v timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],2), 'roof', round(d['roofline']['frac'],4), 'fapply_us', round(d['fapply']['us_per_apply'],1), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])
" >> gpurun_out/ab3.txt
  done
done
done
