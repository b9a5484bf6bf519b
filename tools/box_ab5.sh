#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_golden.py -q -x -k "cfg5_s3 or cfg4_s10" > gpurun_out/pytest_ab5.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_ab5.log
for rep in 1 2; do
for v in "TCG_SY_GROUP=0" "TCG_SY_GROUP=1"; do
  for c in cfg5 cfg4; do
    echo "== $v $c rep $rep" >> gpurun_out/ab5.txt
    env $v timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],2), 'roof', round(d['roofline']['frac'],4), 'fapply_us', round(d['fapply']['us_per_apply'],1), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])
" >> gpurun_out/ab5.txt
  done
done
done
for v in 0 1; do TCG_SY_GROUP=$v timeout 300 python tools/phase_timing.py cfg5 2>&1 | grep -E "iters" >> gpurun_out/ab5.txt; done
