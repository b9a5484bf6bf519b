#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for v in "TCG_ND_LEAF=32" "TCG_ND_LEAF=64" "TCG_ND_LEAF=128"; do
  for c in cfg4 cfg5; do
    echo "== $v $c rep $rep" >> gpurun_out/ab6.txt
    env $v timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],2), 'roof', round(d['roofline']['frac'],4), 'fapply_us', round(d['fapply']['us_per_apply'],1), 'setup_ms', round(d['setup_ms'],1), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])
" >> gpurun_out/ab6.txt
  done
done
done
for v in 64 128; do TCG_ND_LEAF=$v timeout 300 python tools/coarse_levels.py cfg4 cfg5 >> gpurun_out/ab6.txt 2>&1; done
for v in 64 128; do TCG_ND_LEAF=$v timeout 900 python -m pytest tests/test_gpu_golden.py -q -x -k "cfg4 or cfg5" > gpurun_out/pytest_ab6_$v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab6_$v.log; done
