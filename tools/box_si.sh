#!/bin/bash
# explicit S_bb^-1 in the iteration: full GPU suite, then A/B (TCG_SBBINV=0/1) on cfg3/cfg4/cfg5, same box
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rfE > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
: > gpurun_out/ab_si.txt
for rep in 1 2; do
for v in 0 1; do
 for c in cfg5 cfg3 cfg4; do
  echo "== SBBINV=$v $c rep $rep" >> gpurun_out/ab_si.txt
  TCG_SBBINV=$v timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],3), 'roof', round(d['roofline']['frac'],4), 'fapply_us', round(d['fapply']['us_per_apply'],2), 'fapply_frac', round(d['fapply']['frac'],4), 'it', d['pcg_iters_per_step'], 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab_si.txt
 done
done
done
