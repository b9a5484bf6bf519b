#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/ab_small.txt
for rep in 1 2; do
for v in 0 1; do
 for c in cfg1 cfg2; do
  echo "== SBBINV=$v $c rep $rep" >> gpurun_out/ab_small.txt
  TCG_SBBINV=$v timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 10 --warmup 3 --nonlinear '' 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],2), 'fapply_us', round(d['fapply']['us_per_apply'],2), 'it', d['pcg_iters_per_step'], 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab_small.txt
 done
done
done
