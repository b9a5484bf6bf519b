#!/bin/bash
# left-looking local factorisation: full GPU suite, then A/B (TCG_CHOL=right) on cfg5/cfg3/cfg4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rfE -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
: > gpurun_out/left.txt
for rep in 1 2; do
for v in right left; do
 for c in cfg5 cfg3 cfg4; do
  TCG_CHOL=$v timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); f=d['factorisation']; print('$v $c value', round(d['value'],3), 'setup_ms', round(d['setup_ms'],1), 'fac', round(f['local_TFLOPs'],2), round(f['frac'],3), 'ms_local', round(f['ms_local'],1), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/left.txt
 done
done
done
