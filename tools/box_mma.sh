#!/bin/bash
# 3-stage half-K DMMA stream (2 CTAs/SM): full GPU suite, then cfg5/cfg3 bench (factorisation field)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rfE > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
: > gpurun_out/mma.txt
for c in cfg5 cfg3 cfg4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); f=d['factorisation']; print('$c value', round(d['value'],3), 'setup_ms', round(d['setup_ms'],1), 'fac', round(f['local_TFLOPs'],2), round(f['frac'],3), 'ms_local', round(f['ms_local'],1), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/mma.txt
done
