#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rfE > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
bash tools/box_nlprof.sh
: > gpurun_out/ab_nle.txt
for v in 0 1; do
  TCG_NL_ELEM=$v timeout 600 python bench.py --config cfg2 --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3 --extra-configs cfg1 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); n=d['nonlinear']; print('NL_ELEM=$v nl2', round(n['steps_per_s'],2), 'numeric share', round(n['newton_numeric_share'],3))
" >> gpurun_out/ab_nle.txt
done
