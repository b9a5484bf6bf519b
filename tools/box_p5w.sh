#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_nonlinear.py -q -rfE -k "cfg5 or whole_patch or nl2 or small" > gpurun_out/pytest_p5w.log 2>&1; echo rc=$? >> gpurun_out/pytest_p5w.log
: > gpurun_out/ab_p5w.txt
for rep in 1 2; do
for v in 0 1; do
  echo "== SI_MERGE=$v cfg5 rep $rep" >> gpurun_out/ab_p5w.txt
  TCG_SI_MERGE=$v timeout 300 python bench.py --config cfg5 --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],3), 'roof', round(d['roofline']['frac'],4), 'fapply_us', round(d['fapply']['us_per_apply'],2), 'it', d['pcg_iters_per_step'], 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab_p5w.txt
done
done
timeout 600 python tools/phase_timing.py cfg5 > gpurun_out/phase_r2c.txt 2>&1
