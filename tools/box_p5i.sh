#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_golden.py -q -rfE -x -k "cfg5 or whole_patch" > gpurun_out/pytest_p5i.log 2>&1; echo rc=$? >> gpurun_out/pytest_p5i.log
: > gpurun_out/ab_p5i.txt
for rep in 1 2; do
for v in prev cur; do
  if [ $v = prev ]; then E="TCG_LIBPATH=$PWD/ab_base/libtcg_prev.so"; else E="TCG_X=0"; fi
  echo "== $v rep $rep" >> gpurun_out/ab_p5i.txt
  env $E timeout 300 python bench.py --config cfg5 --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],3), 'roof', round(d['roofline']['frac'],4), 'fapply_us', round(d['fapply']['us_per_apply'],2), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab_p5i.txt
done
done
timeout 600 python tools/phase_timing.py cfg5 > gpurun_out/phase_p5i.txt 2>&1
TCG_HOST_TIMING=1 E2E_REPS=3 timeout 600 python tools/e2e_breakdown.py cfg5 > gpurun_out/e2e_cfg5_default.txt 2>&1
TCG_POOL_RETAIN=1 TCG_HOST_TIMING=1 E2E_REPS=3 timeout 600 python tools/e2e_breakdown.py cfg5 > gpurun_out/e2e_cfg5_retain.txt 2>&1
