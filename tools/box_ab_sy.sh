#!/bin/bash
# whole-patch S_bb apply (default) vs row items (TCG_SY_SPLIT=1) on cfg5, same box; cfg5 golden parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_golden.py -q -rfE -k "cfg5" > gpurun_out/golden_cfg5.log 2>&1; echo rc=$? >> gpurun_out/golden_cfg5.log
: > gpurun_out/ab_sy.txt
for rep in 1 2; do
for v in split patch; do
  if [ $v = split ]; then E="TCG_SY_SPLIT=1"; else E="TCG_X=0"; fi
  echo "== $v rep $rep" >> gpurun_out/ab_sy.txt
  env $E timeout 300 python bench.py --config cfg5 --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],3), 'roof', round(d['roofline']['frac'],4), 'fapply_us', round(d['fapply']['us_per_apply'],2), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab_sy.txt
done
done
