#!/bin/bash
# padding skipped in the whole-patch S_bb / S_bb^-1 / Phi items: GPU suite, A/B vs the previous library, phase timing
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rfE -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
: > gpurun_out/ab_pad.txt
for rep in 1 2; do
for v in prev cur; do
  if [ $v = prev ]; then E="TCG_LIBPATH=$PWD/ab_base/libtcg_prev.so"; else E="TCG_X=0"; fi
  echo "== $v rep $rep" >> gpurun_out/ab_pad.txt
  env $E timeout 300 python bench.py --config cfg5 --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],3), 'roof', round(d['roofline']['frac'],4), 'fapply_us', round(d['fapply']['us_per_apply'],2), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab_pad.txt
done
done
timeout 600 python tools/phase_timing.py cfg5 > gpurun_out/phase_pad.txt 2>&1
