#!/bin/bash
# A/B of TCG_OVL_CHAIN (chain blocks for the coarse levels above the leaves) inside one call
mkdir -p gpurun_out
rm -f gpurun_out/ab_ovl2.txt
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -q -x -k "overlap" > gpurun_out/pytest_ovl2.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_ovl2.log
run() {  # config, env...
  c=$1; shift
  echo "== $* $c" >> gpurun_out/ab_ovl2.txt
  env "$@" timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],2), 'iters/step', d['pcg_iters_per_step'], 'fapply_us', round(d['fapply']['us_per_apply'],1), 'k_steps_frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab_ovl2.txt
}
for rep in 1 2; do
  run cfg4 TCG_OVERLAP=0
  for k in 0 24 48 96 160; do run cfg4 TCG_OVERLAP=1 TCG_OVL_CHAIN=$k; done
  run cfg5 TCG_OVERLAP=0
  for k in 64 128; do run cfg5 TCG_OVERLAP=1 TCG_OVL_CHAIN=$k; done
done
