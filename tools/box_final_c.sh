#!/bin/bash
# fine sweep of TCG_OVL_CHAIN around the default on cfg4, then the driver's round-end sequence
mkdir -p gpurun_out
rm -f gpurun_out/ab_ovl4.txt
run() {  # config, env...
  c=$1; shift
  echo "== $* $c" >> gpurun_out/ab_ovl4.txt
  env "$@" timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],2), 'iters/step', d['pcg_iters_per_step'], 'fapply_us', round(d['fapply']['us_per_apply'],1), 'k_steps_frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab_ovl4.txt
}
run cfg4 TCG_NOP=1
for k in 112 128 144 176; do run cfg4 TCG_OVL_CHAIN=$k; done
run cfg4 TCG_NOP=1
bash tools/box_final_b.sh
