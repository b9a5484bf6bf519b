#!/bin/bash
# same-box A/B of the L2-resident configs against the pre-overlap library (ab_base/libtcg_base.so,
# built from commit HEAD~4), then the driver's round-end sequence
mkdir -p gpurun_out
rm -f gpurun_out/ab_base.txt
run() {  # config, env...
  c=$1; shift
  echo "== $* $c" >> gpurun_out/ab_base.txt
  env "$@" timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],2), 'iters/step', d['pcg_iters_per_step'], 'fapply_us', round(d['fapply']['us_per_apply'],1), 'k_steps_frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab_base.txt
}
for rep in 1 2; do
  for c in cfg1 cfg2 cfg3; do
    run $c TCG_LIBPATH=$PWD/ab_base/libtcg_base.so
    run $c TCG_NOP=1
  done
done
bash tools/box_final_b.sh
