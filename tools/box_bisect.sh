#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do
for v in r1 nopred nohook neither cur; do
  if [ $v = cur ]; then E="TCG_X=0"; else E="TCG_LIBPATH=$PWD/ab_base/libtcg_$v.so"; fi
  for c in cfg2 cfg3 cfg5; do
    echo "== $v $c rep $rep" >> gpurun_out/bisect.txt
    env $E timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],2), 'roof', round(d['roofline']['frac'],4), 'fapply_us', round(d['fapply']['us_per_apply'],2), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/bisect.txt
  done
done
done
