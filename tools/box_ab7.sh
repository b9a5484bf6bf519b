#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -q -x -k "golden or small_cases or cfg1_full or sparse" > gpurun_out/pytest_ab7.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_ab7.log
for rep in 1 2; do
for v in "TCG_LIBPATH=$PWD/ab_base/libtcg_sync.so" "TCG_ND_LEAF=32"; do
  for c in cfg5 cfg3; do
    echo "== $v $c rep $rep" >> gpurun_out/ab7.txt
    env TCG_ND_LEAF=32 $v timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); f=d['factorisation']; print('value', round(d['value'],2), 'setup_ms', round(d['setup_ms'],1), 'factor_TF', round(f['local_TFLOPs'],2), 'ms_local', round(f['ms_local'],1), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab7.txt
  done
done
done
