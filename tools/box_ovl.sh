#!/bin/bash
# A/B of TCG_OVERLAP (S_bb^-1 items under the sparse coarse solve's waits) inside one call,
# parity of the new path first, then the DRAM split diagnostics of cfg5
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -q -x -k "overlap" > gpurun_out/pytest_ovl.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_ovl.log
for rep in 1 2; do
for v in 0 1; do
  for c in cfg4 cfg5; do
    echo "== TCG_OVERLAP=$v $c rep $rep" >> gpurun_out/ab_ovl.txt
    env TCG_OVERLAP=$v timeout 300 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 0 --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('value', round(d['value'],2), 'iters/step', d['pcg_iters_per_step'], 'fapply_us', round(d['fapply']['us_per_apply'],1), 'k_steps_frac', round(d['roofline']['frac'],3), 'clk', d['clocks']['sm_mhz'])
" >> gpurun_out/ab_ovl.txt
  done
done
done
timeout 600 python -m pytest tests/test_gpu_golden.py -q -x -k "cfg4" > gpurun_out/pytest_ovl_cfg4.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_ovl_cfg4.log
bash tools/box_dram_split.sh
