#!/bin/bash
# quick GPU iteration loop: parity subset, phase timing, short benches (no cpu baseline)
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
timeout 300 python -m pytest tests -m gpu -x -q -k "${PYK:-cfg1_full or cfg2_steps or small_cases or virtual or determinism}" 2>&1 | tail -3
fi
timeout 200 python tools/phase_timing.py ${PT_CFGS:-cfg2 cfg3} 2>&1 | grep -v "^$"
for v in ${BENCH_VARIANTS:-default}; do
for c in ${BENCH_CFGS:-cfg2}; do
env $( [ "$v" != default ] && echo $v ) timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 --steps 5 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); ks=d['kernel_shares']['k_steps']
        print('BENCH $v', d['config']['workload'][:4], 'value', round(d['value'],1), 'ms/pass', round(d['ms_per_step'],3), 'k_steps ms', round(ks['ms_per_pass'],3), 'roof', round(d['roofline']['frac'],4), 'setup_ms', round(d['setup_ms'],3), 'fapply GB/s', round((d.get('fapply') or {}).get('GBps',0)), round((d.get('fapply') or {}).get('us_per_apply',0),2), 'us', 'e2e', round(d['e2e']['value'],1), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])
    elif 'Error' in l or 'error' in l: print(l.rstrip())
"
done; done
