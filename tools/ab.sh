#!/bin/bash
# A/B bench: ab_base/ (a git worktree of the baseline commit, built) vs the working tree
summ() { python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); ks=d['kernel_shares'].get('k_steps',{})
        print('$1', d['config']['workload'][:4], 'value', round(d['value'],1), 'ms/pass', round(d['ms_per_step'],3), 'k_steps ms', round(ks.get('ms_per_pass',0),3), 'setup_ms', round(d['setup_ms'],3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])
    elif 'rror' in l: print(l.rstrip())
"; }
for rep in 1 2; do
for c in ${AB_CFGS:-cfg2}; do
 (cd ab_base && timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 --steps 5 2>&1 | summ BASE)
 timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 --steps 5 2>&1 | summ NEW
done; done
