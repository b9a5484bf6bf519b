#!/bin/bash
# quick GPU iteration loop: parity subset, phase timing, short bench (no cpu baseline)
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "cfg1_full or cfg2_steps or small_cases or virtual or determinism" 2>&1 | tail -3
timeout 200 python tools/phase_timing.py ${PT_CFGS:-cfg2 cfg3} 2>&1 | grep -v "^$"
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 --steps 5 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('BENCH', d['config']['workload'][:4], 'value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'roof', round(d['roofline']['frac'],4), 'setup_ms', round(d['setup_ms'],3), 'e2e', round(d['e2e']['value'],1), 'clk', d['clocks'])
    else: print(l.rstrip())
"
