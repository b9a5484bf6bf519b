#!/bin/bash
mkdir -p gpurun_out
TCG_HOST_TIMING=1 E2E_REPS=3 timeout 600 python tools/e2e_breakdown.py cfg5 > gpurun_out/e2e_cfg5.txt 2>&1
timeout 600 python tools/phase_timing.py cfg4 > gpurun_out/phase_cfg4.txt 2>&1
