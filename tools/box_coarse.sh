#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/phase_timing.py cfg4 cfg5 2>&1 | grep -E "cfg|iters" > gpurun_out/coarse_diag.txt
timeout 300 python tools/coarse_levels.py cfg4 cfg5 >> gpurun_out/coarse_diag.txt 2>&1
timeout 300 python tools/coarse_tree.py cfg4 cfg5 >> gpurun_out/coarse_diag.txt 2>&1
TCG_HOST_TIMING=1 timeout 300 python tools/one_pass.py cfg5 1 >> gpurun_out/coarse_diag.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_update|k_xinv_row" --launch-skip 20 --launch-count 4 --csv python tools/one_pass.py cfg5 1 > gpurun_out/ncu_dmma_cfg5.csv 2> gpurun_out/ncu_dmma_cfg5.err
