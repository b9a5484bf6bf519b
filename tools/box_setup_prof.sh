#!/bin/bash
# Launch list of one setup + 1 step (cfg5, cfg3): per-kernel device time, and the FP64-pipe
# utilisation of the factorisation kernels (one launch each).
mkdir -p gpurun_out
for c in cfg5 cfg3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/one_pass.py $c 1 > gpurun_out/launches_setup_$c.csv 2> gpurun_out/launches_setup_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none -k regex:"k_update|k_xinv_row|k_potrf|k_trsm" --launch-skip 40 --launch-count 8 --csv python tools/one_pass.py cfg5 1 > gpurun_out/ncu_factor_cfg5.csv 2> gpurun_out/ncu_factor_cfg5.err
