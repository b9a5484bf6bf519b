#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_paper.py -q -rA > gpurun_out/pytest_paper.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_paper.log
for v in 0 4 8 16; do
  echo "== L2PF=$v" >> gpurun_out/phase_l2pf.txt
  TCG_L2PF=$v timeout 300 python tools/phase_timing.py cfg5 cfg3 2>&1 | grep -E "cfg|iters" >> gpurun_out/phase_l2pf.txt
done
