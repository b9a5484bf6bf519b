#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_paper.py -q -rA -x > gpurun_out/pytest_paper.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_paper.log
timeout 300 python tools/item_costs.py cfg5 > gpurun_out/items_ring.txt 2>&1
TCG_NPF=1 timeout 300 python tools/item_costs.py cfg5 > gpurun_out/items_noring.txt 2>&1
timeout 1200 python tools/paper_sweep.py gpurun_out/paper_fig1_gpu.csv > gpurun_out/paper_sweep.log 2>&1
