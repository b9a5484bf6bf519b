#!/bin/bash
# One gpurun call: the cfg5 oracle golden on the box's host cores (196 GB RAM) in the
# background while the GPU suite runs, then the cfg5 full-size parity test against it.
mkdir -p gpurun_out
STEPS=${GOLDEN_STEPS:-3}
nohup python tools/make_golden.py cfg5 --steps $STEPS --workers 16 > gpurun_out/golden_cfg5.log 2>&1 &
GP=$!
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
wait $GP
cp tests/golden/cfg5_s$STEPS.npz gpurun_out/ 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_golden.py -m gpu -q -s -rA > gpurun_out/pytest_golden.log 2>&1
echo "golden rc=$?" >> gpurun_out/pytest_golden.log
