#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/phase_timing.py cfg5 cfg3 cfg2 > gpurun_out/phase_ring.txt 2>&1
for c in cfg3 cfg5 cfg2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/quick_$c.json 2> gpurun_out/quick_$c.err
done
timeout 1500 python -m pytest tests -m gpu -q -x -rA > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
