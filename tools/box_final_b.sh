#!/bin/bash
# the driver's round-end sequence: gpu tests, smoke, both bench arms (wall-clocked)
mkdir -p gpurun_out
S=$(date +%s); timeout 1800 python -m pytest tests -m gpu -q -rfE > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? wall=$(( $(date +%s) - S ))" > gpurun_out/walls.txt
S=$(date +%s); timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$? wall=$(( $(date +%s) - S ))" >> gpurun_out/walls.txt
S=$(date +%s); timeout 1700 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - S ))" >> gpurun_out/walls.txt
S=$(date +%s); timeout 1700 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "ours rc=$? wall=$(( $(date +%s) - S ))" >> gpurun_out/walls.txt
