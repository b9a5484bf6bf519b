#!/bin/bash
# the driver's bench commands (reference arm first), then the round-2 ncu evidence
mkdir -p gpurun_out
S=$(date +%s); timeout 1700 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - S ))" > gpurun_out/walls.txt
S=$(date +%s); timeout 1700 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "ours rc=$? wall=$(( $(date +%s) - S ))" >> gpurun_out/walls.txt
bash tools/box_ncu_r2.sh
