#!/bin/bash
# the driver's two bench commands (reference arm first, then ours), wall-clocked
mkdir -p gpurun_out
S=$(date +%s); timeout 1700 python bench.py --impl reference --steps ${K:-20} --warmup ${W:-5} > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - S ))" > gpurun_out/bench_walls.txt
S=$(date +%s); timeout 1700 python bench.py --steps ${K:-20} --warmup ${W:-5} > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "ours rc=$? wall=$(( $(date +%s) - S ))" >> gpurun_out/bench_walls.txt
