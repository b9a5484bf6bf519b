#!/bin/bash
# compute-sanitizer on cfg1 (tool = racecheck | synccheck | memcheck), 2 steps
mkdir -p gpurun_out
T=${1:-racecheck}
timeout 1500 compute-sanitizer --tool $T --print-limit 50 python tools/one_pass.py cfg1 2 > gpurun_out/sanitize_$T.txt 2>&1
echo "rc=$?" >> gpurun_out/sanitize_$T.txt
