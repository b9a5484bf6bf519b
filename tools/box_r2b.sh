#!/bin/bash
# nl2 golden test, the default bench (with the nonlinear extra), then compute-sanitizer runs
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nonlinear.py -q -rfE -k golden > gpurun_out/nl_golden.log 2>&1; echo rc=$? >> gpurun_out/nl_golden.log
S=$(date +%s); timeout 1700 python bench.py > gpurun_out/bench_ours.json 2> gpurun_out/bench_ours.err; echo "ours rc=$? wall=$(( $(date +%s) - S ))" > gpurun_out/walls.txt
for spec in "racecheck cfg1" "synccheck cfg1" "memcheck cfg1" "racecheck nl1" "memcheck nl1"; do
  set -- $spec
  timeout 900 compute-sanitizer --tool $1 --print-limit 50 python tools/one_pass.py $2 2 > gpurun_out/sanitize_$1_$2.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$1_$2.txt
done
