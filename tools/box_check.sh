#!/bin/bash
# GPU-box round trip: the GPU test suite, short per-config benches, the full default bench.
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -rA ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
for c in ${QUICK_CFGS:-cfg3 cfg5}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-extras --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/quick_$c.json 2> gpurun_out/quick_$c.err
done
if [ -n "$FULL_BENCH" ]; then
  /usr/bin/time -v timeout 1700 python bench.py ${BENCH_ARGS} > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
fi
