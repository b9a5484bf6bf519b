#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nonlinear.py -q -rfE > gpurun_out/nl_tests.log 2>&1; echo rc=$? >> gpurun_out/nl_tests.log
bash tools/box_nlprof.sh
