#!/bin/bash
# nonlinear (f4) GPU tests, then the whole GPU suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nonlinear.py -x -q -rfE > gpurun_out/nl_tests.log 2>&1; echo rc=$? >> gpurun_out/nl_tests.log
timeout 1500 python -m pytest tests -m gpu -x -q -rfE > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
