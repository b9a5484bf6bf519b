#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/phase_timing.py cfg5 cfg3 > gpurun_out/phase_r2.txt 2>&1; echo rc=$? >> gpurun_out/phase_r2.txt
bash tools/box_nlprof.sh
