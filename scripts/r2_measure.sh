#!/bin/bash
# Round-2 measurement under gpurun: GPU suite, bench line, ncu launch list, full K2 captures.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gpu_tests_full.log 2>&1
tail -15 gpurun_out/gpu_tests_full.log
if [ "${1:-all}" = "tests" ]; then exit 0; fi
bash scripts/round_measure.sh
