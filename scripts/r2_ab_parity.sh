#!/bin/bash
# GPU parity suite of the default build, then per-application K2 times of K2 variants
# (each argument a SAMU_DEFINES string, "" = default); the default build is restored at the end.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_full.log 2>&1; tail -3 gpurun_out/gpu_tests_full.log
T=${T:-1024} bash scripts/variants.sh "$@" > gpurun_out/variants.txt 2>&1; cat gpurun_out/variants.txt
