#!/bin/bash
# GPU parity suite, then the C5 first-step K2 breakdown under runtime switches: each argument is
# an environment assignment list ("" = none), e.g. "SAMU_K2_PDL=0"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_full.log 2>&1; tail -3 gpurun_out/gpu_tests_full.log
for v in "$@"; do
  echo "== $v"; env $v python scripts/k2_breakdown.py ${T:-1024} 2>&1 | grep -v "    dp="
done | tee gpurun_out/env_ab.txt
