#!/bin/bash
# One build -> measure iteration under gpurun: GPU parity suite, per-application K2 times, bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_full.log 2>&1; grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/gpu_tests_full.log | head -20 > gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests_full.log >> gpurun_out/gpu_tests.log
cat gpurun_out/gpu_tests.log
python scripts/k2_breakdown.py ${1:-1024} 2>&1 | grep -v "    dp=" > gpurun_out/breakdown.txt
cat gpurun_out/breakdown.txt
if [ "${2:-bench}" = "bench" ]; then python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json | python -c "import json,sys; d=json.load(sys.stdin); print('bench ms/step', d['ms_per_step'], 'value', d['value'], 'k2 ms', d['roofline']['k2_ms_per_launch'])"; fi
