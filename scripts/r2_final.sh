#!/bin/bash
# End-of-round pass: GPU suite + smoke of the default build, K2 A/B variants (arguments, as in
# scripts/variants.sh), then the measurement set of scripts/round_measure.sh on the default build.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_final.log 2>&1; tail -2 gpurun_out/gpu_tests_final.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; tail -1 gpurun_out/smoke_final.log
if [ $# -gt 0 ]; then T=1024 bash scripts/variants.sh "$@" > gpurun_out/variants.txt 2>&1; grep -E "^==|^all" gpurun_out/variants.txt; fi
bash scripts/round_measure.sh > gpurun_out/round_measure.log 2>&1
python scripts/k2_breakdown.py 1024 > gpurun_out/breakdown_final.txt 2>&1; tail -1 gpurun_out/breakdown_final.txt
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('bench', d['ms_per_step'], d['value'], d['e2e']['value'], d['clocks'])"
