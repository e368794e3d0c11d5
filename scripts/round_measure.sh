#!/bin/bash
# Bench line + launch list + one full K2 capture at the bench configuration (run under gpurun).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --planner-trials 0 > gpurun_out/bench_under_ncu.log 2>&1
# K2 = one launch per mode (FRESH chain summariser, LEAN ensembling / routing): the FRESH launch
# from a two-launch capture, the LEAN one alone (its counters come back nan as the second launch)
ncu --set full --clock-control none --import-source on -k regex:k_simulate -s 2 -c 2 -f -o gpurun_out/k2_bench \
    python scripts/profile_k2.py c5 1024 2 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_simulate -s 3 -c 1 -f -o gpurun_out/k2_bench_lean \
    python scripts/profile_k2.py c5 1024 2 > gpurun_out/ncu_full_lean.log 2>&1
python scripts/ncu_summary.py gpurun_out/k2_bench.ncu-rep,gpurun_out/k2_bench_lean.ncu-rep gpurun_out/ncu_k2_summary.json c5 \
    "ncu --set full --clock-control none --import-source on -k regex:k_simulate -s 2 -c 2 (FRESH) and -s 3 -c 1 (LEAN) python scripts/profile_k2.py c5 1024 2"
cat gpurun_out/bench.json
