#!/bin/bash
# Bench line + launch list + full ncu captures of K2's steady-state launches at the bench
# configuration (run under gpurun).  The first simulate call after an app load groups every tp
# variant (no schedule-sharing hints yet); the steady state is the third call of
# scripts/profile_k2.py: one FRESH launch (chain summariser), one LEAN group launch and one
# LEAN single-candidate launch.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --planner-trials 0 --per-config "" > gpurun_out/bench_under_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_simulate \
    python scripts/profile_k2.py c5 1024 3 2>/dev/null | grep k_simulate > gpurun_out/k2_launches_3calls.csv
n=$(wc -l < gpurun_out/k2_launches_3calls.csv)
reps=""
for s in $(seq $((n - 3)) $((n - 1))); do
  ncu --set full --clock-control none --import-source on -k regex:k_simulate -s $s -c 1 -f -o gpurun_out/k2_steady_$s \
      python scripts/profile_k2.py c5 1024 3 > gpurun_out/ncu_steady_$s.log 2>&1
  reps="$reps,gpurun_out/k2_steady_$s.ncu-rep"
done
python scripts/ncu_summary.py "${reps#,}" gpurun_out/ncu_k2_summary.json c5 \
    "ncu --set full --clock-control none --import-source on -k regex:k_simulate -s S -c 1 python scripts/profile_k2.py c5 1024 3, S = the last three k_simulate launches (steady state: FRESH, LEAN groups, LEAN singles)"
cat gpurun_out/bench.json
