#!/bin/bash
# Source-level ncu captures (instructions / stall samples per SASS address) of the three
# steady-state K2 launches of the bench step (third simulate call of profile_k2: FRESH, LEAN
# groups, LEAN singles); aggregate here with scripts/sass_lines.py against the same libsamu.so.
mkdir -p gpurun_out
T=${1:-1024}
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_simulate \
    python scripts/profile_k2.py c5 $T 3 2>/dev/null | grep k_simulate > gpurun_out/src_launches.csv
n=$(wc -l < gpurun_out/src_launches.csv)
for s in $(seq $((n - 3)) $((n - 1))); do
  ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section Occupancy \
      --clock-control none --import-source on -k regex:k_simulate -s $s -c 1 -f -o gpurun_out/k2_src_$s \
      python scripts/profile_k2.py c5 $T 3 > gpurun_out/ncu_src_$s.log 2>&1
done
ls -la gpurun_out
