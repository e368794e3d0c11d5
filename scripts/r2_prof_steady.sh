#!/bin/bash
# Source-level captures of the steady-state K2 launches of the bench step (third call of
# profile_k2: FRESH, LEAN groups, LEAN singles) + a launch list of the same command
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_simulate python scripts/profile_k2.py c5 1024 3 2>/dev/null | grep k_simulate | awk -F'","' '{print $5, $NF}' > gpurun_out/steady_launches.txt
cat gpurun_out/steady_launches.txt
n1=$(head -4 gpurun_out/steady_launches.txt | wc -l)
for s in 7 8 9; do
ncu --set full --clock-control none --import-source on -k regex:k_simulate -s $s -c 1 -f -o gpurun_out/k2_steady_$s \
    python scripts/profile_k2.py c5 1024 3 > gpurun_out/ncu_steady_$s.log 2>&1
done
ls gpurun_out
