#!/bin/bash
# Source-level K2 captures: a solo chain-summariser replica-sim (latency) and the steady-state
# launches of the bench step (throughput).
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_simulate -s 1 -c 1 -f -o gpurun_out/k2_item10 \
    python scripts/profile_item.py 10 1 1 > gpurun_out/ncu_item.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_simulate -s 1 -c 1 -f -o gpurun_out/k2_item7 \
    python scripts/profile_item.py 7 1 1 >> gpurun_out/ncu_item.log 2>&1
for s in 4 5 6; do
ncu --set full --clock-control none --import-source on -k regex:k_simulate -s $s -c 1 -f -o gpurun_out/k2_steady_$s \
    python scripts/profile_k2.py c5 1024 3 > gpurun_out/ncu_steady_$s.log 2>&1
done
ls -la gpurun_out
