#!/bin/bash
mkdir -p gpurun_out
for it in "10 1 1" "7 1 1" "0 8 1"; do
  n=$(echo $it | tr ' ' '_')
  ncu --set full --clock-control none --import-source on -k regex:k_simulate -s 1 -c 1 -f -o gpurun_out/k2_item_$n \
      python scripts/profile_item.py $it > gpurun_out/ncu_item_$n.log 2>&1
done
ls gpurun_out
