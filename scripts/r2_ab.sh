#!/bin/bash
# A/B of K2 compile-time switches: per-application K2 times + solo summariser item instructions
mkdir -p gpurun_out
for v in "$@"; do
  d="${v%%|*}"
  SAMU_DEFINES="$d" python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)" || continue
  echo "== $v"
  python scripts/k2_breakdown.py ${T:-1024} 2>&1 | grep -v "    dp="
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --csv -k regex:k_simulate -s 1 -c 1 python scripts/profile_item.py 10 1 1 2>/dev/null | grep k_simulate | awk -F'","' '{print "item10", $(NF-3), $NF}'
done
python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)"
