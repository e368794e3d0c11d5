#!/bin/bash
# Build and time K2 variants on the GPU box: each argument is a SAMU_DEFINES string.
# An argument "X|Y" sets SAMU_DEFINES=X and SAMU_NVCC_EXTRA=Y (extra nvcc flags).
for v in "$@"; do
  d="${v%%|*}"; x=""; [[ "$v" == *"|"* ]] && x="${v#*|}"
  SAMU_DEFINES="$d" SAMU_NVCC_EXTRA="$x" python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)" || continue
  echo "== $v"; python scripts/k2_breakdown.py ${T:-1024} 2>&1 | grep -v "    dp="
done
python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)"
