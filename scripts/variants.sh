#!/bin/bash
# Build and time K2 variants on the GPU box: each argument is a SAMU_DEFINES string.
for v in "$@"; do
  SAMU_DEFINES="$v" python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)" || continue
  echo "== $v"; python scripts/k2_breakdown.py ${T:-1024} 2>&1 | grep -v "    dp="
done
python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)"
