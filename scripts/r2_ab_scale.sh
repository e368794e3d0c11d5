#!/bin/bash
# A/B of K2 compile-time switches: per-application K2 times at T=1024 and the trial-share scaling
mkdir -p gpurun_out
for v in "$@"; do
  SAMU_DEFINES="$v" python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)" || continue
  echo "== $v"
  python scripts/k2_breakdown.py 1024 2>&1 | grep -v "    dp="
  python scripts/scaling_probe.py c5 1024,256,128
  python scripts/share128.py 128 | head -3
done
python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)"
