#!/bin/bash
mkdir -p gpurun_out
SAMU_DEFINES=SAMU_K2_STATS python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)"
{ SAMU_DEFINES=SAMU_K2_STATS python scripts/k2_stats.py 1 10:1:1
  SAMU_DEFINES=SAMU_K2_STATS python scripts/k2_stats.py 64 10,7,0; } > gpurun_out/stats.txt 2>&1
cat gpurun_out/stats.txt
