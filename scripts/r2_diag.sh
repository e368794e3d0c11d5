#!/bin/bash
# K2 diagnostics: per-application / per-dp times, trial-share scaling, single-item latencies,
# event statistics (SAMU_K2_STATS build)
mkdir -p gpurun_out
{
echo "== breakdown 1024"; python scripts/k2_breakdown.py 1024
echo "== scaling"; python scripts/scaling_probe.py c5 1024,512,256,128
echo "== share128"; python scripts/share128.py 128
echo "== item latency"; python scripts/item_latency.py
SAMU_DEFINES=SAMU_K2_STATS python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)"
echo "== stats per node T=64"; SAMU_DEFINES=SAMU_K2_STATS python scripts/k2_stats.py 64 0,1,2,3,4,5,6,7,8,9,10
} > gpurun_out/diag.txt 2>&1
cat gpurun_out/diag.txt
