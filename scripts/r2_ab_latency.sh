#!/bin/bash
# GPU parity suite of the default build, then per variant (SAMU_DEFINES strings): the C5 first
# step at T = 1024 (breakdown), the trial-share scaling 1024 / 128 and the single replica-sim
# latencies of the chain summariser (the critical path of small shares); default rebuilt at the end
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_full.log 2>&1; tail -2 gpurun_out/gpu_tests_full.log
for v in "$@"; do
  SAMU_DEFINES="$v" python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)" || continue
  echo "== $v"
  python scripts/k2_breakdown.py 1024 2>&1 | grep -E "^all"
  python scripts/scaling_probe.py c5 1024,128 2>&1 | grep -E "^T="
  python scripts/item_latency.py 2>&1 | grep -E "node 10 dp 1"
done
python -c "from paper_2503_16893_b200 import build as B; B.build(force=True)"
