#!/bin/bash
# 128-trial share (one rank of an 8-GPU run) under FRESH block caps
for cap in 0 2 3 4; do
  echo "== SAMU_K2_BPSM_FRESH=$cap"
  SAMU_K2_BPSM_FRESH=$cap python scripts/scaling_probe.py c5 128,256
done
