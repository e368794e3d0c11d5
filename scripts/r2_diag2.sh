#!/bin/bash
mkdir -p gpurun_out
{
echo "== share per node"; python scripts/share_nodes.py 1024
echo "== variants"; T=1024 bash scripts/variants.sh "" "SAMU_K2_MINB_LEAN=8" "SAMU_K2_MINB=7" "SAMU_K2_MINB=7 SAMU_K2_MINB_LEAN=8"
} > gpurun_out/diag2.txt 2>&1
cat gpurun_out/diag2.txt
