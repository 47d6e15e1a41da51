#!/bin/bash
# ncu --set full of the three K2T GEMM launches of one bench step (S2a, S2d, S5).
cd "$(dirname "$0")/.."
L=${1:-gemm}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -c 3 \
  -o gpurun_out/${L} python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${L}_ncu.log 2>&1
echo "ncu_rc=$?"; tail -3 gpurun_out/${L}_ncu.log
