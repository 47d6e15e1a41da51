#!/bin/bash
# ncu --set full of the S5 preparation kernels (histogram pass, row fill) on the bench's 8 buckets.
cd "$(dirname "$0")/.."
L=${1:-prep}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_hist_kernel|sp_rowfill|profiles_bulk" -c 4 \
  -o gpurun_out/${L} python tools/s5_bench.py --once > gpurun_out/${L}_ncu.log 2>&1
echo "ncu_rc=$?"; tail -2 gpurun_out/${L}_ncu.log
