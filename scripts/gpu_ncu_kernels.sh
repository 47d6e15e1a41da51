#!/bin/bash
# ncu --set full of selected kernels of one bench step: KREGEX (default: rowfill|hist), COUNT launches.
cd "$(dirname "$0")/.."
L=${1:-r02h}
K=${KREGEX:-"regex:sp_rowfill|tc_hist"}
C=${COUNT:-4}
timeout 1200 ncu --set full --clock-control none --import-source on -k "$K" -c $C \
  -o gpurun_out/${L}_kern python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${L}_ncu_kern.log 2>&1
echo "ncu_rc=$?"; tail -3 gpurun_out/${L}_ncu_kern.log
