#!/bin/bash
# Round evidence: full default bench line, launch list, ncu --set full of the three K2T GEMMs.
cd "$(dirname "$0")/.."
L=${1:-r01c}
timeout 900 python bench.py > gpurun_out/${L}_bench.log 2>&1; echo "bench_rc=$?"; grep '^{' gpurun_out/${L}_bench.log | tail -1 | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${L}_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${L}_ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm2?_kernel -c 3 \
  -o gpurun_out/${L}_gemms python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${L}_ncu_full.log 2>&1
echo "ncu_full_rc=$?"
