#!/bin/bash
# Session-3 baseline: GPU tests, default bench line, ncu --set full of the S5 GEMM (3rd GEMM launch).
cd "$(dirname "$0")/.."
L=${1:-s3a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${L}_smi.txt
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/${L}_tests.log 2>&1; echo "tests_rc=$?"; tail -3 gpurun_out/${L}_tests.log
timeout 600 python bench.py --no-e2e > gpurun_out/${L}_bench.log 2>&1; echo "bench_rc=$?"; grep '^{' gpurun_out/${L}_bench.log | tail -1 | head -c 1500; echo
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm2 --launch-skip 2 -c 1 \
  -o gpurun_out/${L}_s5 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${L}_s5_ncu.log 2>&1
echo "ncu_rc=$?"; tail -2 gpurun_out/${L}_s5_ncu.log
