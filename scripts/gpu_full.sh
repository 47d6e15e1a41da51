#!/bin/bash
# Round-end style GPU pass: gpu tests, full default bench line, launch list.
cd "$(dirname "$0")/.."
L=${1:-full}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${L}_tests.log 2>&1; echo "tests_rc=$?"; tail -3 gpurun_out/${L}_tests.log
timeout 900 python bench.py > gpurun_out/${L}_bench.log 2>&1; echo "bench_rc=$?"; grep '^{' gpurun_out/${L}_bench.log | tail -1 | cut -c1-600
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${L}_launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${L}_ncu_launch.log 2>&1; echo "ncu_rc=$?"
