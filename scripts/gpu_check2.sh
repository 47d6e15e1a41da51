#!/bin/bash
# GPU round trip: full GPU test suite + one default bench line.
cd "$(dirname "$0")/.."
L=${1:-r02a}
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${L}_tests.log 2>&1; echo "tests_rc=$?"; tail -5 gpurun_out/${L}_tests.log
timeout 900 python bench.py > gpurun_out/${L}_bench.log 2>&1; echo "bench_rc=$?"; grep '^{' gpurun_out/${L}_bench.log | tail -1 | cut -c1-1500
