#!/bin/bash
# Last check of a build: every GPU test, the default bench line, the driver's exact bench command, the all-config table.
cd "$(dirname "$0")/.."
L=${1:-r02s8}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${L}_tests.log 2>&1; echo "tests_rc=$?"; tail -1 gpurun_out/${L}_tests.log
timeout 900 python bench.py > gpurun_out/${L}_bench.log 2>&1; echo "bench_rc=$?"; grep '^{' gpurun_out/${L}_bench.log | tail -1 | cut -c1-300
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${L}_bench_driver.log 2>&1; echo "bench_driver_rc=$?"; grep '^{' gpurun_out/${L}_bench_driver.log | tail -1 | cut -c1-300
python tools/bench_configs.py --steps 10 --warmup 5 > gpurun_out/${L}_bench_configs.log 2>&1; tail -7 gpurun_out/${L}_bench_configs.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
