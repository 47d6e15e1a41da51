#!/bin/bash
# Round evidence: every GPU test, the default bench line (e2e + cpu_baseline),
# the ncu launch list of one step, ncu --set full of the three K2T GEMMs, N4 timings.
cd "$(dirname "$0")/.."
L=${1:-r02}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${L}_tests.log 2>&1; echo "tests_rc=$?"; tail -5 gpurun_out/${L}_tests.log
timeout 900 python bench.py > gpurun_out/${L}_bench.log 2>&1; echo "bench_rc=$?"; grep '^{' gpurun_out/${L}_bench.log | tail -1 | head -c 3000; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${L}_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${L}_ncu_launch.log 2>&1; echo "ncu_launch_rc=$?"
python tools/launch_shares.py gpurun_out/${L}_launches.csv > gpurun_out/${L}_shares.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm -c 3 \
  -o gpurun_out/${L}_gemms python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${L}_gemms_ncu.log 2>&1
echo "ncu_full_rc=$?"
python tools/tree_bench.py --n 12500 --compare > gpurun_out/${L}_tree.log 2>&1
python tools/tree_bench.py --buckets 8 >> gpurun_out/${L}_tree.log 2>&1; cat gpurun_out/${L}_tree.log | tail -4
